"""Verification harness on the B200 backend: the
reference's adjoint and Taylor tests (verify.cpp:123-297) run through the
device operators, with the fp32 bars of SURVEY §8(d)."""
import pytest

from paper_1608_08658_b200 import verify as V

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,order", [([41, 41], 2), ([41, 41], 4), ([41, 41], 8),
                                        ([21, 22, 23], 4), ([21, 22, 23], 8)])
def test_adjoint(dims, order):
    """acceptance.cpp:85-107: 2-D / 3-D x orders 2/4/8."""
    r = V.adjoint_test(V.AdjointConfig(interior=dims, space_order=order, nt=150))
    assert r.passed, r


def test_taylor_2d():
    r = V.taylor_test(V.TaylorConfig())
    assert r.passed, r
    assert sum(p.e0 >= 1e-4 * r.phi0 for p in r.points) >= 3


def test_taylor_3d():
    r = V.taylor_test(V.TaylorConfig(interior=[33, 33, 33], nbpml=8, sim_time=0.6,
                                     space_order=8))
    assert r.passed, r
