"""Cross-process z slabs on >= 2 GPUs (skipped on a one-GPU box): bench.py
--gpus 2 launches its own two ranks, runs cfg5 (strong scaling, each rank
generating its slab), checks its exchange against one GPU on a small problem
before timing, and reports the exchange it used -- the fused P2P path (CUDA
IPC peer stores + step counters) and, forced, the NCCL fallback."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
def test_two_ranks_bench_and_exchange(exchange):
    if _gpus() < 2:
        pytest.skip("needs two GPUs")
    env = dict(os.environ, SFDB200_EXCHANGE=exchange)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--time-steps", "10", "--steps", "1", "--warmup", "1", "--no-cpu", "--no-1gpu"],
                         capture_output=True, text=True, env=env, timeout=1800, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["workload"].startswith("cfg5")
    check = line["config"]["exchange_check"]
    assert check["ok"] and check["exchange"] == exchange
    assert line["config"]["exchange"].startswith("fused P2P" if exchange == "p2p" else "nccl")
