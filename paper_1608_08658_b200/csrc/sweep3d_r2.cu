// Instantiations of the 3-D sweep for radius 2 (space order 4).
#include "sweep3d.cuh"

namespace sfdb200 {
cudaError_t sweep3d_r2(const FieldGeom& g, const SweepConfig& cfg, const SweepMaps& m,
                       const SweepArgs& a, bool grad, cudaStream_t s, int* occ) {
    return grad ? detail::launch3d_r<2, true>(g, cfg, m, a, s, occ)
                : detail::launch3d_r<2, false>(g, cfg, m, a, s, occ);
}
}  // namespace sfdb200
