// Instantiations of the 3-D sweep for radius 7 (space order 14).
#include "sweep3d.cuh"

namespace sfdb200 {
cudaError_t sweep3d_r7(const FieldGeom& g, const SweepConfig& cfg, const SweepMaps& m,
                       const SweepArgs& a, bool grad, cudaStream_t s, int* occ) {
    return grad ? detail::launch3d_r<7, true>(g, cfg, m, a, s, occ)
                : detail::launch3d_r<7, false>(g, cfg, m, a, s, occ);
}
}  // namespace sfdb200
