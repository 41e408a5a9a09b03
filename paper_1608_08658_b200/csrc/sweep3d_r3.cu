// Instantiations of the 3-D sweep for radius 3 (space order 6).
#include "sweep3d.cuh"

namespace sfdb200 {
cudaError_t sweep3d_r3(const FieldGeom& g, const SweepConfig& cfg, const SweepMaps& m,
                       const SweepArgs& a, bool grad, cudaStream_t s, int* occ) {
    return grad ? detail::launch3d_r<3, true>(g, cfg, m, a, s, occ)
                : detail::launch3d_r<3, false>(g, cfg, m, a, s, occ);
}
}  // namespace sfdb200
