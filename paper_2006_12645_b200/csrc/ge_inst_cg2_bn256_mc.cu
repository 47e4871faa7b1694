// Instantiates the fused kernel family for BN = 256, CTA pairs in multicast clusters of two pairs
// (the pairs share B tiles through TMA multicast; no prologue variants).
#include "ge_launch.cuh"

namespace ge {
cudaError_t launch_cg2_bn256_mc(bool f32, int pro, const Maps& m, const Params& p, int grid,
                               cudaStream_t st) {
    return launch_bn_cg<256, 2, true>(f32, pro, m, p, grid, st);
}
}  // namespace ge
