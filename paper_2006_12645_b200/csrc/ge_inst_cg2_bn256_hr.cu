// Instantiates the fused kernel family for BN = 256, half-row CTA pairs (cta_group 2, M = 128: 64 rows per
// CTA; 6 dtype/prologue variants, layouts are runtime).
#include "ge_launch.cuh"

namespace ge {
cudaError_t launch_cg2_bn256_hr(bool f32, int pro, const Maps& m, const Params& p, int grid, cudaStream_t st) {
    return launch_bn_cg<256, 2, false, true>(f32, pro, m, p, grid, st);
}
}  // namespace ge
