// Instantiates the fused kernel family for BN = 512, cta_group = 2 (24 layout/dtype/prologue variants).
#include "ge_launch.cuh"

namespace ge {
cudaError_t launch_cg2_bn512(bool a_mn, bool b_mn, bool f32, int pro, const Maps& m, const Params& p, int grid,
                            cudaStream_t st) {
    return launch_bn_cg<512, 2>(a_mn, b_mn, f32, pro, m, p, grid, st);
}
}  // namespace ge
