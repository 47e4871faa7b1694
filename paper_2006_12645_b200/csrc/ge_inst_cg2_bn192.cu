// Instantiates the fused kernel family for BN = 192, cta_group = 2 (the K-major-B layout variants).
#include "ge_launch.cuh"

namespace ge {
cudaError_t launch_cg2_bn192(bool f32, int pro, const Maps& m, const Params& p, int grid,
                            cudaStream_t st) {
    return launch_bn_cg<192, 2>(f32, pro, m, p, grid, st);
}
}  // namespace ge
