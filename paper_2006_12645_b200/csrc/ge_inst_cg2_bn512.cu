// Instantiates the fused kernel family for BN = 512, cta_group = 2 (6 dtype/prologue variants; layouts are runtime).
#include "ge_launch.cuh"

namespace ge {
cudaError_t launch_cg2_bn512(bool f32, int pro, const Maps& m, const Params& p, int grid,
                            cudaStream_t st) {
    return launch_bn_cg<512, 2>(f32, pro, m, p, grid, st);
}
}  // namespace ge
