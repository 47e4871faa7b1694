// Instantiates the fused kernel family for BN = 192, cta_group = 1 (6 dtype/prologue variants; layouts are runtime).
#include "ge_launch.cuh"

namespace ge {
cudaError_t launch_cg1_bn192(bool f32, int pro, const Maps& m, const Params& p, int grid,
                            cudaStream_t st) {
    return launch_bn_cg<192, 1>(f32, pro, m, p, grid, st);
}
int clusters_cg1_bn192(int cluster) { return max_active_clusters<192, 1>(cluster); }
}  // namespace ge
