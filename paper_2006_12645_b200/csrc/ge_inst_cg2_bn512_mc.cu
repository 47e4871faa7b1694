// Instantiates the fused kernel family for BN = 512, CTA pairs in multicast clusters of two pairs
// (the pairs share B tiles through TMA multicast; no prologue variants).
#include "ge_launch.cuh"

namespace ge {
cudaError_t launch_cg2_bn512_mc(bool f32, int pro, const Maps& m, const Params& p, int grid,
                               cudaStream_t st) {
    return launch_bn_cg<512, 2, true>(f32, pro, m, p, grid, st);
}
int clusters_mc(int bn) {
    return bn == 512 ? max_active_clusters<512, 2, true>(4) : max_active_clusters<256, 2, true>(4);
}
}  // namespace ge
