// ge_launch.cuh -- per-configuration launchers (instantiated in ge_inst_*.cu, dispatched by ge_api.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "ge_kernel.cuh"

namespace ge {

struct Maps {
    CUtensorMap a, b, c, p, q;      // p, q: second matmul of a sum of matmuls (unused otherwise)
};

// Smem bytes / ring stages of the (BN, CG) configuration, sx: with the Hadamard S stage, hr: half-row
// CTA pairs (host and device agree through Cfg).
int smem_bytes_for(int bn, int cg, bool sx = false, bool hr = false);
int stages_for(int bn, int cg, bool sx = false, bool hr = false);

template <int BN, bool OUT_F32, int PRO, int CG, bool MC = false, bool HR = false>
cudaError_t launch_one(const Maps& m, const Params& p, int grid, cudaStream_t st) {
    auto kern = ge_fused_kernel<BN, OUT_F32, PRO, CG, MC, HR>;
    constexpr int smem = Cfg<BN, CG, PRO == 2, HR>::kSmemBytes;
    static bool attr_done = false;   // benign race: setting the attribute twice is harmless
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(kernel_threads(OUT_F32, PRO != 0), 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    // CTA pairs; or, for split-K single-CTA tiles, one cluster per tile of `splits` CTAs (K-slices)
    // (MC: two CTA pairs sharing B tiles by TMA multicast)
    attr[0].val.clusterDim.x = MC ? 2 * CG : (CG == 1 && p.splits > 1) ? p.splits : CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // programmatic dependent launch: the kernel's prologue may overlap the previous kernel's tail
    // (the kernel waits on griddepcontrol.wait before touching global memory).  GE_PDL=0 disables.
    static const bool pdl = [] {
        const char* e = getenv("GE_PDL");
        return !(e && e[0] == '0');
    }();
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, m.a, m.b, m.c, m.p, m.q, p);
}

// Co-resident clusters of `cluster` CTAs of the (BN, CG) kernel on the current device (0 if the
// query fails); the split-K planner uses it (cluster scheduling is GPC-bound, not SM-count-bound).
template <int BN, int CG, bool MC = false>
int max_active_clusters(int cluster) {
    auto kern = ge_fused_kernel<BN, false, 0, CG, MC>;
    constexpr int smem = Cfg<BN, CG>::kSmemBytes;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster * 64, 1, 1);
    cfg.blockDim = dim3(kernel_threads(false, false), 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cluster;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// Dispatch over the 6 (OUT_F32, PRO in {0, 1, 2}) variants of one (BN, CG) configuration; the operand
// layouts travel in Params (a_mn / b_mn), and the host rejects the one unsupported layout (BN = 192
// CTA pairs stage 96 B rows per CTA: K-major B only, ge_api.cu validate()).
template <int BN, int CG, bool MC = false, bool HR = false>
cudaError_t launch_bn_cg(bool f32, int pro, const Maps& m, const Params& p, int grid, cudaStream_t st) {
    switch ((f32 ? 3 : 0) + pro) {
#define GE_CASE(F, P)                                                             \
    case (F ? 3 : 0) + P:                                                         \
        if constexpr (MC && P) return cudaErrorInvalidValue;                      \
        else return launch_one<BN, F, P, CG, MC, HR>(m, p, grid, st);
        GE_CASE(false, 0)
        GE_CASE(false, 1)
        GE_CASE(false, 2)
        GE_CASE(true, 0)
        GE_CASE(true, 1)
        GE_CASE(true, 2)
#undef GE_CASE
    }
    return cudaErrorInvalidValue;
}

// Defined in ge_inst_*.cu (one translation unit per configuration, compiled in parallel).
cudaError_t launch_cg1_bn64(bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg1_bn128(bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg1_bn192(bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg2_bn192(bool, int, const Maps&, const Params&, int, cudaStream_t);
int clusters_cg1(int bn, int cluster);     // max_active_clusters of the single-CTA kernels (ge_inst_cg1_*.cu)
int clusters_cg1_bn64(int cluster);
int clusters_cg1_bn128(int cluster);
int clusters_cg1_bn192(int cluster);
int clusters_cg1_bn256(int cluster);
cudaError_t launch_cg1_bn256(bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg2_bn128(bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg2_bn256(bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg2_bn512(bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg2_bn512_mc(bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg2_bn256_mc(bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg2_bn128_hr(bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg2_bn256_hr(bool, int, const Maps&, const Params&, int, cudaStream_t);
int clusters_mc(int bn);     // co-resident 4-CTA multicast clusters of the (bn, pair) kernel

}  // namespace ge
