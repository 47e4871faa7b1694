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

// Smem bytes / ring stages of the (BN, CG) configuration, sx: with the Hadamard S stage (host and
// device agree through Cfg).
int smem_bytes_for(int bn, int cg, bool sx = false);
int stages_for(int bn, int cg, bool sx = false);

template <int BN, bool A_MN, bool B_MN, bool OUT_F32, int PRO, int CG, bool MC = false>
cudaError_t launch_one(const Maps& m, const Params& p, int grid, cudaStream_t st) {
    auto kern = ge_fused_kernel<BN, A_MN, B_MN, OUT_F32, PRO, CG, MC>;
    constexpr int smem = Cfg<BN, CG, PRO == 2>::kSmemBytes;
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
    auto kern = ge_fused_kernel<BN, false, false, false, 0, CG, MC>;
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

// Dispatch over the 24 (A_MN, B_MN, OUT_F32, PRO in {0, 1, 2}) variants of one (BN, CG) configuration.
template <int BN, int CG, bool MC = false>
cudaError_t launch_bn_cg(bool a_mn, bool b_mn, bool f32, int pro, const Maps& m, const Params& p, int grid,
                         cudaStream_t st) {
    const int key = (a_mn ? 4 : 0) | (b_mn ? 2 : 0) | (f32 ? 1 : 0);
    switch (key * 3 + pro) {
// (BN = 192 with CTA pairs stages 96 B rows per CTA: only K-major B, whose TMA box takes any row
// count; an MN-major B stage is built from 64-column swizzle atoms.)
#define GE_CASE(K, AM, BM, F, P)                                                  \
    case K * 3 + P:                                                               \
        if constexpr ((BM && BN == 192 && CG == 2) || (MC && P)) return cudaErrorInvalidValue; \
        else return launch_one<BN, AM, BM, F, P, CG, MC>(m, p, grid, st);
#define GE_CASES(K, AM, BM, F) GE_CASE(K, AM, BM, F, 0) GE_CASE(K, AM, BM, F, 1) GE_CASE(K, AM, BM, F, 2)
        GE_CASES(0, false, false, false)
        GE_CASES(1, false, false, true)
        GE_CASES(2, false, true, false)
        GE_CASES(3, false, true, true)
        GE_CASES(4, true, false, false)
        GE_CASES(5, true, false, true)
        GE_CASES(6, true, true, false)
        GE_CASES(7, true, true, true)
#undef GE_CASES
#undef GE_CASE
    }
    return cudaErrorInvalidValue;
}

// Defined in ge_inst_*.cu (one translation unit per configuration, compiled in parallel).
cudaError_t launch_cg1_bn64(bool, bool, bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg1_bn128(bool, bool, bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg1_bn192(bool, bool, bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg2_bn192(bool, bool, bool, int, const Maps&, const Params&, int, cudaStream_t);
int clusters_cg1(int bn, int cluster);     // max_active_clusters of the single-CTA kernels (ge_inst_cg1_*.cu)
int clusters_cg1_bn64(int cluster);
int clusters_cg1_bn128(int cluster);
int clusters_cg1_bn192(int cluster);
int clusters_cg1_bn256(int cluster);
cudaError_t launch_cg1_bn256(bool, bool, bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg2_bn128(bool, bool, bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg2_bn256(bool, bool, bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg2_bn512(bool, bool, bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg2_bn512_mc(bool, bool, bool, int, const Maps&, const Params&, int, cudaStream_t);
cudaError_t launch_cg2_bn256_mc(bool, bool, bool, int, const Maps&, const Params&, int, cudaStream_t);
int clusters_mc(int bn);     // co-resident 4-CTA multicast clusters of the (bn, pair) kernel

}  // namespace ge
