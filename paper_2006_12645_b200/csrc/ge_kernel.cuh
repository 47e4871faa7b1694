// ge_kernel.cuh -- the fused fp16 GEMM + bias + ReLU kernel for sm_100a.
//
// One persistent, warp-specialised kernel computes, per output tile,
//     S1:   acc = prologue(A) . B      (tcgen05.mma, fp32 accumulator in TMEM)
//     S2:   C = relu_add(acc, beta)    (epilogue warps, registers only)
// with no global write of acc (Sec. VII-A).  The paper's Volta design
// (register-staged 128-bit copies, swizzled smem, mma.sync macro-MMAs, smem reorder of
// accumulator fragments, one-tile-ahead prefetch: PAPER.md:749-941) is replaced by its sm_100a
// counterparts:
//   * TMA bulk-tensor loads with 128-B swizzle into an S-stage smem ring guarded by
//     full/empty mbarriers (prefetch S-1 k-blocks ahead instead of one);
//   * one thread issues tcgen05.mma (M = 128 per CTA, N = BN, K = 16) reading both operands
//     through smem descriptors; K-major vs MN-major is a descriptor bit, which serves the four
//     layout specialisations of PAPER.md:609-610 with one code path;
//   * the accumulator lives in Tensor Memory, double-buffered so the epilogue of tile t
//     overlaps the mainloop of tile t+1;
//   * the epilogue warps drain TMEM with tcgen05.ld (each thread owns one output row, so no
//     reorder exchange is needed), add bias, apply ReLU, round once to
//     fp16 (RNE) and store through a swizzled smem chunk with TMA;
//   * CG == 2 runs a CTA pair (cluster of 2) on a 256-row tile with tcgen05 cta_group::2: each
//     CTA stages half of A and half of B, halving per-SM operand traffic;
//   * an optional transform warpgroup applies the prologue op to the A stage in smem between
//     the TMA landing and the MMA (Sec. VII-C: "performed during the data
//     movement", smem footprint unchanged).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>

#include "ge_ptx.cuh"

namespace ge {

constexpr int kBK = 64;                 // K per pipeline stage (64 fp16 = one 128-B swizzle row)
constexpr int kUmmaK = 16;              // K per tcgen05.mma for 16-bit inputs
constexpr int kRowsPerCta = 128;        // accumulator rows per CTA (= TMEM lanes)
constexpr int kSmemBudget = 232448;     // 227 KB dynamic smem per CTA on sm_100
constexpr int kEpiWarps = 4;
constexpr int kXformWarps = 4;
constexpr int kStagingBytes = kEpiWarps * 2 * 32 * 128;   // 2 x (32 rows x 128 B) per epilogue warp

enum : int { BIAS_NONE = -1, BIAS_ROW = 0, BIAS_COL = 1, BIAS_FULL = 2 };
enum : int { PRO_NONE = 0, PRO_SCALE_K = 1, PRO_RELU = 2 };

struct Params {
    int M, N, K, batch;
    int num_m_tiles, num_n_tiles, num_k_blocks;
    int group_m;                    // raster group (m-tiles per group) for L2 locality
    long long num_tiles;
    // epilogue
    const __half* bias;
    int bias_mode;                  // BIAS_*
    int bias_vec;                   // 16-B vector loads of bias are legal
    long long ldbias, stride_bias;
    int relu;
    // prologue
    const float* scale;
    int prologue;                   // PRO_*
    int scale_vec;
    // output
    void* C;
    long long ldc, stride_c;
    int c_tma;                      // 1: TMA store; 0: st.global fallback
};

template <int BN, int CG>
struct Cfg {
    static constexpr int kTileM = kRowsPerCta * CG;
    static constexpr int kBRows = BN / CG;                        // B rows (N) staged per CTA
    static constexpr int kAStage = kRowsPerCta * kBK * 2;         // 16 KB
    static constexpr int kBStage = kBRows * kBK * 2;
    static constexpr int kStageBytes = kAStage + kBStage;
    static constexpr int kBarBytes = 1024;
    static constexpr int kStagesRaw = (kSmemBudget - 1024 - kStagingBytes - kBarBytes) / kStageBytes;
    static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
    static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kStagingBytes + kBarBytes;
    static constexpr int kTmemCols = 2 * BN;                       // double-buffered fp32 accumulator
    static_assert(kStages >= 2, "not enough smem for a pipeline");
    static_assert(kSmemBytes <= kSmemBudget, "smem overflow");
    static_assert(BN == 64 || BN == 128 || BN == 256, "BN");
};

__device__ __forceinline__ void decode_tile(const Params& p, long long t, int tile_m, int& b, int& mt, int& nt) {
    const long long per_batch = static_cast<long long>(p.num_m_tiles) * p.num_n_tiles;
    b = static_cast<int>(t / per_batch);
    const long long r = t - static_cast<long long>(b) * per_batch;
    const long long per_group = static_cast<long long>(p.group_m) * p.num_n_tiles;
    const int g = static_cast<int>(r / per_group);
    const int first_m = g * p.group_m;
    const int gsz = min(p.num_m_tiles - first_m, p.group_m);
    const int rr = static_cast<int>(r - static_cast<long long>(g) * per_group);
    mt = first_m + rr % gsz;
    nt = rr / gsz;
    (void)tile_m;
}

// fp32 epilogue value: v = acc + beta, then relu (y = v > 0 ? v : +0, DESIGN.md R-C5).
__device__ __forceinline__ float epi(float acc, float beta, int relu) {
    const float v = acc + beta;
    return relu ? (v > 0.0f ? v : 0.0f) : v;
}

template <int BN, bool A_MN, bool B_MN, bool OUT_F32, bool PRO, int CG>
__global__ void __launch_bounds__(PRO ? 384 : 256, 1)
ge_fused_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                const __grid_constant__ CUtensorMap tmap_c, const Params p) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
    using C_ = Cfg<BN, CG>;
    constexpr int S = C_::kStages;
    constexpr int W = OUT_F32 ? 32 : 64;                 // output columns per epilogue chunk (128 B rows)
    constexpr int NCHUNK = BN / W;
    constexpr uint32_t IDESC = ptx::make_idesc_f16(kRowsPerCta * CG, BN, A_MN, B_MN);

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + S * C_::kAStage;
    uint8_t* smem_c = smem_b + S * C_::kBStage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_c + kStagingBytes);
    uint64_t* full_bar = bars;                  // [S] TMA -> MMA (or -> transform)
    uint64_t* empty_bar = bars + S;             // [S] MMA -> TMA
    uint64_t* xform_bar = bars + 2 * S;         // [S] transform -> MMA (PRO only)
    uint64_t* tfull_bar = bars + 3 * S;         // [2] MMA -> epilogue
    uint64_t* tempty_bar = bars + 3 * S + 2;    // [2] epilogue -> MMA
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 4);

    const int warp = threadIdx.x / 32;
    const uint32_t lane = threadIdx.x % 32;
    const uint32_t rank = (CG == 2) ? ptx::cluster_ctarank() : 0;
    const bool leader = rank == 0;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tmap_a);
        ptx::tma_prefetch(&tmap_b);
        if (p.c_tma) ptx::tma_prefetch(&tmap_c);
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < S; ++s) {
            // pair mode without a transform: both CTAs' TMA bytes land on the leader's barrier and
            // only the leader's producer arrives (expecting both CTAs' bytes).
            ptx::mbar_init(&full_bar[s], 1);
            ptx::mbar_init(&empty_bar[s], 1);
            ptx::mbar_init(&xform_bar[s], kXformWarps * CG);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&tfull_bar[b], 1);
            ptx::mbar_init(&tempty_bar[b], kEpiWarps * CG);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc<CG>(tmem_slot, C_::kTmemCols);
    ptx::tc_fence_before();
    if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int cluster_id = blockIdx.x / CG;
    const int num_clusters = gridDim.x / CG;
    const int nkb = p.num_k_blocks;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            int s = 0;
            uint32_t phase = 0;
            for (long long t = cluster_id; t < p.num_tiles; t += num_clusters) {
                int b, mt, nt;
                decode_tile(p, t, C_::kTileM, b, mt, nt);
                const int m0 = mt * C_::kTileM + rank * kRowsPerCta;
                const int n0 = nt * BN + rank * C_::kBRows;
                for (int kb = 0; kb < nkb; ++kb) {
                    ptx::mbar_wait(&empty_bar[s], phase ^ 1);
                    const int k0 = kb * kBK;
                    uint8_t* sa = smem_a + s * C_::kAStage;
                    uint8_t* sb = smem_b + s * C_::kBStage;
                    if constexpr (CG == 2 && !PRO) {
                        // The peer's bytes can only land after the leader's barrier entered this
                        // phase (the peer first waits on its empty[s], released by the MMA that
                        // consumed the previous phase), so a transiently negative tx-count is safe.
                        if (leader) ptx::mbar_arrive_expect_tx(&full_bar[s], 2 * C_::kStageBytes);
                        if constexpr (A_MN) {
#pragma unroll
                            for (int i = 0; i < kRowsPerCta / 64; ++i)
                                ptx::tma_load_3d_pair(sa + i * 8192, &tmap_a, &full_bar[s], m0 + i * 64, k0, b);
                        } else {
                            ptx::tma_load_3d_pair(sa, &tmap_a, &full_bar[s], k0, m0, b);
                        }
                        if constexpr (B_MN) {
#pragma unroll
                            for (int i = 0; i < C_::kBRows / 64; ++i)
                                ptx::tma_load_3d_pair(sb + i * 8192, &tmap_b, &full_bar[s], n0 + i * 64, k0, b);
                        } else {
                            ptx::tma_load_3d_pair(sb, &tmap_b, &full_bar[s], k0, n0, b);
                        }
                    } else {
                        ptx::mbar_arrive_expect_tx(&full_bar[s], C_::kStageBytes);
                        if constexpr (A_MN) {
#pragma unroll
                            for (int i = 0; i < kRowsPerCta / 64; ++i)
                                ptx::tma_load_3d(sa + i * 8192, &tmap_a, &full_bar[s], m0 + i * 64, k0, b);
                        } else {
                            ptx::tma_load_3d(sa, &tmap_a, &full_bar[s], k0, m0, b);
                        }
                        if constexpr (B_MN) {
#pragma unroll
                            for (int i = 0; i < C_::kBRows / 64; ++i)
                                ptx::tma_load_3d(sb + i * 8192, &tmap_b, &full_bar[s], n0 + i * 64, k0, b);
                        } else {
                            ptx::tma_load_3d(sb, &tmap_b, &full_bar[s], k0, n0, b);
                        }
                    }
                    if (++s == S) { s = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA, one thread) =====================
        if (leader && lane == 0 && nkb > 0) {
            int s = 0;
            uint32_t phase = 0;
            int it = 0;
            const uint32_t a_base = ptx::smem_u32(smem_a);
            const uint32_t b_base = ptx::smem_u32(smem_b);
            for (long long t = cluster_id; t < p.num_tiles; t += num_clusters, ++it) {
                const int acc = it & 1;
                const uint32_t acc_phase = (it >> 1) & 1;
                ptx::mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = 0; kb < nkb; ++kb) {
                    ptx::mbar_wait(PRO ? &xform_bar[s] : &full_bar[s], phase);
                    ptx::tc_fence_after();
                    const uint32_t sa = a_base + s * C_::kAStage;
                    const uint32_t sb = b_base + s * C_::kBStage;
#pragma unroll
                    for (int k = 0; k < kBK / kUmmaK; ++k) {
                        // K-major: +32 B per K=16 step inside the 128-B swizzle row; SBO = 8 rows x 128 B.
                        // MN-major: +16 rows x 128 B per step; LBO = next 64-wide MN atom (64 x 128 B),
                        // SBO = next 8-row K group (1024 B).
                        const uint64_t ad = A_MN ? ptx::make_sw128_desc(sa + k * 2048, 8192, 1024)
                                                 : ptx::make_sw128_desc(sa + k * 32, 0, 1024);
                        const uint64_t bd = B_MN ? ptx::make_sw128_desc(sb + k * 2048, 8192, 1024)
                                                 : ptx::make_sw128_desc(sb + k * 32, 0, 1024);
                        ptx::mma_f16<CG>(d_tmem, ad, bd, IDESC, (kb | k) != 0);
                    }
                    ptx::mma_commit<CG>(&empty_bar[s]);          // smem slot free once these MMAs finish
                    if (kb == nkb - 1) ptx::mma_commit<CG>(&tfull_bar[acc]);
                    if (++s == S) { s = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp >= 4 && warp < 4 + kEpiWarps) {
        // ===================== epilogue: TMEM -> regs -> bias/ReLU -> smem -> TMA store ======
        const int q = warp & 3;                                  // TMEM lane quarter of this warp
        uint8_t* stage_c = smem_c + (warp - 4) * (2 * 32 * 128);
        int buf = 0;
        int it = 0;
        for (long long t = cluster_id; t < p.num_tiles; t += num_clusters, ++it) {
            int b, mt, nt;
            decode_tile(p, t, C_::kTileM, b, mt, nt);
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            const int row0 = mt * C_::kTileM + rank * kRowsPerCta + q * 32;   // first row of this warp
            const int row = row0 + lane;
            if (nkb > 0) {
                ptx::mbar_wait(&tfull_bar[acc], acc_phase);
                ptx::tc_fence_after();
            }
            float beta_col = 0.0f;
            if (p.bias_mode == BIAS_COL && row < p.M)
                beta_col = __half2float(p.bias[b * p.stride_bias + row]);
            const __half* bias_b = p.bias ? p.bias + b * p.stride_bias : nullptr;
#pragma unroll 1
            for (int c = 0; c < NCHUNK; ++c) {
                uint32_t v[W];
                if (nkb > 0) {
                    const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c * W;
                    ptx::tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
                    if constexpr (W == 64)
                        ptx::tmem_ld_32x32b_x32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
                    ptx::tmem_ld_wait();
                } else {
#pragma unroll
                    for (int e = 0; e < W; ++e) v[e] = 0u;
                }
                if (c == NCHUNK - 1 && nkb > 0) {
                    // accumulator buffer fully read: hand it back to the MMA warp
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if (CG == 2 && !leader) ptx::mbar_arrive_cluster(&tempty_bar[acc], 0);
                        else ptx::mbar_arrive(&tempty_bar[acc]);
                    }
                }
                const int col0 = nt * BN + c * W;
                // ---- bias + ReLU in fp32, convert, pack into 8 x 16-B vectors
                float f[W];
#pragma unroll
                for (int e = 0; e < W; ++e) f[e] = __uint_as_float(v[e]);
                if (p.bias_mode == BIAS_ROW) {
                    if (p.bias_vec && col0 + W <= p.N) {
#pragma unroll
                        for (int g = 0; g < W / 8; ++g) {
                            const uint4 hb = __ldg(reinterpret_cast<const uint4*>(bias_b + col0 + g * 8));
                            const __half2* h2 = reinterpret_cast<const __half2*>(&hb);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float2 bf = __half22float2(h2[e]);
                                f[g * 8 + 2 * e] = epi(f[g * 8 + 2 * e], bf.x, p.relu);
                                f[g * 8 + 2 * e + 1] = epi(f[g * 8 + 2 * e + 1], bf.y, p.relu);
                            }
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < W; ++e) {
                            const int col = col0 + e;
                            const float bv = col < p.N ? __half2float(bias_b[col]) : 0.0f;
                            f[e] = epi(f[e], bv, p.relu);
                        }
                    }
                } else if (p.bias_mode == BIAS_FULL) {
                    const __half* brow = bias_b + static_cast<long long>(row) * p.ldbias;
                    if (p.bias_vec && col0 + W <= p.N && row < p.M) {
#pragma unroll
                        for (int g = 0; g < W / 8; ++g) {
                            const uint4 hb = __ldg(reinterpret_cast<const uint4*>(brow + col0 + g * 8));
                            const __half2* h2 = reinterpret_cast<const __half2*>(&hb);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float2 bf = __half22float2(h2[e]);
                                f[g * 8 + 2 * e] = epi(f[g * 8 + 2 * e], bf.x, p.relu);
                                f[g * 8 + 2 * e + 1] = epi(f[g * 8 + 2 * e + 1], bf.y, p.relu);
                            }
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < W; ++e) {
                            const int col = col0 + e;
                            const float bv = (col < p.N && row < p.M) ? __half2float(brow[col]) : 0.0f;
                            f[e] = epi(f[e], bv, p.relu);
                        }
                    }
                } else {
                    const float bv = (p.bias_mode == BIAS_COL) ? beta_col : 0.0f;
#pragma unroll
                    for (int e = 0; e < W; ++e) f[e] = epi(f[e], bv, p.relu);
                }
                uint4 out[8];
                if constexpr (OUT_F32) {
#pragma unroll
                    for (int g = 0; g < 8; ++g)
                        out[g] = make_uint4(__float_as_uint(f[4 * g]), __float_as_uint(f[4 * g + 1]),
                                            __float_as_uint(f[4 * g + 2]), __float_as_uint(f[4 * g + 3]));
                } else {
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        uint32_t w4[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const __half2 h = __floats2half2_rn(f[8 * g + 2 * e], f[8 * g + 2 * e + 1]);
                            w4[e] = *reinterpret_cast<const uint32_t*>(&h);
                        }
                        out[g] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                    }
                }
                if (p.c_tma) {
                    // ---- swizzled staging chunk (32 rows x 128 B), then one TMA store per warp
                    if (lane == 0) ptx::bulk_wait_read<1>();        // the store that last used `buf` has read it
                    __syncwarp();
                    uint8_t* sc = stage_c + buf * (32 * 128);
#pragma unroll
                    for (int g = 0; g < 8; ++g)
                        *reinterpret_cast<uint4*>(sc + lane * 128 + ((g ^ (lane & 7)) * 16)) = out[g];
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::tma_store_3d(&tmap_c, sc, col0, row0, b);
                        ptx::bulk_commit();
                    }
                    buf ^= 1;
                } else if (row < p.M) {
                    // ---- st.global fallback for a C whose base/ldc breaks the TMA alignment rules
                    const long long off = static_cast<long long>(b) * p.stride_c + static_cast<long long>(row) * p.ldc;
                    if constexpr (OUT_F32) {
                        float* crow = reinterpret_cast<float*>(p.C) + off;
#pragma unroll
                        for (int e = 0; e < W; ++e)
                            if (col0 + e < p.N) crow[col0 + e] = f[e];
                    } else {
                        __half* crow = reinterpret_cast<__half*>(p.C) + off;
                        const __half* hv = reinterpret_cast<const __half*>(out);
#pragma unroll
                        for (int e = 0; e < W; ++e)
                            if (col0 + e < p.N) crow[col0 + e] = hv[e];
                    }
                }
            }
        }
        if (p.c_tma && lane == 0) ptx::bulk_wait<0>();
    } else if (PRO && warp >= 4 + kEpiWarps) {
        // ===================== prologue transform of the A stage (in place, in smem) ==========
        const int xt = threadIdx.x - (4 + kEpiWarps) * 32;      // 0..127
        int s = 0;
        uint32_t phase = 0;
        for (long long t = cluster_id; t < p.num_tiles; t += num_clusters) {
            for (int kb = 0; kb < nkb; ++kb) {
                ptx::mbar_wait(&full_bar[s], phase);
                uint8_t* sa = smem_a + s * C_::kAStage;
                const int k0 = kb * kBK;
#pragma unroll 2
                for (int i = 0; i < C_::kAStage / 16 / 128; ++i) {
                    const int o = (i * 128 + xt) * 16;               // byte offset of a 16-B chunk
                    uint4 x = *reinterpret_cast<uint4*>(sa + o);
                    __half2* h2 = reinterpret_cast<__half2*>(&x);
                    if (p.prologue == PRO_RELU) {
                        // a' = max(a, +0): clear every lane with the sign bit set (exact, -0 -> +0)
                        uint32_t* w = reinterpret_cast<uint32_t*>(&x);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            uint32_t u = w[e];
                            if (u & 0x8000u) u &= 0xFFFF0000u;
                            if (u & 0x80000000u) u &= 0x0000FFFFu;
                            w[e] = u;
                        }
                    } else {
                        float sc[8];
                        if constexpr (A_MN) {
                            // MN-major stage: 128-B rows are K, the 8 values share one k.
                            const int k = k0 + (o & 8191) / 128;
                            const float sv = k < p.K ? __ldg(p.scale + k) : 0.0f;
#pragma unroll
                            for (int e = 0; e < 8; ++e) sc[e] = sv;
                        } else {
                            // K-major stage: row m = o / 128, swizzled chunk -> logical k chunk.
                            const int r = o / 128;
                            const int kc = ((o / 16) & 7) ^ (r & 7);
                            const int k = k0 + kc * 8;
                            if (p.scale_vec && k + 8 <= p.K) {
                                const float4 s0 = __ldg(reinterpret_cast<const float4*>(p.scale + k));
                                const float4 s1 = __ldg(reinterpret_cast<const float4*>(p.scale + k + 4));
                                sc[0] = s0.x; sc[1] = s0.y; sc[2] = s0.z; sc[3] = s0.w;
                                sc[4] = s1.x; sc[5] = s1.y; sc[6] = s1.z; sc[7] = s1.w;
                            } else {
#pragma unroll
                                for (int e = 0; e < 8; ++e) sc[e] = (k + e < p.K) ? __ldg(p.scale + k + e) : 0.0f;
                            }
                        }
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float2 a = __half22float2(h2[e]);
                            h2[e] = __floats2half2_rn(sc[2 * e] * a.x, sc[2 * e + 1] * a.y);
                        }
                    }
                    *reinterpret_cast<uint4*>(sa + o) = x;
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if (CG == 2 && !leader) ptx::mbar_arrive_cluster(&xform_bar[s], 0);
                    else ptx::mbar_arrive(&xform_bar[s]);
                }
                if (++s == S) { s = 0; phase ^= 1; }
            }
        }
    }

    // ---- teardown: every role done; the allocating warp frees TMEM
    __syncwarp();
    ptx::tc_fence_before();
    if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<CG>(tmem_base, C_::kTmemCols);
    }
#endif
}

}  // namespace ge
