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

// Diagnostics counters (GE_DEBUG_STATS) exist only in the debug build (_build.py --debug-stats).
#ifndef GE_DBG
#define GE_DBG 0
#endif
// Stage release in pairs (one tcgen05.commit per two k-blocks) and an early readiness test of the
// next stage; both trim the fixed per-k-block issue cost that bounds small-N tiles.
#ifndef GE_PAIR_RELEASE
#define GE_PAIR_RELEASE 1
#endif
#ifndef GE_EARLY_TEST
#define GE_EARLY_TEST 0
#endif
#ifndef GE_EPI_ONE_WAITER
#define GE_EPI_ONE_WAITER 1
#endif
// Straight-line epilogue block for the measured configuration (ROW bias, ReLU); 0 = general code only.
// End of the epilogue: wait for the TMA stores' smem reads only (1) or for their completion (0).
#ifndef GE_END_WAIT_READ
#define GE_END_WAIT_READ 0
#endif
// Fast epilogue loop drains two TMEM chunks per iteration (both loads in flight together).
#ifndef GE_EPI_PAIRLD
#define GE_EPI_PAIRLD 0
#endif
// The fast epilogue also for the 512-wide pair tile (fp16 bias slice).
#ifndef GE_EPI_FAST512
#define GE_EPI_FAST512 1
#endif
#ifndef GE_EPI_FAST
#define GE_EPI_FAST 1
#endif
// The MMA warp polls its stage barriers without the try_wait suspend hint (a suspended warp wakes
// some time after the phase completes; the tensor pipe idles meanwhile).
#ifndef GE_MMA_SPIN
#define GE_MMA_SPIN 0
#endif
// Paired acquire: the two k-blocks of a ring-slot pair land on ONE full barrier (the even slot's)
// and the MMA warp waits once per pair (single-accumulator-half kernels without a prologue or
// multicast); halves the per-k-block barrier round trips that bound narrow tiles.
#ifndef GE_PAIR_ACQ
#define GE_PAIR_ACQ 0
#endif
// Producer as a converged warp issuing TMA through elect.sync (1), or lane 0 alone (0).
#ifndef GE_PROD_WARP
#define GE_PROD_WARP 1
#endif
// Split producer: warp 0 issues the A (and S) loads and arms the full barrier, warp 3 issues the B
// loads of the same stage in parallel (converged-warp producers only).
#ifndef GE_PROD_SPLIT
#define GE_PROD_SPLIT 0
#endif
// Early fill: single-CTA kernels issue their first ring pass of loads before the setup barrier
// (measured slower on 1024^3 and the split-K shapes, profiles/r02_ab_early_fill.txt: off).
#ifndef GE_EARLY_FILL
#define GE_EARLY_FILL 0
#endif
// Stage release group: the MMA warp commits once per GE_RELEASE_GROUP ring slots (2 = paired
// release; 4 where the ring holds a multiple of 4 stages).
#ifndef GE_RELEASE_GROUP
#define GE_RELEASE_GROUP 2
#endif
// tcgen05.fence::after_thread_sync after every full-barrier wait of the MMA warp (1), or only after
// the waits that order TMEM accesses (tile starts, accumulator-empty waits) (0): the TMA bytes a full
// barrier announces are async-proxy writes the MMA (async proxy) may read once the phase completed.
// Teardown cluster barrier without the release fence (execution sync only; see cluster_sync_relaxed).
#ifndef GE_TEARDOWN_RELAXED
#define GE_TEARDOWN_RELAXED 1
#endif
// griddepcontrol.launch_dependents ahead of griddepcontrol.wait (off the critical path)
#ifndef GE_EARLY_TRIGGER
#define GE_EARLY_TRIGGER 1
#endif
// the lean producer's griddepcontrol.wait sits right before its first TMA load
#ifndef GE_PROD_LATE_WAIT
#define GE_PROD_LATE_WAIT 1
#endif
#ifndef GE_DBG_NOLOAD_BUILD
#define GE_DBG_NOLOAD_BUILD 0
#endif
#ifndef GE_FENCE_FULL
#define GE_FENCE_FULL 1
#endif

namespace ge {

constexpr int kBK = 64;                 // K per pipeline stage (64 fp16 = one 128-B swizzle row)
constexpr int kUmmaK = 16;              // K per tcgen05.mma for 16-bit inputs
constexpr int kRowsPerCta = 128;        // accumulator rows per CTA (= TMEM lanes)
constexpr int kSmemBudget = 232448;     // 227 KB dynamic smem per CTA on sm_100
#ifndef GE_XFORM_WARPS
#define GE_XFORM_WARPS 4
#endif
constexpr int kXformWarps = GE_XFORM_WARPS;    // prologue transform warps (PRO kernels)
constexpr int kStagingSetBytes = 16384; // one staging buffer per epilogue warp: 8 x 2 KB (fp16) or 4 x 4 KB (fp32)

enum : int { BIAS_NONE = -1, BIAS_ROW = 0, BIAS_COL = 1, BIAS_FULL = 2 };
enum : int { PRO_NONE = 0, PRO_SCALE_K = 1, PRO_RELU = 2, PRO_HADAMARD = 3 };
enum : int { ACT_NONE = 0, ACT_RELU = 1, ACT_SIGMOID = 2, ACT_TANH = 3 };

struct Params {
    int M, N, K, batch;
    int num_m_tiles, num_n_tiles, num_k_blocks;
    int num_k_blocks1;              // k-blocks of A.B; the rest come from P.Q (sum of matmuls, Listing 4)
    int a_mn, b_mn;                 // operand majorness: A column-major (MN-major), B row-major (MN-major)
    int group_m;                    // raster group (m-tiles per group) for L2 locality
    long long num_tiles;
    // epilogue
    const __half* bias;
    int bias_mode;                  // BIAS_*
    int bias_vec;                   // 16-B vector loads of bias are legal
    long long ldbias, stride_bias;
    int act;                        // ACT_* applied at the root of the epilogue
    float bias_sign;                // +1 add, -1 subtract the bias
    int literal;                    // paper-literal rounding point (DESIGN.md R-C3): fp16(fp16(acc) +- bias)
    // prologue (PRO kernels): the TMA lands the A stage (and, for HADAMARD, the S stage) and the
    // transform warps rewrite A in place in smem before the MMA reads it
    const float* scale;             // SCALE_K: s[k], fp32
    int prologue;                   // PRO_*
    int scale_vec;
    int s_batched;                  // HADAMARD: 1 = one S per batch item, 0 = one S shared by all items
    // output
    void* C;
    long long ldc, stride_c;
    int c_tma;                      // 1: TMA store; 0: st.global path
    int c_vec;                      // st.global path may use 16-B vector stores (aligned rows)
    int c_trans;                    // swap-AB launch: the kernel computes
                                    // C^T = B^T A^T, so element (row, col) goes to C[col * ldc + row]
    int c_ext;                      // TMA store: inner extent of the C map (C's width rounded down to
                                    // 16 B; kernel columns, or kernel rows with c_trans)
    // L2 eviction priority of the operand loads / output stores (0 normal, 1 first, 2 last)
    int hint_a, hint_b, hint_c;
    // stream-K: tiles [dp_tiles, num_tiles) are split into sk_units
    // k-block units shared evenly by all clusters; partial accumulators go to sk_ws (one fp32
    // 128 x BN slot per CTA), announced through sk_flags (one per CTA, reset by the consumer)
    long long dp_tiles, sk_units;
    float* sk_ws;
    unsigned int* sk_flags;
    // split-K: splits > 1 (single-CTA tiles only) launches clusters of
    // `splits` CTAs per tile, CTA rank = K-slice; the fp32 partials are reduce-scattered through
    // distributed shared memory inside the cluster
    int splits;
    // diagnostics (GE_DEBUG_STATS): per-CTA blocked-cycle counters, or nullptr
    unsigned long long* dbg;
    // timing experiments, read only by the diagnostics build (GE_DBG = 1; the production kernels
    // compile these branches out, so no environment variable can change their results)
    int dbg_noload;                 // GE_DEBUG_NOLOAD: stop issuing TMA after the ring is full once
    int dbg_flags;                  // GE_DEBUG_FLAGS: 1 skip epilogue, 8 no epilogue math, 16 no stores
    unsigned long long* tl;         // timeline of CTA 0 (ge_debug_set_timeline), or nullptr
};

// Timeline stamps (%globaltimer ns) of CTA 0 per launch (diagnostics build): word 0 of the buffer
// counts launches, launch i writes words 1 + 16 i + TL_*.
enum : int { TL_ENTRY = 0, TL_SETUP = 1, TL_WAIT = 2, TL_FIRST_FULL = 3, TL_LAST_COMMIT = 4, TL_EPI_TFULL = 5,
             TL_EPI_END = 6, TL_TEARDOWN = 7, TL_EXIT = 8, TL_PROD_FIRST = 9, TL_PROD_LAST = 10,
             // producer's first k-block: tile decoded, empty slot acquired, expect_tx armed, A loads issued
             TL_P_DECODE = 11, TL_P_EMPTY = 12, TL_P_EXPECT = 13, TL_P_LOADA = 14, TL_N = 24,
             // setup phases (same slots as unused producer stamps of the lean loop)
             TL_S_BARINIT = 12, TL_S_ALLOC = 15,
             // MMA warp lane 0: after the work sequence is built, after the L2 policies
             TL_S_WORKSEQ = 16, TL_S_POLICY = 17 };

// Diagnostics slots per CTA (cycles blocked on each barrier; see ge_debug_read in the header).
enum : int { DBG_TOTAL = 0, DBG_PROD_EMPTY = 1, DBG_MMA_FULL = 2, DBG_MMA_TEMPTY = 3, DBG_EPI_TFULL = 4,
             DBG_EPI_REL0 = 5, DBG_EPI_REL1 = 6, DBG_EPI_TILE = 7, DBG_EPI_TMEMLD = 8,
             DBG_EPI_MATH = 9, DBG_SK_WAIT = 10, DBG_SK_WRITE = 11, DBG_SK_PIECES = 12, DBG_EPI_END = 13,
             DBG_MMA_END = 14, DBG_FIRST_MMA = 15,
             // %globaltimer (ns) of: kernel entry, end of setup (barriers, TMEM, cluster sync), the end
             // of this CTA's epilogue, and its exit (after teardown)
             DBG_G_ENTRY = 16, DBG_G_START = 17, DBG_G_EPI_END = 18, DBG_G_EXIT = 19,
             // prologue transform warps: cycles blocked on a landed stage, cycles rewriting stages
             DBG_XF_WAIT = 20, DBG_XF_WORK = 21,
             // MMA warp (single-accumulator-half kernels): cycles issuing the k-block MMAs, cycles in commits
             DBG_MMA_ISSUE = 22, DBG_MMA_COMMIT = 23,
             // TMA producer: cycles from a free slot to its loads issued, and the whole producer loop
             DBG_PROD_ISSUE = 24, DBG_PROD_TOTAL = 25,
             // split-K owner phases (summed over warps): TMEM load, partial adds, math, stores
             DBG_OWN_LD = 26, DBG_OWN_ADD = 27, DBG_OWN_MATH = 28, DBG_OWN_ST = 29, DBG_SLOTS = 30 };

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// SX: the Hadamard prologue's S tile is staged like A (same box, same swizzle) in its own ring slot.
// HR: half-row CTA pairs (cta_group::2 with M = 128: 64 rows per CTA, DESIGN.md "Half-row pair
// tiles"): each CTA stages a 64-row A block and half of B, and its 64 x BN accumulator occupies all
// 128 TMEM lanes over BN/2 columns (columns [0, BN/2) in lanes 0-63, [BN/2, BN) in lanes 64-127).
template <int BN, int CG, bool SX = false, bool HR = false>
struct Cfg {
    static constexpr int kRows = HR ? 64 : kRowsPerCta;                // A rows (tile rows) per CTA
    static constexpr int kBNT = HR ? BN / 2 : BN;                     // TMEM columns per accumulator
    static constexpr int kTileM = kRows * CG;
    static constexpr int kUmmaN = BN < 256 ? BN : 256;                // N of one tcgen05.mma
    static constexpr int kNHalves = BN / kUmmaN;                      // MMAs per K step (BN = 512: 2)
    static constexpr int kBBlockRows = kUmmaN / CG;                   // B rows per CTA per MMA
    static constexpr int kBBlockBytes = kBBlockRows * kBK * 2;
    static constexpr int kBRows = BN / CG;                            // B rows (N) staged per CTA
    static constexpr int kAStage = kRows * kBK * 2;                   // 16 KB (8 KB half-row)
    static constexpr int kBStage = kBRows * kBK * 2;
    static constexpr int kSStage = SX ? kAStage : 0;
    static constexpr int kStageBytes = kAStage + kBStage + kSStage;
    static constexpr int kBarBytes = 320;                             // (3S + 8) mbarriers + TMEM slot
    // Epilogue staging buffers per warp (double-buffered TMA stores).
    static constexpr int kStagingBufs = 2;
    static constexpr int kStagingBytes = kStagingBufs * kStagingSetBytes;
    // tile's ROW-bias slice: fp32 with the bias sign applied (no per-element conversion in the
    // epilogue) where the smem budget allows it, fp16 for the 256 x 512 pair tile (4 stages need it)
    static constexpr bool kBiasF32 = BN <= 256;
    static constexpr int kBiasBytes = BN * (kBiasF32 ? 4 : 2);
    static constexpr int kStagesRaw = (kSmemBudget - 1024 - kStagingBytes - kBiasBytes - kBarBytes) / kStageBytes;
    // paired stage release needs an even ring; a 3-stage ring (the Hadamard prologue's 64 KB stages)
    // keeps its third stage and releases stage by stage
    static constexpr int kStages = kStagesRaw > 8 ? 8 : (GE_PAIR_RELEASE && kStagesRaw >= 4 ? kStagesRaw & ~1 : kStagesRaw);
    static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kStagingBytes + kBiasBytes + kBarBytes;
    // fp32 accumulator in TMEM: double-buffered when two fit in the 512 columns, else one buffer
    // drained half by half (per-half barriers let the next tile's first MMAs start early).
    static constexpr int kAccStages = 2 * kBNT <= 512 ? 2 : 1;
    static constexpr int kTmemUsed = kAccStages * kBNT;
    // tcgen05.alloc takes a power of two >= 32 columns
    static constexpr int kTmemCols = kTmemUsed <= 32 ? 32 : kTmemUsed <= 64 ? 64 : kTmemUsed <= 128 ? 128
                                   : kTmemUsed <= 256 ? 256 : 512;
    static_assert(kStages >= 2, "not enough smem for a pipeline");

    static_assert(kBarBytes >= (3 * 8 + 8) * 8 + 4, "barrier area");
    static_assert(kSmemBytes <= kSmemBudget, "smem overflow");
    static_assert(BN == 64 || BN == 128 || BN == 192 || BN == 256 || (BN == 512 && CG == 2), "BN");
    static_assert(kTmemUsed <= 512, "TMEM");
    static_assert(!HR || (CG == 2 && BN <= 256 && BN >= 128), "half-row tiles are CTA pairs with BN 128 / 256");
};

__device__ __forceinline__ void decode_tile(const Params& p, long long t, int tile_m, int& b, int& mt, int& nt) {
    (void)tile_m;
    if (p.num_tiles <= 0x7fffffffll) {
        // 32-bit unsigned divisions (a 64-bit division is a long subroutine on the GPU and the
        // producer's first decode sits right after griddepcontrol.wait)
        const uint32_t ut = static_cast<uint32_t>(t);
        const uint32_t per_batch = static_cast<uint32_t>(p.num_m_tiles) * static_cast<uint32_t>(p.num_n_tiles);
        const uint32_t ub = ut / per_batch;
        const uint32_t r = ut - ub * per_batch;
        const uint32_t per_group = static_cast<uint32_t>(p.group_m) * static_cast<uint32_t>(p.num_n_tiles);
        const uint32_t g = r / per_group;
        const uint32_t first_m = g * static_cast<uint32_t>(p.group_m);
        const uint32_t rem_m = static_cast<uint32_t>(p.num_m_tiles) - first_m;
        const uint32_t gsz = rem_m < static_cast<uint32_t>(p.group_m) ? rem_m : static_cast<uint32_t>(p.group_m);
        const uint32_t rr = r - g * per_group;
        const uint32_t q = rr / gsz;
        b = static_cast<int>(ub);
        mt = static_cast<int>(first_m + (rr - q * gsz));
        nt = static_cast<int>(q);
        return;
    }
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
}

// Work of one cluster, in the order the producer and MMA process it: data-parallel tiles
// t = cid, cid + G, ... < dp_tiles, then the cluster's share [u0, u1) of the stream-K units
// (k-blocks of tiles dp_tiles .. num_tiles-1, tile-major), cut at tile boundaries.  The host keeps
// the stream-K tiles fewer than the clusters, so a share spans at most two pieces.
enum : int { PIECE_FULL = 0, PIECE_OWNER = 1, PIECE_PARTIAL = 2, PIECE_SPLIT = 3 };
struct Piece {
    long long tile;
    int kb0, kb1;                   // k-block range [kb0, kb1) of the tile
    int kind;                       // FULL (whole tile), OWNER (holds the tile's last k-block), PARTIAL
};

struct WorkSeq {
    long long dp_tiles, units, u0, u1;
    int cid, G, nkb, n_dp, n_sk, splits;
    __device__ __forceinline__ WorkSeq(const Params& p, int cid_, int G_) {
        cid = cid_;
        G = G_;
        nkb = p.num_k_blocks;
        splits = p.splits;
        if (splits > 1) {                   // split-K: one K-slice of one tile per cluster
            dp_tiles = units = u0 = u1 = 0;
            n_dp = 0;
            n_sk = (cid < p.num_tiles * splits) ? 1 : 0;
            return;
        }
        dp_tiles = p.dp_tiles;
        units = p.sk_units;
        // 32-bit division where the tile count allows it (64-bit division is a long subroutine and
        // this runs ahead of the setup barrier)
        if (dp_tiles <= cid) n_dp = 0;
        else if (dp_tiles <= 0x7fffffffll)
            n_dp = static_cast<int>((static_cast<uint32_t>(dp_tiles - cid) + static_cast<uint32_t>(G) - 1u) / static_cast<uint32_t>(G));
        else
            n_dp = static_cast<int>((dp_tiles - cid + G - 1) / G);
        n_sk = 0;
        u0 = u1 = 0;
        if (units > 0) {                    // stream-K launches only
            u0 = range_begin(cid);
            u1 = range_begin(cid + 1);
            if (u1 > u0) n_sk = (u1 > (u0 / nkb + 1) * nkb) ? 2 : 1;
        }
    }
    __device__ __forceinline__ long long range_begin(int c) const { return units * c / G; }
    __device__ __forceinline__ int count() const { return n_dp + n_sk; }
    __device__ __forceinline__ Piece get(int i) const {
        Piece pc;
        if (splits > 1) {
            const int j = cid % splits;
            pc.tile = cid / splits;
            pc.kb0 = j * nkb / splits;
            pc.kb1 = (j + 1) * nkb / splits;
            pc.kind = PIECE_SPLIT;
            return pc;
        }
        if (i < n_dp) {
            pc.tile = cid + static_cast<long long>(i) * G;
            pc.kb0 = 0;
            pc.kb1 = nkb;
            pc.kind = PIECE_FULL;
            return pc;
        }
        // With two pieces, the PARTIAL head of the next tile is processed first and the tail of the
        // current tile (OWNER or FULL) last, so every partial is published while its cluster's
        // MMAs are still busy and owners never wait at the end of the kernel.
        const long long split = (u0 / nkb + 1) * nkb;
        const long long u = (n_sk == 2) ? ((i == n_dp) ? split : u0) : u0;
        const long long rel = u / nkb;
        const long long end = u1 < (rel + 1) * nkb ? u1 : (rel + 1) * nkb;
        pc.tile = dp_tiles + rel;
        pc.kb0 = static_cast<int>(u - rel * nkb);
        pc.kb1 = static_cast<int>(end - rel * nkb);
        pc.kind = (pc.kb0 == 0 && pc.kb1 == nkb) ? PIECE_FULL : (pc.kb1 == nkb ? PIECE_OWNER : PIECE_PARTIAL);
        return pc;
    }
    // Partial pieces come first in every cluster's order, so a partial is never behind an owner
    // wait (no wait chains across clusters); the epilogue follows the MMA order.
    __device__ __forceinline__ int epi_index(int j) const { return j; }
    // Clusters holding the other pieces of stream-K tile `tile` are the NON-EMPTY ranges among
    // [first_contributor, cid): every cluster whose range ends after the tile's first unit.
    __device__ __forceinline__ int first_contributor(long long tile) const {
        const long long x0 = (tile - dp_tiles) * nkb;
        int c = cid;
        while (c > 0 && range_begin(c) > x0) --c;      // range_begin(c) <= x0 < range_end(c) unless empty
        return c;
    }
    __device__ __forceinline__ bool has_units(int c) const { return range_begin(c + 1) > range_begin(c); }
};

// Activation at the root of the pointwise epilogue, fp32 (DESIGN.md
// R-C7): ReLU y = v > 0 ? v : +0 (R-C5) and Tanh (tanhf) are IEEE/library-accurate; Sigmoid uses
// the fast __expf (ex2.approx) and the RN reciprocal, relative error ~1e-7, far below the
// fp16 output rounding the bound allows.
__device__ __forceinline__ void activate(float* f, int n, int act) {
    if (act == ACT_RELU) {
#pragma unroll
        for (int e = 0; e < n; ++e) f[e] = f[e] > 0.0f ? f[e] : 0.0f;
    } else if (act == ACT_SIGMOID) {
        // ex2.approx-based exp and a fast reciprocal: relative error ~1e-7, far below the fp16
        // output rounding (2^-11) the bound allows; saturates to 0 / 1 at the extremes.
#pragma unroll
        for (int e = 0; e < n; ++e) f[e] = __frcp_rn(1.0f + __expf(-f[e]));
    } else if (act == ACT_TANH) {
#pragma unroll
        for (int e = 0; e < n; ++e) f[e] = tanhf(f[e]);
    }
}

// Epilogue warps: 8 (two per TMEM lane quarter) for the fp16 fast path, 4 when the fp32 staging
// or the prologue transform warps need the room.  Non-epilogue warps: 0 TMA, 1 MMA, 2 TMEM, 3 idle.
__host__ __device__ constexpr int epi_warps(bool out_f32, bool pro) { return (out_f32 || pro) ? 4 : 8; }
__host__ __device__ constexpr int kernel_threads(bool out_f32, bool pro) {
    return 32 * (4 + epi_warps(out_f32, pro) + (pro ? kXformWarps : 0));
}

// MC: clusters of two CTA pairs stacked along M that share the B tile: each CTA loads half of its
// B block and multicasts it to the CTA at the same position in the other pair (a third less L2->SM
// operand traffic per flop); data-parallel tiles only (no prologue, stream-K or split-K).
// PRO: 0 no prologue; 1 in-place prologue op on the A stage (SCALE_K / RELU); 2 the same with the
// Hadamard tile S staged by TMA next to A (its second input dataspace).
// The operand layouts (K- or MN-major A and B) are runtime parameters (Params::a_mn / b_mn): one
// instantiation serves the four layout pairs, so a step that alternates layouts runs one kernel.
template <int BN, bool OUT_F32, int PRO, int CG, bool MC = false, bool HR = false>
__global__ void __launch_bounds__(kernel_threads(OUT_F32, PRO != 0), 1)
ge_fused_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                const __grid_constant__ CUtensorMap tmap_c, const __grid_constant__ CUtensorMap tmap_p,
                const __grid_constant__ CUtensorMap tmap_q, const Params p) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
    using C_ = Cfg<BN, CG, PRO == 2, HR>;
    constexpr int S = C_::kStages;
    constexpr int W = 32;                                // output columns per epilogue chunk (one tcgen05.ld)
    constexpr int NCHUNK = BN / W;
    constexpr int EPI_WARPS = epi_warps(OUT_F32, PRO != 0);
    constexpr int NH = C_::kNHalves;
    constexpr int HALF_COLS = BN / NH;
    constexpr bool kPairAcq = GE_PAIR_ACQ && !PRO && NH == 1 && !MC && GE_PAIR_RELEASE && S % 2 == 0;
    constexpr int kRel = (GE_PAIR_RELEASE && !kPairAcq && S % 2 == 0) ? ((GE_RELEASE_GROUP == 4 && S % 4 == 0) ? 4 : 2) : 1;
    const bool A_MN = p.a_mn != 0, B_MN = p.b_mn != 0;       // MN-major (row-major B / col-major A)
    const uint32_t IDESC = ptx::make_idesc_f16(C_::kRows * CG, C_::kUmmaN, A_MN, B_MN);

    const unsigned long long g_entry = GE_DBG ? globaltimer() : 0ull;

    unsigned long long* tl = nullptr;      // timeline slot of this launch (CTA 0, diagnostics build)
    (void)tl;
#if GE_DBG
#define GE_TL(k, cond) do { if (tl && (cond)) tl[k] = globaltimer(); } while (0)
#else
#define GE_TL(k, cond) do { } while (0)
#endif
    extern __shared__ uint8_t smem_raw[];
    // 1024-B alignment for the 128-B swizzle atoms, by pointer arithmetic on the __shared__ array so
    // the compiler keeps the shared address space (LDS/STS instead of generic LD/ST)
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + S * C_::kAStage;
    uint8_t* smem_s = smem_b + S * C_::kBStage;         // Hadamard S stages (PRO == 2 only)
    uint8_t* smem_c = smem_s + S * C_::kSStage;
    __half* smem_bias = reinterpret_cast<__half*>(smem_c + C_::kStagingBytes);
    float* smem_bias_f = reinterpret_cast<float*>(smem_c + C_::kStagingBytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_c + C_::kStagingBytes + C_::kBiasBytes);
    uint64_t* full_bar = bars;                  // [S] TMA -> MMA (or -> transform)
    uint64_t* empty_bar = bars + S;             // [S] MMA -> TMA
    uint64_t* xform_bar = bars + 2 * S;         // [S] transform -> MMA (PRO only)
    uint64_t* tfull_bar = bars + 3 * S;         // [acc] MMA -> epilogue
    uint64_t* tempty_bar = bars + 3 * S + 2;    // [acc * NH + half] epilogue -> MMA
    uint64_t* peer_ready_bar = bars + 3 * S + 6;  // split-K: every peer's ring is free to receive
    uint64_t* recv_full_bar = bars + 3 * S + 7;   // split-K: all partials addressed to this CTA landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 8);
#if GE_DBG
    int& tl_slot = reinterpret_cast<int*>(tmem_slot)[1];   // spare word of the barrier area
    if (threadIdx.x == 0) tl_slot = (p.tl && blockIdx.x == 0) ? static_cast<int>(atomicAdd(p.tl, 1ull)) : -1;
#endif
    const bool split_cluster = (CG == 1) && p.splits > 1;

    const int warp = threadIdx.x / 32;
    const uint32_t lane = threadIdx.x % 32;
    static_assert(!MC || (CG == 2 && !PRO), "multicast clusters: CTA pairs without a prologue");
    constexpr int CL = MC ? 2 * CG : CG;                 // CTAs per cluster
    constexpr int TILE_M = C_::kTileM * (MC ? 2 : 1);    // rows of one scheduled tile
    const uint32_t crank = (CG == 2) ? ptx::cluster_ctarank() : 0;
    const uint32_t rank = crank & 1;                     // rank inside the CTA pair
    const uint32_t pair = MC ? (crank >> 1) : 0;         // pair inside a multicast cluster
    const bool leader = rank == 0;
    const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2 * pair));

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tmap_a);
        ptx::tma_prefetch(&tmap_b);
        if (p.num_k_blocks1 < p.num_k_blocks) {
            ptx::tma_prefetch(&tmap_p);
            ptx::tma_prefetch(&tmap_q);
        }
        if (PRO == 2) ptx::tma_prefetch(&tmap_p);      // Hadamard S (the P slot: no sum of matmuls here)
        if (p.c_tma) ptx::tma_prefetch(&tmap_c);
    }
    // Work sequence and diagnostics registers (independent of the setup barrier below).
    const int cluster_id = blockIdx.x / CL;
    const int num_clusters = gridDim.x / CL;
    const int nkb = p.num_k_blocks;
    const WorkSeq work(p, cluster_id, num_clusters);
    const unsigned long long t_ws = GE_DBG ? globaltimer() : 0ull;
    // Diagnostics accumulate in registers (a global read-modify-write per barrier wait would add
    // an L2 round trip to every pipeline step) and are flushed once per thread at teardown.
    const bool dbg = GE_DBG && p.dbg != nullptr;
    unsigned long long dl[DBG_SLOTS];
#pragma unroll
    for (int i = 0; i < DBG_SLOTS; ++i) dl[i] = 0;
    long long t_start = 0;

    // ---- TMA producer loop, resumable (state kept across calls): `produce(n)` issues the loads of
    // at most n more k-blocks of this CTA's work sequence, waiting for free ring slots as needed.
    constexpr bool kSplitProd = GE_PROD_SPLIT && GE_PROD_WARP;
    int pr_wi = 0, pr_kb = 0, pr_s = 0;
    uint32_t pr_phase = 0;
    bool pr_open = false;
    int pr_issued = 0;                  // k-blocks issued: the first ring pass finds every slot free
    Piece pr_pc{};                      // the open piece and its decoded tile origin
    int pr_b = 0, pr_m0 = 0, pr_n0 = 0;
    const uint64_t pol_a = ptx::l2_policy(p.hint_a);
    const unsigned long long t_pol = GE_DBG ? globaltimer() : 0ull;
    const uint64_t pol_b = ptx::l2_policy(p.hint_b);
    // Opening a piece decodes its tile (integer divisions); the first one is opened before the setup
    // barrier and griddepcontrol.wait, so the first loads issue right after the wait.
    auto open_piece = [&]() {
        pr_pc = work.get(pr_wi);
        pr_kb = pr_pc.kb0;
        pr_open = true;
        int mt, nt;
        decode_tile(p, pr_pc.tile, TILE_M, pr_b, mt, nt);
        pr_m0 = mt * TILE_M + pair * C_::kTileM + rank * C_::kRows;
        pr_n0 = nt * BN + rank * C_::kBBlockRows;             // + h * kUmmaN per MMA block
    };
    auto produce = [&](int budget) {
        int& s = pr_s;
        uint32_t& phase = pr_phase;
        while (pr_wi < work.count() && budget > 0) {
            const int wi = pr_wi;
            if (!pr_open) open_piece();
            const Piece pc = pr_pc;
            const int b = pr_b, m0 = pr_m0, n0 = pr_n0;
            GE_TL(TL_P_DECODE, lane == 0 && wi == 0 && pr_kb == pc.kb0);
            for (; pr_kb < pc.kb1 && budget > 0; ++pr_kb, --budget) {
                const int kb = pr_kb;
                const bool first_pass = pr_issued < S;
                ++pr_issued;
                    // paired release: the MMA warp commits only the odd stage of each pair (that
                    // commit covers the even stage's MMAs too), so wait once per pair on it
                    if (first_pass) {
                        // slots of the first ring pass are free (their barriers' previous-phase parity)
                    } else if (kPairAcq) {
                        if ((s & 1) == 0) ptx::mbar_wait_timed(&empty_bar[s + 1], phase ^ 1, dbg && lane == 0, dl[DBG_PROD_EMPTY]);
                    } else if (s % kRel == 0) {
                        ptx::mbar_wait_timed(&empty_bar[s + kRel - 1], phase ^ 1, dbg && lane == 0, dl[DBG_PROD_EMPTY]);
                    }
                    // paired acquire: both slots of a pair signal the even slot's full barrier, armed
                    // once for the pair's bytes; a piece with an odd k-block count ends on a single
                    // (the odd slot is skipped, MMA and producer agree on the rule)
                    const bool pair_two = kPairAcq && (s & 1) == 0 && kb + 1 < pc.kb1;
                    uint64_t* const fb = kPairAcq ? &full_bar[s & ~1] : &full_bar[s];
                    const bool arm = !kPairAcq || (s & 1) == 0;
                    const uint32_t n_sub = pair_two ? 2u : 1u;
                    const long long tp0 = dbg ? clock64() : 0;
                    // sum of matmuls (Listing 4): k-blocks past A.B's come from P.Q, same accumulator
                    const bool second = kb >= p.num_k_blocks1;
                    const CUtensorMap* map_a = second ? &tmap_p : &tmap_a;
                    const CUtensorMap* map_b = second ? &tmap_q : &tmap_b;
                    const int k0 = (second ? kb - p.num_k_blocks1 : kb) * kBK;
                    uint8_t* sa = smem_a + s * C_::kAStage;
                    uint8_t* sb = smem_b + s * C_::kBStage;
                    if (GE_DBG && p.dbg_noload && (wi != 0 || kb >= S)) {
                        // timing experiment (GE_DEBUG_NOLOAD): operands stay resident, results invalid
                        if ((CG == 1 || leader) && (!GE_PROD_WARP || lane == 0) && warp == 0) ptx::mbar_arrive(&full_bar[s]);
                        if (++s == S) { s = 0; phase ^= 1; }
                        continue;
                    }
                    GE_TL(TL_P_EMPTY, lane == 0 && wi == 0 && kb == pc.kb0);
                    auto expect = [&](uint32_t bytes) {
                        if (GE_PROD_WARP) ptx::mbar_arrive_expect_tx_elect(fb, bytes);
                        else ptx::mbar_arrive_expect_tx(fb, bytes);
                    };
                    // split producer: warp 0 arms the barrier and loads A (and S), warp 3 loads B; bytes
                    // landing before the arm only make the tx-count transiently negative (the phase
                    // still needs warp 0's arrival)
                    const bool do_a = !kSplitProd || warp == 0, do_b = !kSplitProd || warp == 3;
                    if constexpr (CG == 2 && !PRO) {
                        // The peer's bytes can only land after the leader's barrier entered this
                        // phase (the peer first waits on its empty[s], released by the MMA that
                        // consumed the previous phase), so a transiently negative tx-count is safe.
                        if (leader && arm && do_a) expect(2 * n_sub * C_::kStageBytes);
                    } else {
                        // single CTAs, and every CTA of a prologue pair: its own transform warps wait
                        // for its own stage
                        if (arm && do_a) expect(n_sub * C_::kStageBytes);
                    }
                    auto load = [&](void* dst, const CUtensorMap* map, int c0, int c1, uint64_t pol, int cb) {
                        if (GE_PROD_WARP) {
                            if constexpr (CG == 2 && !PRO) ptx::tma_load_3d_pair_elect(dst, map, fb, c0, c1, cb);
                            else ptx::tma_load_3d_elect(dst, map, fb, c0, c1, cb);
                        } else {
                            if constexpr (CG == 2 && !PRO) ptx::tma_load_3d_pair(dst, map, fb, c0, c1, cb, pol);
                            else ptx::tma_load_3d(dst, map, fb, c0, c1, cb, pol);
                        }
                    };
                    // A, and the Hadamard tile S with A's box and swizzle (element-aligned with A in smem)
                    auto load_a = [&](uint8_t* dst, const CUtensorMap* map, int cb) {
                        if (A_MN) {
#pragma unroll
                            for (int i = 0; i < C_::kRows / 64; ++i) load(dst + i * 8192, map, m0 + i * 64, k0, pol_a, cb);
                        } else {
                            load(dst, map, k0, m0, pol_a, cb);
                        }
                    };
                    GE_TL(TL_P_EXPECT, lane == 0 && wi == 0 && kb == pc.kb0);
                    if (do_a) {
                        load_a(sa, map_a, b);
                        GE_TL(TL_P_LOADA, lane == 0 && wi == 0 && kb == pc.kb0);
                        if constexpr (PRO == 2) load_a(smem_s + s * C_::kSStage, &tmap_p, p.s_batched ? b : 0);
                    }
#pragma unroll
                    for (int h = 0; h < NH && do_b; ++h) {
                        uint8_t* sbh = sb + h * C_::kBBlockBytes;
                        const int nh = n0 + h * C_::kUmmaN;
                        if constexpr (MC) {
                            // this CTA's 64-row half `pair` of the block, to both pairs' CTAs of rank `rank`
                            // (an MN-major half is one 64-wide swizzle atom; the K-major map's box is 64 rows)
                            const uint16_t mask = static_cast<uint16_t>((1u << rank) | (1u << (rank + 2)));
                            const int c0 = B_MN ? nh + pair * 64 : k0, c1 = B_MN ? k0 : nh + pair * 64;
                            if (GE_PROD_WARP) ptx::tma_load_3d_pair_mc_elect(sbh + pair * 8192, map_b, &full_bar[s], c0, c1, b, mask);
                            else ptx::tma_load_3d_pair_mc(sbh + pair * 8192, map_b, &full_bar[s], c0, c1, b, mask, pol_b);
                        } else if (B_MN) {
#pragma unroll
                            for (int i = 0; i < C_::kBBlockRows / 64; ++i)
                                load(sbh + i * 8192, map_b, nh + i * 64, k0, pol_b, b);
                        } else {
                            load(sbh, map_b, k0, nh, pol_b, b);
                        }
                    }
                    if (dbg && lane == 0) dl[DBG_PROD_ISSUE] += static_cast<unsigned long long>(clock64() - tp0);
                    GE_TL(TL_PROD_FIRST, lane == 0 && wi == 0 && kb == pc.kb0);
                    GE_TL(TL_PROD_LAST, lane == 0);
                    if (kPairAcq && (s & 1) == 0 && !pair_two) ++s;   // single at the end of a piece
                    if (++s == S) { s = 0; phase ^= 1; }
            }
            if (pr_kb >= pc.kb1) {
                ++pr_wi;
                pr_open = false;
            }
        }
    };
    // Early fill (single-CTA tiles): warp 0 initialises the barriers and issues the first ring pass
    // of loads right away, so their latency overlaps the TMEM allocation and the setup barrier (the
    // TMA touches only this CTA's barriers; pairs and multicast clusters signal peer barriers and
    // must wait for the cluster barrier).
    constexpr bool kEarly = GE_EARLY_FILL && CG == 1 && !MC && !kSplitProd;
    // lean producer loop for every configuration except the dev-flag variants (paired acquire,
    // split producer, early fill) and the diagnostics build's no-load experiment
#ifndef GE_LEAN_PROD
#define GE_LEAN_PROD 1
#endif
    constexpr bool kLeanProd = GE_LEAN_PROD && !kPairAcq && !kSplitProd && !kEarly && !GE_DBG_NOLOAD_BUILD;
    if (warp == (kEarly ? 0 : 1)) {
        // one barrier per lane (the ring has at most 8 stages: 3 x 8 + 8 <= 32 barriers)
        static_assert(3 * S + 8 <= 32, "barrier init: one per lane");
        if (lane < S) {
            // pair mode without a transform: both CTAs' TMA bytes land on the leader's barrier and
            // only the leader's producer arrives (expecting both CTAs' bytes).
            ptx::mbar_init(&full_bar[lane], 1);
            ptx::mbar_init(&empty_bar[lane], MC ? 2 : 1);   // MC: both pairs' MMAs read stage s's B
            ptx::mbar_init(&xform_bar[lane], kXformWarps * CG);
        } else if (lane < S + 2) {
            ptx::mbar_init(&tfull_bar[lane - S], 1);
        } else if (lane < S + 6) {
            ptx::mbar_init(&tempty_bar[lane - S - 2], EPI_WARPS * CG);
        } else if (lane == S + 6) {
            ptx::mbar_init(peer_ready_bar, split_cluster ? p.splits - 1 : 1);
        } else if (lane == S + 7) {
            ptx::mbar_init(recv_full_bar, 1);
        }
        ptx::fence_mbar_init();
    }
    if (kEarly && warp == 0) {
        __syncwarp();
        ptx::grid_dependency_wait();                 // inputs may come from the previous kernel
        if (GE_PROD_WARP || lane == 0) produce(S);
    }
    if ((warp == 0 || (kSplitProd && warp == 3)) && !kEarly && work.count() > 0) open_piece();
    if (warp == 2) ptx::tmem_alloc<CG>(tmem_slot, C_::kTmemCols);
    // setup-phase stamps (diagnostics build), written once the launch's timeline slot is known
    const unsigned long long t_setup_phase = (GE_DBG && (warp == 1 || warp == 2)) ? globaltimer() : 0ull;
    (void)t_setup_phase;
    ptx::tc_fence_before();
    if (CG == 2 || split_cluster) ptx::cluster_sync(); else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
#if GE_DBG
    tl = tl_slot >= 0 ? p.tl + 1 + static_cast<long long>(tl_slot) * TL_N : nullptr;
    if (tl && threadIdx.x == 0) {
        tl[TL_ENTRY] = g_entry;
        tl[TL_SETUP] = globaltimer();
    }
    if (tl && lane == 0 && warp == 1) {
        tl[TL_S_BARINIT] = t_setup_phase;
        tl[TL_S_WORKSEQ] = t_ws;
        tl[TL_S_POLICY] = t_pol;
    }
    if (tl && lane == 0 && warp == 2) tl[TL_S_ALLOC] = t_setup_phase;
#endif
    // Programmatic dependent launch: everything above (barrier init, TMEM allocation, descriptor
    // prefetch, cluster sync) overlapped the previous kernel's tail; wait for it to complete before
    // touching global memory, then let the next launch in the stream get scheduled.
#if GE_EARLY_TRIGGER
    // let the next launch in the stream get scheduled before waiting on the previous one: its CTAs
    // still wait (griddepcontrol.wait) for this grid's completion before touching memory.  The
    // lean producer waits by itself right before its first load (below), so the code ahead of that
    // load -- and its instruction-cache misses -- runs while the previous grid finishes.
    ptx::launch_dependents();
    if (!(kLeanProd && GE_PROD_LATE_WAIT && warp == 0)) ptx::grid_dependency_wait();
#else
    ptx::grid_dependency_wait();
    ptx::launch_dependents();
#endif
    GE_TL(TL_WAIT, threadIdx.x == 0);

    t_start = clock64();
    if (dbg && warp == 1 && lane == 0) {
        dl[DBG_G_ENTRY] = g_entry;
        dl[DBG_G_START] = globaltimer();
    }
    if (kLeanProd && warp == 0) {
        // ===================== TMA producer (lean loop) =====================
        // One thread, every loop variable derived from launch-uniform values so ptxas keeps them in
        // uniform registers, shared-window addresses precomputed, no elect / cache-hint operands:
        // the per-k-block issue path was the bound of narrow tiles (DESIGN.md "TMA producer issue
        // cost": a lean issue loop sustains ~220 B/ns per SM, the general one ~40).
        if (lane == 0 && work.count() > 0) {
            const uint32_t a_s0 = ptx::smem_u32(smem_a), b_s0 = ptx::smem_u32(smem_b), x_s0 = ptx::smem_u32(smem_s);
            const uint32_t fb0 = ptx::smem_u32(full_bar), eb0 = ptx::smem_u32(empty_bar);
            // every CTA arms its own stage, except CTA pairs without a transform: the leader expects
            // both CTAs' bytes (the peer's loads signal the leader's barrier)
            const bool arm = (CG == 1) || (PRO != 0) || leader;
            const uint32_t bytes = (CG == 2 && !PRO) ? 2u * C_::kStageBytes : static_cast<uint32_t>(C_::kStageBytes);
            const uint16_t mc_mask = static_cast<uint16_t>((1u << rank) | (1u << (rank + 2)));
            int stage = 0, issued = 0;
            uint32_t ph = 0;
            for (int wi = 0; wi < work.count(); ++wi) {
                if (wi > 0 || !pr_open) {
                    pr_wi = wi;
                    open_piece();
                }
                const int b = pr_b, m0 = pr_m0, n0 = pr_n0;
                const int kb0 = pr_pc.kb0, kb1 = pr_pc.kb1;
                for (int kb = kb0; kb < kb1; ++kb) {
                    GE_TL(TL_P_DECODE, wi == 0 && kb == kb0);
                    if (issued >= S && stage % kRel == 0) ptx::mbar_wait_u32(eb0 + 8u * (stage + kRel - 1), ph ^ 1u);
                    ++issued;
                    const uint32_t fb = fb0 + 8u * stage;
                    if (arm) ptx::mbar_expect_tx_u32(fb, bytes);
                    GE_TL(TL_P_EXPECT, wi == 0 && kb == kb0);
                    const bool second = kb >= p.num_k_blocks1;
                    const CUtensorMap* map_a = second ? &tmap_p : &tmap_a;
                    const CUtensorMap* map_b = second ? &tmap_q : &tmap_b;
                    const int k0 = (second ? kb - p.num_k_blocks1 : kb) * kBK;
                    if (GE_EARLY_TRIGGER && GE_PROD_LATE_WAIT && issued == 1) ptx::grid_dependency_wait();
                    auto ld = [&](uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2) {
                        if constexpr (CG == 2 && !PRO) ptx::tma_ld3_pair(dst, map, fb, c0, c1, c2);
                        else ptx::tma_ld3(dst, map, fb, c0, c1, c2);
                    };
                    auto ld_a = [&](uint32_t dst, const CUtensorMap* map, int cb) {
                        if (A_MN) {
#pragma unroll
                            for (int i = 0; i < C_::kRows / 64; ++i) ld(dst + i * 8192, map, m0 + i * 64, k0, cb);
                        } else {
                            ld(dst, map, k0, m0, cb);
                        }
                    };
                    ld_a(a_s0 + stage * C_::kAStage, map_a, b);
                    GE_TL(TL_P_LOADA, wi == 0 && kb == kb0);
                    if constexpr (PRO == 2) ld_a(x_s0 + stage * C_::kSStage, &tmap_p, p.s_batched ? b : 0);
                    const uint32_t sb = b_s0 + stage * C_::kBStage;
#pragma unroll
                    for (int h = 0; h < NH; ++h) {
                        const uint32_t sbh = sb + h * C_::kBBlockBytes;
                        const int nh = n0 + h * C_::kUmmaN;
                        if constexpr (MC) {
                            const int c0 = B_MN ? nh + pair * 64 : k0, c1 = B_MN ? k0 : nh + pair * 64;
                            ptx::tma_ld3_pair_mc(sbh + pair * 8192, map_b, fb, c0, c1, b, mc_mask);
                        } else if (B_MN) {
#pragma unroll
                            for (int i = 0; i < C_::kBBlockRows / 64; ++i) ld(sbh + i * 8192, map_b, nh + i * 64, k0, b);
                        } else {
                            ld(sbh, map_b, k0, nh, b);
                        }
                    }
                    GE_TL(TL_PROD_FIRST, wi == 0 && kb == kb0);
                    GE_TL(TL_PROD_LAST, true);
                    if (++stage == S) {
                        stage = 0;
                        ph ^= 1u;
                    }
                }
                pr_open = false;
            }
        }
    } else if (warp == 0 || (kSplitProd && warp == 3)) {
        // ===================== TMA producer =====================
        // GE_PROD_WARP: the whole warp runs the loop converged (warp-uniform state) and one elected
        // lane issues each TMA / expect_tx; otherwise lane 0 alone.  With the early fill the first
        // ring pass was issued before the setup barrier; this continues where it stopped.
        if (GE_PROD_WARP || lane == 0) produce(0x7fffffff);
        if (dbg && lane == 0) dl[DBG_PROD_TOTAL] = static_cast<unsigned long long>(clock64() - t_start);
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA, one thread) =====================
        if (leader && nkb > 0) {
            // The whole warp runs this loop converged (warp-uniform state, so the descriptors live
            // in uniform registers); one elected lane issues each tcgen05 instruction.  The tensor
            // pipe queues only about one MMA, so the code between consecutive MMAs (barrier wait,
            // fence, commit) is kept minimal: it shows up directly as tensor idle time.
            // stage s is ready when its TMA bytes landed (full) or, with a prologue, when the
            // transform warps of every CTA of the pair rewrote its A in place (xform)
            auto wait_ready = [&](int st, uint32_t ph, unsigned long long& acc) {
                uint64_t* bar = PRO ? &xform_bar[st] : &full_bar[st];
                if (GE_MMA_SPIN && !dbg) ptx::mbar_wait_spin(bar, ph);
                else ptx::mbar_wait_timed(bar, ph, dbg && lane == 0, acc);
            };
            const uint32_t a_base = ptx::smem_u32(smem_a);
            const uint32_t b_base = ptx::smem_u32(smem_b);
            int s = 0, it = 0;
            uint32_t phase = 0;
            bool next_ready = false;
            for (; it < work.count(); ++it) {
                const Piece pc = work.get(it);
                const int acc = (C_::kAccStages == 2) ? (it & 1) : 0;
                const uint32_t acc_phase = (C_::kAccStages == 2) ? ((it >> 1) & 1) : (it & 1);
                const uint32_t d_tmem = tmem_base + acc * C_::kBNT;
                if (dbg && lane == 0 && it == 0) dl[DBG_FIRST_MMA] = static_cast<unsigned long long>(clock64() - t_start);
                // K-major: +32 B per K=16 step inside the 128-B swizzle row; SBO = 8 rows x 128 B.
                // MN-major: +16 rows x 128 B per step; LBO = next 64-wide MN atom (64 x 128 B),
                // SBO = next 8-row K group (1024 B).  Descriptors of a stage are the stage-0 ones
                // plus the stage offset (the 14-bit address field cannot carry: smem < 256 KB).
                const uint64_t a_desc0 = ptx::make_sw128_desc(a_base, A_MN ? 8192 : 0, 1024);
                const uint64_t b_desc0 = ptx::make_sw128_desc(b_base, B_MN ? 8192 : 0, 1024);
                const uint64_t A_STEP = A_MN ? 2048 / 16 : 32 / 16;
                const uint64_t B_STEP = B_MN ? 2048 / 16 : 32 / 16;
                auto desc_a = [&](int stage) {
                    return a_desc0 + static_cast<uint64_t>((stage * C_::kAStage) >> 4);
                };
                auto desc_b = [&](int stage, int h) {
                    return b_desc0 + static_cast<uint64_t>((stage * C_::kBStage + h * C_::kBBlockBytes) >> 4);
                };
                auto release_stage = [&](int stage) {
                    // MC: the stage's B halves came from both pairs, so both pairs' producers wait for it
                    if (stage % kRel == kRel - 1) ptx::mma_commit_elect<CG>(&empty_bar[stage], MC ? 0xF : 0x3);
                };
                auto mma_half = [&](int stage, int kb, int h) {
                    ptx::mma_kblock<CG>(d_tmem + h * C_::kUmmaN, desc_a(stage), desc_b(stage, h), IDESC, kb != pc.kb0,
                                        A_STEP, B_STEP);
                };
                if constexpr (NH == 2) {
                    // Single 512-column accumulator, drained half by half by the epilogue.  Half-0
                    // MMAs start as soon as half 0 is drained; while half 1 is still being drained the
                    // half-1 MMAs of the first stages are deferred (their stages stay held) and caught
                    // up in order once it is free, so the drain overlaps up to S stages of MMA work.
                    int npend = 0, s_pend = s;
                    bool h1_free = false;
                    for (int kb = pc.kb0; kb < pc.kb1; ++kb) {
                        if (npend == S) {          // every stage is held: block until half 1 is drained
                            ptx::mbar_wait_timed(&tempty_bar[1], acc_phase ^ 1,
                                                 dbg && lane == 0, dl[DBG_MMA_TEMPTY]);
                            h1_free = true;
                        }
                        if (h1_free && npend > 0) {
                            ptx::tc_fence_after();
                            for (int i = 0; i < npend; ++i) {
                                const int st = (s_pend + i) % S;
                                mma_half(st, pc.kb0 + i, 1);
                                release_stage(st);
                            }
                            npend = 0;
                        }
                        wait_ready(s, phase, dl[DBG_MMA_FULL]);
                        GE_TL(TL_FIRST_FULL, lane == 0 && it == 0 && kb == pc.kb0);
                        ptx::tc_fence_after();
                        if (kb == pc.kb0) {
                            ptx::mbar_wait_timed(&tempty_bar[0], acc_phase ^ 1,
                                                 dbg && lane == 0, dl[DBG_MMA_TEMPTY]);
                            ptx::tc_fence_after();
                            h1_free = ptx::mbar_test(&tempty_bar[1], acc_phase ^ 1);
                            if (h1_free) ptx::tc_fence_after();
                            s_pend = s;
                        }
                        if (h1_free) {
                            ptx::mma_kblock2<CG>(d_tmem, desc_a(s), desc_b(s, 0), desc_b(s, 1), IDESC, kb != pc.kb0,
                                                 A_STEP, B_STEP);
                            release_stage(s);
                        } else {
                            mma_half(s, kb, 0);
                            ++npend;
                            h1_free = ptx::mbar_test(&tempty_bar[1], acc_phase ^ 1);
                        }
                        if (++s == S) { s = 0; phase ^= 1; }
                    }
                    if (npend > 0) {               // short tile: catch up before signalling the epilogue
                        ptx::mbar_wait_timed(&tempty_bar[1], acc_phase ^ 1,
                                             dbg && lane == 0, dl[DBG_MMA_TEMPTY]);
                        ptx::tc_fence_after();
                        for (int i = 0; i < npend; ++i) {
                            const int st = (s_pend + i) % S;
                            mma_half(st, pc.kb0 + i, 1);
                            release_stage(st);
                        }
                    }
                    ptx::mma_commit_elect<CG>(&tfull_bar[acc], pair_mask);
                    GE_TL(TL_LAST_COMMIT, lane == 0);
                } else if constexpr (kPairAcq) {
                    // paired acquire: one barrier wait and one commit per ring-slot pair
                    for (int kb = pc.kb0; kb < pc.kb1;) {
                        const bool two = kb + 1 < pc.kb1;
                        wait_ready(s, phase, dl[DBG_MMA_FULL]);
                        ptx::tc_fence_after();
                        if (kb == pc.kb0) {
                            ptx::mbar_wait_timed(&tempty_bar[acc], acc_phase ^ 1,
                                                 dbg && lane == 0, dl[DBG_MMA_TEMPTY]);
                            ptx::tc_fence_after();
                        }
                        mma_half(s, kb, 0);
                        if (two) mma_half(s + 1, kb + 1, 0);
                        ptx::mma_commit_elect<CG>(&empty_bar[s + 1], 0x3);   // frees both slots
                        kb += two ? 2 : 1;
                        if (kb == pc.kb1) ptx::mma_commit_elect<CG>(&tfull_bar[acc], pair_mask);
                        s += 2;
                        if (s == S) { s = 0; phase ^= 1; }
                    }
                } else {
                    for (int kb = pc.kb0; kb < pc.kb1; ++kb) {
                        if (!(GE_EARLY_TEST && next_ready)) wait_ready(s, phase, dl[DBG_MMA_FULL]);
                        GE_TL(TL_FIRST_FULL, lane == 0 && it == 0 && kb == pc.kb0);
                        if (GE_FENCE_FULL || PRO) ptx::tc_fence_after();
                        if (kb == pc.kb0) {
                            // first k-block of a tile: the epilogue must have drained this buffer
                            ptx::mbar_wait_timed(&tempty_bar[acc], acc_phase ^ 1,
                                                 dbg && lane == 0, dl[DBG_MMA_TEMPTY]);
                            ptx::tc_fence_after();
                        }
                        if (GE_EARLY_TEST) {
                            // readiness of the next stage, tested before this stage's MMAs are issued
                            // so the barrier round trip overlaps the issue
                            const int sn = s + 1 == S ? 0 : s + 1;
                            next_ready = ptx::mbar_test(PRO ? &xform_bar[sn] : &full_bar[sn], s + 1 == S ? phase ^ 1 : phase);
                        }
                        const long long ti0 = dbg ? clock64() : 0;
                        mma_half(s, kb, 0);
                        const long long ti1 = dbg ? clock64() : 0;
                        release_stage(s);                         // smem slot free once these MMAs finish
                        if (kb == pc.kb1 - 1) ptx::mma_commit_elect<CG>(&tfull_bar[acc], pair_mask);
                        GE_TL(TL_LAST_COMMIT, lane == 0 && kb == pc.kb1 - 1);
                        if (dbg && lane == 0) {
                            dl[DBG_MMA_ISSUE] += static_cast<unsigned long long>(ti1 - ti0);
                            dl[DBG_MMA_COMMIT] += static_cast<unsigned long long>(clock64() - ti1);
                        }
                        if (++s == S) { s = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp >= 4 && warp < 4 + EPI_WARPS) {
        // ===================== epilogue: TMEM -> regs -> bias/ReLU -> smem -> TMA store ======
        // EPI_WARPS / 4 column groups: warp e drains TMEM lane quarter (e % 4) for the 32-column
        // chunks c = h*CPH_ALL + j*NG + e/4 of each accumulator half h.
        const int e_idx = warp - 4;
        const int q = warp & 3;                                  // TMEM lane quarter of this warp
        const int grp = e_idx / 4;
        constexpr int NG = EPI_WARPS / 4;
        constexpr int ES = OUT_F32 ? 4 : 2;
        constexpr int ROWB = W * ES;                             // staged bytes per row: 64 (fp16) / 128 (fp32)
        constexpr int STG = 32 * ROWB;                           // one staging buffer (32 rows)
        constexpr int NV = ROWB / 16;                            // 16-B vectors per row
        constexpr int NWORD = ROWB / 4;                          // 32-bit words per row
        constexpr int CPH_ALL = (HR ? C_::kBNT : HALF_COLS) / W;  // 32-column TMEM chunks per accumulator half
        // half-row pairs: lanes 64-127 hold tile columns [BN/2, BN) (a chunk offset for quarters 2, 3)
        const int qc = HR ? (q >> 1) * (C_::kBNT / W) : 0;
        constexpr int CPH = CPH_ALL / NG;                        // ... owned by this warp
        // Single-buffered accumulator (BN = 512), fp16 out: compute all of this warp's chunks of a
        // half into packed registers first and release the half before any store, so the next
        // tile's MMAs restart as early as possible.  Otherwise drain chunk by chunk.
        constexpr bool BATCH = (C_::kAccStages == 1) && !OUT_F32 && NG == 2;
        constexpr int NBUF = C_::kStagingBufs;
        uint8_t* stage_c = smem_c + e_idx * (NBUF * STG);
        const uint64_t pol_c = ptx::l2_policy(p.hint_c);
        // ROW bias (staged in smem) or COL bias (one value per thread: swap-AB turns the ROW bias of
        // C into a COL bias of C^T), ReLU, single rounding
        const bool epi_fast = (C_::kBiasF32 || (GE_EPI_FAST512 && p.bias_sign > 0.0f)) && !p.literal && p.act == ACT_RELU &&
                              (p.bias_mode == BIAS_ROW || p.bias_mode == BIAS_COL) && !(GE_DBG && p.dbg_flags);
        int buf = 0;
        for (int jj = 0; jj < work.count(); ++jj) {
            const int it = work.epi_index(jj);
            const Piece pc = work.get(it);
            const long long t = pc.tile;
            int b, mt, nt;
            decode_tile(p, t, TILE_M, b, mt, nt);
            const int acc = (C_::kAccStages == 2) ? (it & 1) : 0;
            const uint32_t acc_phase = (C_::kAccStages == 2) ? ((it >> 1) & 1) : (it & 1);
            const int row0 = mt * TILE_M + pair * C_::kTileM + rank * C_::kRows + (HR ? (q & 1) : q) * 32;   // first row of this warp
            const int row = row0 + lane;
            const __half* bias_b = p.bias ? p.bias + b * p.stride_bias : nullptr;
            // Bias operands are fetched while this tile's MMAs still run (global loads would miss
            // the ~2 KB of L1 the smem carve-out leaves): the ROW slice goes to smem as fp32.
            float beta_col = 0.0f;
            if (p.bias_mode == BIAS_COL && row < p.M) beta_col = __half2float(bias_b[row]);
            if (p.bias_mode == BIAS_ROW && pc.kind != PIECE_PARTIAL) {
                ptx::named_bar_sync(1, EPI_WARPS * 32);            // previous tile's reads are done
                for (int i = threadIdx.x - 128; i < BN; i += EPI_WARPS * 32) {
                    const int col = nt * BN + i;
                    if constexpr (C_::kBiasF32) smem_bias_f[i] = col < p.N ? p.bias_sign * __half2float(bias_b[col]) : 0.0f;
                    else smem_bias[i] = col < p.N ? bias_b[col] : __float2half_rn(0.0f);
                }
                ptx::named_bar_sync(1, EPI_WARPS * 32);
            }
            // straight-line chunk loop of the measured configuration (see compute_fast)
            const bool fast_loop = GE_EPI_FAST && epi_fast && NH == 1 && !BATCH && pc.kind != PIECE_OWNER &&
                                   pc.kind != PIECE_PARTIAL && pc.kind != PIECE_SPLIT && nkb > 0;
            // One warp polls the accumulator barrier; the others sleep on a hardware named barrier
            // (8 polling warps would contend with the MMA and TMA threads for the mbarrier unit
            // during the whole mainloop).
            auto wait_acc = [&]() {
                if (GE_EPI_ONE_WAITER) {
                    if (e_idx == 0)
                        ptx::mbar_wait_timed(&tfull_bar[acc], acc_phase, dbg && lane == 0, dl[DBG_EPI_TFULL]);
                    ptx::named_bar_sync(3, EPI_WARPS * 32);
                } else {
                    ptx::mbar_wait_timed(&tfull_bar[acc], acc_phase, dbg && e_idx == 0 && lane == 0, dl[DBG_EPI_TFULL]);
                }
                ptx::tc_fence_after();
            };
            if (nkb > 0) wait_acc();
            GE_TL(TL_EPI_TFULL, e_idx == 0 && lane == 0);
            const long long t_epi0 = (dbg && e_idx == 0) ? clock64() : 0;
            const uint32_t tm_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * C_::kBNT;

            // TMEM columns of chunk c -> registers (zeros when K == 0)
            auto load = [&](const int c, uint32_t* v) {
                if (nkb > 0) {
                    ptx::tmem_ld_32x32b_x32(tm_row + c * W, v);
                } else {
#pragma unroll
                    for (int e = 0; e < W; ++e) v[e] = 0u;
                }
            };
            // hand accumulator half h back to the MMA warp (all of this warp's reads are done)
            auto release = [&](const int h) {
                if (nkb == 0) return;
                if (dbg && e_idx == 0 && lane == 0)
                    dl[h == 0 ? DBG_EPI_REL0 : DBG_EPI_REL1] += static_cast<unsigned long long>(clock64() - t_epi0);
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (CG == 2 && !leader) ptx::mbar_arrive_cluster(&tempty_bar[acc * NH + h], 2 * pair);
                    else ptx::mbar_arrive(&tempty_bar[acc * NH + h]);
                }
            };
            // The measured configuration (ROW bias staged as pre-signed fp32, ReLU, one rounding) as
            // a short straight-line block: paired fp32 adds (FADD2, IEEE RN like two FADDs), ReLU as
            // max(v, +0) (-0 and NaN -> +0, R-C5), one RNE pack per two outputs.  The last tile's
            // drain is exposed on single-wave shapes and was instruction-fetch bound (ncu: no_inst)
            // with the general code inline, so it also gets its own chunk loop below.
            auto compute_fast = [&](const int ct, const uint32_t* v, uint32_t* w) {
                const int c = ct + qc;                               // tile column chunk
                uint32_t r[W];
                if (p.bias_mode == BIAS_COL) {
                    const float bc = p.bias_sign * beta_col;
#pragma unroll
                    for (int e = 0; e < W / 2; ++e) ptx::add_f32x2(v[2 * e], v[2 * e + 1], bc, bc, r[2 * e], r[2 * e + 1]);
                } else if constexpr (C_::kBiasF32) {
                    const float4* bs = reinterpret_cast<const float4*>(smem_bias_f + c * W);  // broadcast reads
#pragma unroll
                    for (int g = 0; g < W / 4; ++g) {
                        const float4 bf = bs[g];
                        ptx::add_f32x2(v[4 * g], v[4 * g + 1], bf.x, bf.y, r[4 * g], r[4 * g + 1]);
                        ptx::add_f32x2(v[4 * g + 2], v[4 * g + 3], bf.z, bf.w, r[4 * g + 2], r[4 * g + 3]);
                    }
                } else {
                    // 512-wide tiles stage the slice as fp16 (no smem left for fp32); added bias only
                    const uint4* bs = reinterpret_cast<const uint4*>(smem_bias + c * W);       // broadcast reads
#pragma unroll
                    for (int g = 0; g < W / 8; ++g) {
                        const uint4 hb = bs[g];
                        const __half2* h2 = reinterpret_cast<const __half2*>(&hb);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float2 bf = __half22float2(h2[e]);
                            ptx::add_f32x2(v[8 * g + 2 * e], v[8 * g + 2 * e + 1], bf.x, bf.y, r[8 * g + 2 * e],
                                           r[8 * g + 2 * e + 1]);
                        }
                    }
                }
                if constexpr (OUT_F32) {
#pragma unroll
                    for (int e = 0; e < W; ++e) w[e] = __float_as_uint(fmaxf(__uint_as_float(r[e]), 0.0f));
                } else {
#pragma unroll
                    for (int e = 0; e < W / 2; ++e) {
                        const __half2 hh = __floats2half2_rn(fmaxf(__uint_as_float(r[2 * e]), 0.0f),
                                                             fmaxf(__uint_as_float(r[2 * e + 1]), 0.0f));
                        w[e] = *reinterpret_cast<const uint32_t*>(&hh);
                    }
                }
            };
            // S2 of Listing 1: v = acc + beta, relu, one RNE conversion; packed into NWORD words
            auto compute = [&](const int ct, const uint32_t* v, uint32_t* w) {
                if (GE_EPI_FAST && epi_fast) {
                    compute_fast(ct, v, w);
                    return;
                }
                const int c = ct + qc;                               // tile column chunk
                const int col0 = nt * BN + c * W;
                const float bsg = p.bias_sign;
                float f[W];
#pragma unroll
                for (int e = 0; e < W; ++e) f[e] = __uint_as_float(v[e]);
                // paper-literal reading: the accumulator is converted to fp16
                // before the pointwise op, and the fp16 add rounds again (fp32 add + RNE to fp16 is
                // the correctly rounded fp16 sum: 24 >= 2*11 + 2 bits, no double-rounding error)
                auto to_f16 = [&]() {
#pragma unroll
                    for (int e = 0; e < W; ++e) f[e] = __half2float(__float2half_rn(f[e]));
                };
                if (p.literal) to_f16();
                if (C_::kBiasF32 && p.bias_mode == BIAS_ROW) {
                    const float4* bs = reinterpret_cast<const float4*>(smem_bias_f + c * W);  // broadcast reads
#pragma unroll
                    for (int g = 0; g < W / 4; ++g) {
                        const float4 bf = bs[g];
                        f[4 * g] += bf.x;
                        f[4 * g + 1] += bf.y;
                        f[4 * g + 2] += bf.z;
                        f[4 * g + 3] += bf.w;
                    }
                } else if (p.bias_mode == BIAS_ROW) {
                    const uint4* bs = reinterpret_cast<const uint4*>(smem_bias + c * W);     // broadcast reads
#pragma unroll
                    for (int g = 0; g < W / 8; ++g) {
                        const uint4 hb = bs[g];
                        const __half2* h2 = reinterpret_cast<const __half2*>(&hb);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float2 bf = __half22float2(h2[e]);
                            f[g * 8 + 2 * e] += bsg * bf.x;
                            f[g * 8 + 2 * e + 1] += bsg * bf.y;
                        }
                    }
                } else if (p.bias_mode == BIAS_FULL) {
                    const __half* bsrc = bias_b + static_cast<long long>(row) * p.ldbias;
                    const bool in_row = row < p.M;
                    if (p.bias_vec && col0 + W <= p.N && in_row) {
#pragma unroll
                        for (int g = 0; g < W / 8; ++g) {
                            const uint4 hb = __ldg(reinterpret_cast<const uint4*>(bsrc + col0 + g * 8));
                            const __half2* h2 = reinterpret_cast<const __half2*>(&hb);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float2 bf = __half22float2(h2[e]);
                                f[g * 8 + 2 * e] += bsg * bf.x;
                                f[g * 8 + 2 * e + 1] += bsg * bf.y;
                            }
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < W; ++e) {
                            const int col = col0 + e;
                            const float bv = (col < p.N && in_row) ? __half2float(bsrc[col]) : 0.0f;
                            f[e] += bsg * bv;
                        }
                    }
                } else {
                    const float bv = (p.bias_mode == BIAS_COL) ? beta_col : 0.0f;
#pragma unroll
                    for (int e = 0; e < W; ++e) f[e] += bsg * bv;
                }
                if (p.literal && p.bias_mode != BIAS_NONE) to_f16();
                activate(f, W, p.act);
                if constexpr (OUT_F32) {
#pragma unroll
                    for (int e = 0; e < W; ++e) w[e] = __float_as_uint(f[e]);
                } else {
#pragma unroll
                    for (int e = 0; e < W / 2; ++e) {
                        const __half2 hh = __floats2half2_rn(f[2 * e], f[2 * e + 1]);
                        w[e] = *reinterpret_cast<const uint32_t*>(&hh);
                    }
                }
            };
            // element-wise st.global of this thread's row of chunk c: columns [lo, N) of it (normal), or,
            // swap-AB, the thread's row is a column of C and the 32 lanes of the warp hold 32 consecutive
            // C columns, so each store instruction writes one contiguous 64-B / 128-B segment of a C row
            auto store_scalar = [&](const int col0, const uint32_t* w, const int lo) {
                if (p.c_trans) {
                    const long long cb = static_cast<long long>(b) * p.stride_c + row;
#pragma unroll
                    for (int e = 0; e < W; ++e) {
                        if (col0 + e >= p.N) continue;
                        const long long o = cb + static_cast<long long>(col0 + e) * p.ldc;
                        if constexpr (OUT_F32) reinterpret_cast<float*>(p.C)[o] = __uint_as_float(w[e]);
                        else reinterpret_cast<__half*>(p.C)[o] = reinterpret_cast<const __half*>(w)[e];
                    }
                } else {
                    const long long off = static_cast<long long>(b) * p.stride_c + static_cast<long long>(row) * p.ldc;
#pragma unroll
                    for (int e = 0; e < W; ++e) {
                        if (col0 + e < lo || col0 + e >= p.N) continue;
                        if constexpr (OUT_F32) reinterpret_cast<float*>(p.C)[off + col0 + e] = __uint_as_float(w[e]);
                        else reinterpret_cast<__half*>(p.C)[off + col0 + e] = reinterpret_cast<const __half*>(w)[e];
                    }
                }
            };
            // packed row of chunk c -> C (TMA store through a swizzled staging chunk, or st.global)
            auto store = [&](const int ct, const uint32_t* w) {
                const int col0 = nt * BN + (ct + qc) * W;
                if (p.c_tma) {
                    // The swizzle matches the C tensor map: 128-B rows use SWIZZLE_128B (16-B chunk
                    // ^= row % 8), 64-B rows SWIZZLE_64B (chunk ^= (row / 2) % 4); both are
                    // bank-conflict-free for a warp's 16-B stores.
                    if (lane == 0) ptx::bulk_wait_read<NBUF - 1>(); // the store that last used `buf` has read it
                    __syncwarp();
                    uint8_t* sc = stage_c + buf * STG;
                    if (p.c_trans) {
                        // swap-AB: the warp's 32 x 32 block of C^T is a 32 x 32 block of C (rows col0..,
                        // columns row0..): staged transposed (smem row e = C row col0 + e, this lane's
                        // element at column lane), one 64-B / 128-B row segment per element index, then
                        // one TMA store into C's own tensor map (rows / columns past C clipped)
#pragma unroll
                        for (int e = 0; e < W; ++e) {
                            if constexpr (OUT_F32) {
                                const int pc = (lane >> 2) ^ (e & 7);
                                *reinterpret_cast<uint32_t*>(sc + e * ROWB + pc * 16 + (lane & 3) * 4) = w[e];
                            } else {
                                const int pc = (lane >> 3) ^ ((e >> 1) & 3);
                                *reinterpret_cast<uint16_t*>(sc + e * ROWB + pc * 16 + (lane & 7) * 2) =
                                    static_cast<uint16_t>((e & 1) ? (w[e >> 1] >> 16) : (w[e >> 1] & 0xFFFFu));
                            }
                        }
                    } else {
#pragma unroll
                        for (int g = 0; g < NV; ++g) {
                            const int pc = (ROWB == 128) ? (g ^ (lane & 7)) : (g ^ ((lane >> 1) & 3));
                            *reinterpret_cast<uint4*>(sc + lane * ROWB + pc * 16) =
                                make_uint4(w[4 * g], w[4 * g + 1], w[4 * g + 2], w[4 * g + 3]);
                        }
                    }
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if (p.c_trans) ptx::tma_store_3d(&tmap_c, sc, row0, col0, b, pol_c);
                        else ptx::tma_store_3d(&tmap_c, sc, col0, row0, b, pol_c);
                        ptx::bulk_commit();
                    }
                    buf = (buf + 1 == NBUF) ? 0 : buf + 1;
                    // The TMA store clips the inner dimension at 16-B granularity, so the map's inner
                    // extent is C's width rounded down to 16 B (c_ext) and the < 16 B ragged edge
                    // [c_ext, width) goes out element-wise (the caller's padding past C stays untouched)
                    if (p.c_trans) {
                        if (row >= p.c_ext && row < p.M) store_scalar(col0, w, 0);
                    } else if (col0 + W > p.c_ext && row < p.M) {
                        store_scalar(col0, w, p.c_ext);
                    }
                } else if (row < p.M) {
                    // st.global path: C whose base/ldc breaks the TMA alignment rules (scalar stores),
                    // or 16-B aligned rows written straight from registers (c_vec)
                    if (!p.c_trans && p.c_vec && col0 + W <= p.N) {
                        const long long off = static_cast<long long>(b) * p.stride_c + static_cast<long long>(row) * p.ldc;
                        uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(p.C) + (off + col0) * ES);
#pragma unroll
                        for (int g = 0; g < NV; ++g) dst[g] = make_uint4(w[4 * g], w[4 * g + 1], w[4 * g + 2], w[4 * g + 3]);
                    } else {
                        store_scalar(col0, w, 0);
                    }
                }
            };

            // ---- stream-K pieces (double-buffered configurations only)
            // Workspace slot of a CTA: 128 x BN fp32 in [chunk][vec][row] float4 order (private
            // layout), so the 32 lanes of a warp (32 consecutive rows) touch 512 contiguous bytes.
            const int trow = q * 32 + lane;
            auto ws_slot = [&](int cluster) {
                return reinterpret_cast<float4*>(p.sk_ws) + static_cast<size_t>(cluster * CG + rank) * (kRowsPerCta * BN / 4);
            };
            int c_first = cluster_id;
            if constexpr (C_::kAccStages == 2) {
                if (pc.kind == PIECE_SPLIT) {
                    // Split-K reduce-scatter over distributed shared memory.
                    // The cluster's S CTAs hold the S K-slices of one tile.  Its output is cut into
                    // U = 4 x NCHUNK units (TMEM lane quarter q x 32-column chunk c, u = 4c + q) and
                    // split js owns units [u_lo(js), u_lo(js + 1)).  Every CTA st.async-es its fp32
                    // partial of each unit it does not own into the owner's (now idle) pipeline
                    // ring; the owner adds the S - 1 received partials to its own in ascending
                    // split order (deterministic) and runs the usual bias / activation / store.
                    const int S = p.splits;
                    const int js = cluster_id % S;                     // == %cluster_ctarank
                    constexpr int U = 4 * NCHUNK;
                    constexpr int UB = 32 * W * 4;                     // bytes of one unit (32 rows x 32 fp32)
                    auto owner = [&](int c) { return (4 * c + q) * S / U; };
                    auto u_lo = [&](int o) { return (o * U + S - 1) / S; };
                    const uint32_t recv_base = ptx::smem_u32(smem_a);
                    if (e_idx == 0 && lane == 0) {
                        // incoming bytes of this CTA's units; then tell every peer its ring is free
                        ptx::mbar_arrive_expect_tx(recv_full_bar, static_cast<uint32_t>((u_lo(js + 1) - u_lo(js)) * (S - 1) * UB));
                        for (int jj = 0; jj < S; ++jj)
                            if (jj != js) ptx::mbar_arrive_cluster(peer_ready_bar, static_cast<uint32_t>(jj));
                    }
                    const long long tw0 = clock64();
                    ptx::mbar_wait(peer_ready_bar, 0);
                    if (dbg && e_idx == 0 && lane == 0) dl[DBG_SK_WAIT] += static_cast<unsigned long long>(clock64() - tw0);
#pragma unroll 1
                    for (int j = 0; j < CPH; ++j) {
                        const int c = j * NG + grp;
                        const int o = owner(c);
                        if (o == js) continue;
                        uint32_t v[W];
                        load(c, v);
                        ptx::tmem_ld_wait_regs(v);
                        const int slot = (4 * c + q - u_lo(o)) * (S - 1) + (js < o ? js : js - 1);
                        const uint32_t dst = ptx::mapa_shared(recv_base + slot * UB + lane * 16, static_cast<uint32_t>(o));
                        const uint32_t rbar = ptx::mapa_shared(ptx::smem_u32(recv_full_bar), static_cast<uint32_t>(o));
#pragma unroll
                        for (int g = 0; g < W / 4; ++g)
                            ptx::st_async_v4(dst + g * 512, v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3], rbar);
                    }
                    const long long tr0 = clock64();
                    if (dbg && lane == 0) dl[DBG_EPI_TMEMLD] += static_cast<unsigned long long>(tr0 - tw0);  // sends
                    ptx::mbar_wait(recv_full_bar, 0);
                    if (dbg && e_idx == 0 && lane == 0) dl[DBG_SK_WRITE] += static_cast<unsigned long long>(clock64() - tr0);
                    const long long to0 = clock64();
#pragma unroll 1
                    for (int j = 0; j < CPH; ++j) {
                        const int c = j * NG + grp;
                        if (owner(c) != js) continue;
                        const long long tq0 = dbg ? clock64() : 0;
                        uint32_t v[W];
                        load(c, v);
                        ptx::tmem_ld_wait_regs(v);
                        const long long tq1 = dbg ? clock64() : 0;
                        const uint8_t* rb = smem_a + (4 * c + q - u_lo(js)) * (S - 1) * UB + lane * 16;
#pragma unroll 1
                        for (int s2 = 0; s2 < S - 1; ++s2) {
#pragma unroll
                            for (int g = 0; g < W / 4; ++g) {
                                const float4 pv = *reinterpret_cast<const float4*>(rb + s2 * UB + g * 512);
                                v[4 * g] = __float_as_uint(__uint_as_float(v[4 * g]) + pv.x);
                                v[4 * g + 1] = __float_as_uint(__uint_as_float(v[4 * g + 1]) + pv.y);
                                v[4 * g + 2] = __float_as_uint(__uint_as_float(v[4 * g + 2]) + pv.z);
                                v[4 * g + 3] = __float_as_uint(__uint_as_float(v[4 * g + 3]) + pv.w);
                            }
                        }
                        const long long tq2 = dbg ? clock64() : 0;
                        uint32_t w[NWORD];
                        compute(c, v, w);
                        const long long tq3 = dbg ? clock64() : 0;
                        store(c, w);
                        if (dbg && lane == 0) {
                            dl[DBG_OWN_LD] += static_cast<unsigned long long>(tq1 - tq0);
                            dl[DBG_OWN_ADD] += static_cast<unsigned long long>(tq2 - tq1);
                            dl[DBG_OWN_MATH] += static_cast<unsigned long long>(tq3 - tq2);
                            dl[DBG_OWN_ST] += static_cast<unsigned long long>(clock64() - tq3);
                        }
                    }
                    if (dbg && lane == 0) dl[DBG_EPI_MATH] += static_cast<unsigned long long>(clock64() - to0);   // owner
                    release(0);
                    if (dbg && e_idx == 0 && lane == 0) dl[DBG_EPI_TILE] += static_cast<unsigned long long>(clock64() - t_epi0);
                    continue;
                }
                if (dbg && e_idx == 0 && lane == 0 && pc.kind != PIECE_FULL) dl[DBG_SK_PIECES] += 1;
                if (pc.kind == PIECE_PARTIAL) {
                    const long long tw0 = clock64();
                    // partial accumulator -> this CTA's workspace slot (fp32, row = TMEM lane), then
                    // publish it; bias and ReLU are applied once, by the owner, after the full
                    // reduction (DESIGN.md R-C13)
#pragma unroll 1
                    for (int j = 0; j < CPH; ++j) {
                        const int c = j * NG + grp;
                        uint32_t v[W];
                        load(c, v);
                        ptx::tmem_ld_wait_regs(v);
                        if (j == CPH - 1) release(0);
                        float4* dst = ws_slot(cluster_id) + static_cast<size_t>(c * (W / 4)) * kRowsPerCta + trow;
#pragma unroll
                        for (int g = 0; g < W / 4; ++g)
                            __stcg(dst + g * kRowsPerCta,
                                   make_float4(__uint_as_float(v[4 * g]), __uint_as_float(v[4 * g + 1]),
                                               __uint_as_float(v[4 * g + 2]), __uint_as_float(v[4 * g + 3])));
                    }
                    __threadfence();
                    ptx::named_bar_sync(2, EPI_WARPS * 32);
                    if (e_idx == 0 && lane == 0) ptx::st_release_gpu(p.sk_flags + cluster_id * CG + rank, 1u);
                    if (dbg && e_idx == 0 && lane == 0) dl[DBG_SK_WRITE] += static_cast<unsigned long long>(clock64() - tw0);
                    continue;
                }
                if (pc.kind == PIECE_OWNER) {
                    // wait until every earlier piece of this tile is in its cluster's workspace slot
                    c_first = work.first_contributor(t);
                    const long long tw0 = clock64();
                    if (e_idx == 0 && lane == 0)
                        for (int c2 = c_first; c2 < cluster_id; ++c2)
                            if (work.has_units(c2)) ptx::spin_acquire_gpu(p.sk_flags + c2 * CG + rank, 1u);
                    ptx::named_bar_sync(2, EPI_WARPS * 32);
                    if (dbg && e_idx == 0 && lane == 0) dl[DBG_SK_WAIT] += static_cast<unsigned long long>(clock64() - tw0);
                }
            }
            // owner: add the published partials (ascending cluster order: deterministic)
            auto add_partials = [&](const int c, uint32_t* v) {
                if constexpr (C_::kAccStages == 2) {
                    for (int c2 = c_first; c2 < cluster_id; ++c2) {
                        if (!work.has_units(c2)) continue;
                        const float4* src = ws_slot(c2) + static_cast<size_t>(c * (W / 4)) * kRowsPerCta + trow;
                        float4 pvs[W / 4];
#pragma unroll
                        for (int g = 0; g < W / 4; ++g) pvs[g] = __ldcg(src + g * kRowsPerCta);
#pragma unroll
                        for (int g = 0; g < W / 4; ++g) {
                            const float4 pv = pvs[g];
                            v[4 * g] = __float_as_uint(__uint_as_float(v[4 * g]) + pv.x);
                            v[4 * g + 1] = __float_as_uint(__uint_as_float(v[4 * g + 1]) + pv.y);
                            v[4 * g + 2] = __float_as_uint(__uint_as_float(v[4 * g + 2]) + pv.z);
                            v[4 * g + 3] = __float_as_uint(__uint_as_float(v[4 * g + 3]) + pv.w);
                        }
                    }
                }
            };

            if (GE_DBG && (p.dbg_flags & 1)) {   // timing experiment (debug build only): release without draining
#pragma unroll
                for (int h = 0; h < NH; ++h) release(h);
                continue;
            }
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                if constexpr (BATCH) {
                    static_assert(CPH % 2 == 0, "paired drain");
                    // chunks are drained two at a time (both TMEM loads in flight together), so the
                    // half is released after CPH/2 - 1 chunk pairs of math instead of CPH - 1 chunks
                    uint32_t packed[CPH][NWORD];
#pragma unroll
                    for (int j = 0; j < CPH; j += 2) {
                        uint32_t va[W], vb[W];
                        load(h * CPH_ALL + j * NG + grp, va);
                        load(h * CPH_ALL + (j + 1) * NG + grp, vb);
                        if (nkb > 0) {
                            ptx::tmem_ld_wait_regs(va);
                            ptx::tmem_ld_wait_regs(vb);
                        }
                        if (j + 2 >= CPH) release(h);
                        compute(h * CPH_ALL + j * NG + grp, va, packed[j]);
                        compute(h * CPH_ALL + (j + 1) * NG + grp, vb, packed[j + 1]);
                    }
#pragma unroll
                    for (int j = 0; j < CPH; ++j) store(h * CPH_ALL + j * NG + grp, packed[j]);
                } else if (fast_loop) {
                    if constexpr (GE_EPI_PAIRLD && CPH % 2 == 0) {
                        // two chunks' TMEM loads in flight together (the last tile's drain is
                        // exposed on single-wave shapes)
#pragma unroll 1
                        for (int j = 0; j < CPH; j += 2) {
                            const int c0 = h * CPH_ALL + j * NG + grp, c1 = c0 + NG;
                            uint32_t va[W], vb[W];
                            ptx::tmem_ld_32x32b_x32(tm_row + c0 * W, va);
                            ptx::tmem_ld_32x32b_x32(tm_row + c1 * W, vb);
                            ptx::tmem_ld_wait_regs(va);
                            ptx::tmem_ld_wait_regs(vb);
                            if (j + 2 >= CPH) release(h);
                            uint32_t w[NWORD];
                            compute_fast(c0, va, w);
                            store(c0, w);
                            compute_fast(c1, vb, w);
                            store(c1, w);
                        }
                    } else {
#pragma unroll 1
                        for (int j = 0; j < CPH; ++j) {
                            const int c = h * CPH_ALL + j * NG + grp;
                            uint32_t v[W];
                            ptx::tmem_ld_32x32b_x32(tm_row + c * W, v);
                            ptx::tmem_ld_wait_regs(v);
                            if (j == CPH - 1) release(h);
                            uint32_t w[NWORD];
                            compute_fast(c, v, w);
                            store(c, w);
                        }
                    }
                } else {
#pragma unroll 1
                    for (int j = 0; j < CPH; ++j) {
                        const int c = h * CPH_ALL + j * NG + grp;
                        uint32_t v[W];
                        load(c, v);
                        if (nkb > 0) ptx::tmem_ld_wait_regs(v);
                        if (j == CPH - 1) release(h);
                        if (pc.kind == PIECE_OWNER) add_partials(c, v);
                        uint32_t w[NWORD];
                        if (GE_DBG && (p.dbg_flags & 8)) {   // timing experiment (debug build only): no epilogue math
#pragma unroll
                            for (int e = 0; e < NWORD; ++e) w[e] = v[e];
                        } else {
                            compute(c, v, w);
                        }
                        if (!(GE_DBG && (p.dbg_flags & 16))) store(c, w);   // 16: timing experiment (debug build), no stores
                        else if (p.dbg && w[0] == 0x12345678u && w[NWORD - 1] == 0x9abcdef0u) p.dbg[0] = 1;
                    }
                }
            }
            if constexpr (C_::kAccStages == 2) {
                if (pc.kind == PIECE_OWNER) {
                    // partials consumed: reset the contributors' flags for the next launch
                    ptx::named_bar_sync(2, EPI_WARPS * 32);
                    if (e_idx == 0 && lane == 0)
                        for (int c2 = c_first; c2 < cluster_id; ++c2)
                            if (work.has_units(c2)) ptx::st_relaxed_gpu(p.sk_flags + c2 * CG + rank, 0u);
                }
            }
            if (dbg && e_idx == 0 && lane == 0) dl[DBG_EPI_TILE] += static_cast<unsigned long long>(clock64() - t_epi0);
        }
        // Only the staging reads must finish before the CTA exits: the stores' global writes
        // complete with the grid (they are visible to the next kernel / PDL dependent and to the
        // stream, as for any async-proxy write), so the exposed tail skips their write latency.
        if (p.c_tma && lane == 0) {
            if (GE_END_WAIT_READ) ptx::bulk_wait_read<0>();
            else ptx::bulk_wait<0>();
        }
        GE_TL(TL_EPI_END, e_idx == 0 && lane == 0);
        if (dbg && e_idx == 0 && lane == 0) {
            dl[DBG_EPI_END] = static_cast<unsigned long long>(clock64() - t_start);
            dl[DBG_G_EPI_END] = globaltimer();
        }
    } else if (PRO && warp >= 4 + EPI_WARPS) {
        // ===================== prologue transform of the A stage (in place, in smem) ==========
        // (Sec. VII-C.)  The TMA lands A (and S) in the swizzled stage; these warps
        // rewrite A in place and hand the stage to the MMA.  Measured alternative (round 2, DESIGN.md
        // "Prologue"): loading A through registers (ld.global -> op -> st.shared, the paper's Volta copy
        // path) saves two smem passes but its global loads could not be kept in flight deep enough
        // (2-4x slower at 4096^3), so the TMA stays the loader.
        constexpr int XT = kXformWarps * 32;                     // transform threads
        const int xt = threadIdx.x - (4 + EPI_WARPS) * 32;      // 0 .. XT-1
        // Thread xt rewrites the 16-B chunks o = (i*XT + xt)*16, i < 16 KB / 16 / XT, of each A stage.
        //  K-major stage (row = m, 128-B rows of 64 k, 128-B swizzle): the logical k-chunk of all its
        //   chunks is kc = (xt % 8) ^ ((xt / 8) % 8) (XT is a multiple of 64), so the thread needs
        //   scale[k0+8kc .. +8];
        //  MN-major stage (row = k, 64-m atoms of 8 KB): chunk i lies on k = k0 + ((i*XT + xt)/8) % 64.
        // The 8 scale values of the NEXT k-block are prefetched while the current one is
        // transformed (the scale vector would otherwise cost an L2 round trip per chunk).
        const bool scale_k = p.prologue == PRO_SCALE_K;
        const int kc = (xt & 7) ^ ((xt >> 3) & 7);
        auto fetch = [&](int kb, float* dst) {
            const int k0 = kb * kBK;
            if (A_MN) {
#pragma unroll
                for (int i = 0; i < C_::kAStage / 16 / XT; ++i) {
                    const int k = k0 + (((i * XT + xt) >> 3) & 63);
                    dst[i] = k < p.K ? __ldg(p.scale + k) : 0.0f;
                }
            } else {
                const int k = k0 + kc * 8;
                if (p.scale_vec && k + 8 <= p.K) {
                    const float4 s0 = __ldg(reinterpret_cast<const float4*>(p.scale + k));
                    const float4 s1 = __ldg(reinterpret_cast<const float4*>(p.scale + k + 4));
                    dst[0] = s0.x; dst[1] = s0.y; dst[2] = s0.z; dst[3] = s0.w;
                    dst[4] = s1.x; dst[5] = s1.y; dst[6] = s1.z; dst[7] = s1.w;
                } else {
#pragma unroll
                    for (int e = 0; e < 8; ++e) dst[e] = (k + e < p.K) ? __ldg(p.scale + k + e) : 0.0f;
                }
            }
        };
        float sc_cur[8], sc_nxt[8];
        if (scale_k && nkb > 0 && work.count() > 0) fetch(work.get(0).kb0, sc_nxt);
        int s = 0;
        uint32_t phase = 0;
        for (int wi = 0; wi < work.count(); ++wi) {
            const Piece pc = work.get(wi);
            for (int kb = pc.kb0; kb < pc.kb1; ++kb) {
                if (scale_k) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) sc_cur[e] = sc_nxt[e];
                    int kn = kb + 1;                                  // next k-block this thread transforms
                    if (kn == pc.kb1) kn = (wi + 1 < work.count()) ? work.get(wi + 1).kb0 : 0;
                    fetch(kn, sc_nxt);                                // in flight during this stage
                }
                const long long tx0 = dbg ? clock64() : 0;
                ptx::mbar_wait(&full_bar[s], phase);
                const long long tx1 = dbg ? clock64() : 0;
                uint8_t* sa = smem_a + s * C_::kAStage;
                constexpr int NCH = C_::kAStage / 16 / XT;           // chunks per thread
                uint4 x[NCH];
#pragma unroll
                for (int i = 0; i < NCH; ++i) x[i] = *reinterpret_cast<const uint4*>(sa + (i * XT + xt) * 16);
                if constexpr (PRO == 2) {
                    // HADAMARD: a' = RNE_fp16(s(i,k) * a(i,k)); S sits at the same swizzled offsets as A
                    // (same box, same swizzle), and the fp16 x fp16 product is exact before its one
                    // rounding (mul.rn.f16x2; DESIGN.md R-C18)
                    const uint8_t* ss = smem_s + s * C_::kSStage;
#pragma unroll
                    for (int i = 0; i < NCH; ++i) {
                        const uint4 y = *reinterpret_cast<const uint4*>(ss + (i * XT + xt) * 16);
                        __half2* h2 = reinterpret_cast<__half2*>(&x[i]);
                        const __half2* s2 = reinterpret_cast<const __half2*>(&y);
#pragma unroll
                        for (int e = 0; e < 4; ++e) h2[e] = __hmul2(h2[e], s2[e]);
                    }
                }
#pragma unroll
                for (int i = 0; i < NCH && PRO == 1; ++i) {
                    if (!scale_k) {
                        // RELU: a' = max(a, +0): clear every lane with the sign bit set (exact, -0 -> +0)
                        uint32_t* w = reinterpret_cast<uint32_t*>(&x[i]);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            uint32_t u = w[e];
                            if (u & 0x8000u) u &= 0xFFFF0000u;
                            if (u & 0x80000000u) u &= 0x0000FFFFu;
                            w[e] = u;
                        }
                    } else {
                        // SCALE_K: a' = RNE_fp16(s_k * a) (DESIGN.md R-C12)
                        __half2* h2 = reinterpret_cast<__half2*>(&x[i]);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float2 a = __half22float2(h2[e]);
                            const float s0 = A_MN ? sc_cur[i] : sc_cur[2 * e];
                            const float s1 = A_MN ? sc_cur[i] : sc_cur[2 * e + 1];
                            h2[e] = __floats2half2_rn(s0 * a.x, s1 * a.y);
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < NCH; ++i) *reinterpret_cast<uint4*>(sa + (i * XT + xt) * 16) = x[i];
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if (CG == 2 && !leader) ptx::mbar_arrive_cluster(&xform_bar[s], 0);
                    else ptx::mbar_arrive(&xform_bar[s]);
                }
                if (dbg && lane == 0) {
                    dl[DBG_XF_WAIT] += static_cast<unsigned long long>(tx1 - tx0);
                    dl[DBG_XF_WORK] += static_cast<unsigned long long>(clock64() - tx1);
                }
                if (++s == S) { s = 0; phase ^= 1; }
            }
        }
    }

    // ---- teardown: every role done; the allocating warp frees TMEM
    __syncwarp();
    if (dbg) {
        if (warp == 1 && lane == 0) dl[DBG_TOTAL] = static_cast<unsigned long long>(clock64() - t_start);
        unsigned long long* dg = p.dbg + blockIdx.x * DBG_SLOTS;
#pragma unroll
        for (int i = 0; i < DBG_SLOTS; ++i)
            if (dl[i]) atomicAdd(dg + i, dl[i]);
    }
    ptx::tc_fence_before();
    if (CG == 2 || split_cluster) {
        if (GE_TEARDOWN_RELAXED) ptx::cluster_sync_relaxed();
        else ptx::cluster_sync();
    } else {
        __syncthreads();
    }
    GE_TL(TL_TEARDOWN, threadIdx.x == 0);
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<CG>(tmem_base, C_::kTmemCols);
        GE_TL(TL_EXIT, lane == 0);
        if (GE_DBG && p.dbg != nullptr && lane == 0) atomicAdd(p.dbg + blockIdx.x * DBG_SLOTS + DBG_G_EXIT, globaltimer());
    }
#endif
}

#undef GE_TL

}  // namespace ge
