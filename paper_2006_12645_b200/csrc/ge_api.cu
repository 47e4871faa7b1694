// ge_api.cu -- host runtime behind include/gemm_epilogue.h: argument validation, the tile
// configuration heuristic, TMA tensor-map encoding, persistent grid sizing and the launch.
//
// Launch inference in the paper comes from schedule constraints (one
// 128x128 block per output tile, grid (N/128, M/128)).  Here the grid is
// persistent: min(#tiles, #SMs) CTAs (CTA pairs for cta_group 2) walk the tile sequence.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/gemm_epilogue.h"
#include "ge_launch.cuh"

namespace {

thread_local std::string g_detail;
std::atomic<uint64_t> g_launches{0};

ge_status fail(ge_status s, const std::string& why) {
    g_detail = why;
    return s;
}

constexpr int64_t kMaxDim = (1ll << 31) - 1;

struct Dev {
    bool probed = false;
    bool ok = false;
    int sms = 0;
};
std::mutex g_dev_mu;
Dev g_devs[64];

ge_status device_info(int* sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        cudaGetLastError();
        return fail(GE_ERR_UNSUPPORTED_DEVICE, "no CUDA device");
    }
    std::lock_guard<std::mutex> lk(g_dev_mu);
    Dev& d = g_devs[dev];
    if (!d.probed) {
        int major = 0, minor = 0, n = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cudaGetLastError();
        d.ok = (major == 10 && minor == 0);
        d.sms = n;
        d.probed = true;
    }
    if (!d.ok) return fail(GE_ERR_UNSUPPORTED_DEVICE, "device is not sm_100 (B200); this library targets sm_100a");
    *sms = d.sms;
    return GE_OK;
}

// ------------------------------------------------------------------ validation
struct Args {
    int64_t batch, M, N, K;
    int32_t la, lb;
    const void* A;
    int64_t lda, sA;
    const void* B;
    int64_t ldb, sB;
    const void* bias;
    int64_t sBias;
    void* C;
    int64_t ldc, sC;
    int32_t op;
    ge_options o;
    // second matmul of a sum of matmuls (gemm2_epilogue, Listing 4): P (layout of A), Q (of B)
    int64_t K2 = 0;
    const void* P = nullptr;
    int64_t ldp = 0;
    const void* Q = nullptr;
    int64_t ldq = 0;
};

int64_t extent_bytes(int64_t batch, int64_t outer, int64_t inner, int64_t ld, int64_t stride, int es) {
    if (batch == 0 || outer == 0 || inner == 0) return 0;
    return ((batch - 1) * stride + (outer - 1) * ld + inner) * es;
}

bool overlap(const void* a, int64_t na, const void* b, int64_t nb) {
    if (!a || !b || na <= 0 || nb <= 0) return false;
    const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
    return x < y + static_cast<uintptr_t>(nb) && y < x + static_cast<uintptr_t>(na);
}

// op bit flags (include/gemm_epilogue.h): bit 0 bias, bit 1 ReLU, bit 2 Sigmoid, bit 3 Tanh,
// bit 4 subtract the bias, bit 5 paper-literal fp16 rounding of the intermediate; at most one
// activation, subtraction only with a bias.
bool op_valid(int32_t op) {
    if (op < 0 || op > 63) return false;
    const int acts = ((op >> 1) & 1) + ((op >> 2) & 1) + ((op >> 3) & 1);
    return acts <= 1 && (!(op & GE_EPI_SUB) || (op & GE_EPI_BIAS));
}
bool has_bias(int32_t op) { return (op & GE_EPI_BIAS) != 0; }
int act_of(int32_t op) {
    return (op & GE_EPI_RELU) ? ge::ACT_RELU : (op & GE_EPI_SIGMOID) ? ge::ACT_SIGMOID
                                                  : (op & GE_EPI_TANH) ? ge::ACT_TANH : ge::ACT_NONE;
}

// Option and enum checks shared by validate() and ge_plan() (no pointers involved).
ge_status validate_options(const Args& a) {
    const ge_options& o = a.o;
    if ((a.la != GE_ROW_MAJOR && a.la != GE_COL_MAJOR) || (a.lb != GE_ROW_MAJOR && a.lb != GE_COL_MAJOR))
        return fail(GE_ERR_INVALID_VALUE, "layout must be GE_ROW_MAJOR or GE_COL_MAJOR");
    if (o.bias_mode < GE_BIAS_ROW || o.bias_mode > GE_BIAS_FULL) return fail(GE_ERR_INVALID_VALUE, "bad bias_mode");
    if (o.prologue < GE_PRO_NONE || o.prologue > GE_PRO_HADAMARD) return fail(GE_ERR_INVALID_VALUE, "bad prologue");
    if (o.ld_prologue_tile < 0 || o.stride_prologue_tile < 0)
        return fail(GE_ERR_INVALID_VALUE, "negative ld_prologue_tile / stride_prologue_tile");
    if (o.out_dtype != GE_OUT_F16 && o.out_dtype != GE_OUT_F32) return fail(GE_ERR_INVALID_VALUE, "bad out_dtype");
    if (o.tile_n != 0 && o.tile_n != 64 && o.tile_n != 128 && o.tile_n != 192 && o.tile_n != 256 && o.tile_n != 512)
        return fail(GE_ERR_INVALID_VALUE, "tile_n must be 0, 64, 128, 192, 256 or 512");
    if (o.cta_group < 0 || o.cta_group > 2) return fail(GE_ERR_INVALID_VALUE, "cta_group must be 0, 1 or 2");
    if (o.cta_group == 2 && o.tile_n == 64) return fail(GE_ERR_INVALID_VALUE, "cta_group 2 needs tile_n >= 128");
    if (o.cta_group == 1 && o.tile_n == 512) return fail(GE_ERR_INVALID_VALUE, "tile_n 512 needs cta_group 2");
    if (o.cta_group == 2 && o.tile_n == 192 && a.lb == GE_ROW_MAJOR)
        return fail(GE_ERR_INVALID_VALUE, "tile_n 192 with cta_group 2 needs a column-major (K-major) B");
    if (o.stream_k < 0 || o.stream_k > 2) return fail(GE_ERR_INVALID_VALUE, "stream_k must be 0, 1 or 2");
    if (o.multicast < 0 || o.multicast > 2) return fail(GE_ERR_INVALID_VALUE, "multicast must be 0, 1 or 2");
    if (o.multicast == 2 && (o.prologue != GE_PRO_NONE || o.stream_k == 2 || (o.cta_group && o.cta_group != 2) ||
                             (o.tile_n && o.tile_n != 256 && o.tile_n != 512)))
        return fail(GE_ERR_INVALID_VALUE, "multicast = 2 needs no prologue, stream_k != 2, cta_group 0/2, tile_n 0/256/512");
    if (o.swap_ab < 0 || o.swap_ab > 2) return fail(GE_ERR_INVALID_VALUE, "swap_ab must be 0, 1 or 2");
    if (o.tile_m != 0 && o.tile_m != 128 && o.tile_m != 256) return fail(GE_ERR_INVALID_VALUE, "tile_m must be 0, 128 or 256");
    if (o.tile_m == 256 && o.cta_group == 1) return fail(GE_ERR_INVALID_VALUE, "tile_m 256 needs cta_group 2");
    if (o.tile_m == 128 && o.cta_group == 2 &&
        (o.tile_n == 64 || o.tile_n == 192 || o.tile_n == 512 || o.multicast == 2 || o.stream_k == 2))
        return fail(GE_ERR_INVALID_VALUE,
                    "half-row pair tiles (tile_m 128, cta_group 2) take tile_n 0/128/256, no multicast, no forced stream-K");
    if (o.workspace_bytes < 0 || (o.workspace && (reinterpret_cast<uintptr_t>(o.workspace) & 15)))
        return fail(GE_ERR_INVALID_VALUE, "workspace must be 16-byte aligned with a non-negative size");
    return GE_OK;
}

// Normalises ld/stride defaults in place and checks everything that can be checked on the host.
ge_status validate(Args& a) {
    char buf[256];
    if (a.batch < 0 || a.M < 0 || a.N < 0 || a.K < 0)
        return fail(GE_ERR_INVALID_VALUE, "negative size");
    if (a.M > kMaxDim || a.N > kMaxDim || a.K > kMaxDim || a.batch > kMaxDim)
        return fail(GE_ERR_INVALID_VALUE, "size exceeds 2^31-1");
    if ((a.la != GE_ROW_MAJOR && a.la != GE_COL_MAJOR) || (a.lb != GE_ROW_MAJOR && a.lb != GE_COL_MAJOR))
        return fail(GE_ERR_INVALID_VALUE, "layout must be GE_ROW_MAJOR or GE_COL_MAJOR");
    if (!op_valid(a.op)) return fail(GE_ERR_INVALID_VALUE, "bad epilogue op (see ge_epilogue_op flags)");
    {
        const ge_status so = validate_options(a);
        if (so != GE_OK) return so;
    }
    // packed defaults
    const bool arow = a.la == GE_ROW_MAJOR, brow = a.lb == GE_ROW_MAJOR;
    const int64_t minlda = arow ? a.K : a.M, minldb = brow ? a.N : a.K;
    if (a.lda == 0) a.lda = std::max<int64_t>(minlda, 1);
    if (a.ldb == 0) a.ldb = std::max<int64_t>(minldb, 1);
    if (a.ldc == 0) a.ldc = std::max<int64_t>(a.N, 1);
    if (a.lda < minlda || a.ldb < minldb || a.ldc < a.N || a.lda < 0 || a.ldb < 0 || a.ldc < 0) {
        snprintf(buf, sizeof buf, "leading dimension too small (lda=%lld ldb=%lld ldc=%lld)", (long long)a.lda,
                 (long long)a.ldb, (long long)a.ldc);
        return fail(GE_ERR_INVALID_VALUE, buf);
    }
    const int64_t outerA = arow ? a.M : a.K, outerB = brow ? a.K : a.N;
    if (a.sA == 0) a.sA = outerA * a.lda;
    if (a.sB == 0) a.sB = outerB * a.ldb;
    if (a.sC == 0) a.sC = a.M * a.ldc;
    if (a.o.bias_mode == GE_BIAS_FULL && a.o.ldbias == 0) a.o.ldbias = a.N;
    if (a.sA < 0 || a.sB < 0 || a.sC < 0 || a.sBias < 0 || a.o.ldbias < 0)
        return fail(GE_ERR_INVALID_VALUE, "negative stride");
    if (a.o.bias_mode == GE_BIAS_FULL && a.o.ldbias < a.N) return fail(GE_ERR_INVALID_VALUE, "ldbias < N");
    if (a.batch > 1 && a.sC < a.M * a.ldc)
        return fail(GE_ERR_INVALID_VALUE, "strideC smaller than one output item (items would overlap)");
    if (a.batch == 0 || a.M == 0 || a.N == 0) return GE_OK;   // no-op
    if (!a.C) return fail(GE_ERR_INVALID_VALUE, "C is NULL");
    if (a.K > 0 && (!a.A || !a.B)) return fail(GE_ERR_INVALID_VALUE, "A or B is NULL");
    if (has_bias(a.op) && !a.bias) return fail(GE_ERR_INVALID_VALUE, "bias is NULL but the op adds a bias");
    if (a.o.prologue == GE_PRO_SCALE_K && a.K > 0 && !a.o.prologue_scale)
        return fail(GE_ERR_INVALID_VALUE, "prologue_scale is NULL for GE_PRO_SCALE_K");
    if (a.o.prologue == GE_PRO_HADAMARD && a.K > 0) {
        // S: M x K in A's layout (DESIGN.md R-C18), read with 16-byte vector loads like A
        if (!a.o.prologue_tile) return fail(GE_ERR_INVALID_VALUE, "prologue_tile is NULL for GE_PRO_HADAMARD");
        const int64_t minlds = arow ? a.K : a.M;
        if (a.o.ld_prologue_tile == 0) a.o.ld_prologue_tile = std::max<int64_t>(minlds, 1);
        if (a.o.ld_prologue_tile < minlds) return fail(GE_ERR_INVALID_VALUE, "ld_prologue_tile too small");
        if (a.batch > 1 && a.o.stride_prologue_tile != 0 &&
            a.o.stride_prologue_tile < (arow ? a.M : a.K) * a.o.ld_prologue_tile)
            return fail(GE_ERR_INVALID_VALUE, "stride_prologue_tile smaller than one item");
        if ((reinterpret_cast<uintptr_t>(a.o.prologue_tile) & 15) || (a.o.ld_prologue_tile * 2) % 16 ||
            (a.o.stride_prologue_tile * 2) % 16)
            return fail(GE_ERR_MISALIGNED, "prologue_tile must be 16-byte aligned with ld/stride multiples of 8 elements");
    }
    if (a.K2 < 0 || a.K2 > kMaxDim) return fail(GE_ERR_INVALID_VALUE, "K2 out of range");
    if (a.K2 > 0) {
        if (a.o.prologue != GE_PRO_NONE)
            return fail(GE_ERR_INVALID_VALUE, "the prologue is not supported with a sum of matmuls");
        const int64_t minldp = arow ? a.K2 : a.M, minldq = brow ? a.N : a.K2;
        if (a.ldp == 0) a.ldp = std::max<int64_t>(minldp, 1);
        if (a.ldq == 0) a.ldq = std::max<int64_t>(minldq, 1);
        if (a.ldp < minldp || a.ldq < minldq) return fail(GE_ERR_INVALID_VALUE, "ldp or ldq too small");
        if (!a.P || !a.Q) return fail(GE_ERR_INVALID_VALUE, "P or Q is NULL");
        if ((reinterpret_cast<uintptr_t>(a.P) & 15) || (reinterpret_cast<uintptr_t>(a.Q) & 15))
            return fail(GE_ERR_MISALIGNED, "P and Q must be 16-byte aligned (TMA)");
        if ((a.ldp * 2) % 16 || (a.ldq * 2) % 16)
            return fail(GE_ERR_MISALIGNED, "ldp and ldq must be multiples of 8 elements (16 bytes, TMA)");
        const int es2 = a.o.out_dtype == GE_OUT_F32 ? 4 : 2;
        const int64_t nC2 = extent_bytes(a.batch, a.M, a.N, a.ldc, a.sC, es2);
        if (overlap(a.C, nC2, a.P, extent_bytes(1, arow ? a.M : a.K2, arow ? a.K2 : a.M, a.ldp, 0, 2)) ||
            overlap(a.C, nC2, a.Q, extent_bytes(1, brow ? a.K2 : a.N, brow ? a.N : a.K2, a.ldq, 0, 2)))
            return fail(GE_ERR_ALIASING, "C overlaps P or Q");
    }
    if (a.K > 0) {
        if ((reinterpret_cast<uintptr_t>(a.A) & 15) || (reinterpret_cast<uintptr_t>(a.B) & 15))
            return fail(GE_ERR_MISALIGNED, "A and B must be 16-byte aligned (TMA)");
        if ((a.lda * 2) % 16 || (a.ldb * 2) % 16)
            return fail(GE_ERR_MISALIGNED, "lda and ldb must be multiples of 8 elements (16 bytes, TMA)");
        if (a.batch > 1 && ((a.sA * 2) % 16 || (a.sB * 2) % 16))
            return fail(GE_ERR_MISALIGNED, "strideA and strideB must be multiples of 8 elements (TMA)");
        if (a.batch > 1 && (a.sA == 0 || a.sB == 0))
            return fail(GE_ERR_INVALID_VALUE, "strideA/strideB must be positive for batch > 1");
    }
    // aliasing: C must not overlap any input
    const int es = a.o.out_dtype == GE_OUT_F32 ? 4 : 2;
    const int64_t nC = extent_bytes(a.batch, a.M, a.N, a.ldc, a.sC, es);
    const int64_t nA = extent_bytes(a.batch, outerA, arow ? a.K : a.M, a.lda, a.sA, 2);
    const int64_t nB = extent_bytes(a.batch, outerB, brow ? a.N : a.K, a.ldb, a.sB, 2);
    int64_t nBias = 0;
    if (has_bias(a.op)) {
        if (a.o.bias_mode == GE_BIAS_ROW) nBias = ((a.batch - 1) * a.sBias + a.N) * 2;
        else if (a.o.bias_mode == GE_BIAS_COL) nBias = ((a.batch - 1) * a.sBias + a.M) * 2;
        else nBias = extent_bytes(a.batch, a.M, a.N, a.o.ldbias, a.sBias, 2);
    }
    const int64_t nS = (a.o.prologue == GE_PRO_SCALE_K) ? a.K * 4 : 0;
    const int64_t nT = (a.o.prologue == GE_PRO_HADAMARD && a.K)
                           ? extent_bytes(a.o.stride_prologue_tile ? a.batch : 1, outerA, arow ? a.K : a.M,
                                          a.o.ld_prologue_tile, a.o.stride_prologue_tile, 2)
                           : 0;
    if (overlap(a.C, nC, a.A, a.K ? nA : 0) || overlap(a.C, nC, a.B, a.K ? nB : 0) ||
        overlap(a.C, nC, a.bias, nBias) || overlap(a.C, nC, a.o.prologue_scale, nS) ||
        overlap(a.C, nC, a.o.prologue_tile, nT))
        return fail(GE_ERR_ALIASING, "C overlaps an input buffer");
    return GE_OK;
}

// ------------------------------------------------------------------ plan
struct Plan {
    int bn, cg, stages;
    bool mc = false;       // multicast cluster of two CTA pairs (tile 512 x bn, B shared by TMA multicast)
    int64_t tiles;
    int64_t sk_tiles;      // tiles of the last, partial wave split stream-K across all clusters (0 = none)
    int64_t clusters;      // persistent clusters launched
    int splits = 0;        // split-K: clusters per tile (0 = off; then clusters = tiles * splits)
    bool hr = false;       // half-row CTA pair: tile 128 x bn, 64 rows per CTA (cta_group::2, M = 128)
};

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Relative tensor-pipe efficiency of each kernel configuration on large shapes, measured on
// B200 (profiles/: 8192^3, all layouts).  N = 128/64 tiles are shared-memory bandwidth bound
// (operand bytes per MMA flop double), the CTA pair halves per-SM B traffic, and the 256 x 512
// pair tile moves the least operand data per flop (L2 and HBM) at the cost of a single,
// non-double-buffered accumulator (its drain is partly exposed: kExposedK below).
// Multicast clusters of two pairs read a third less operand data from L2 per flop (B is shared).
// Measured on B200 (profiles/r01_tune_sweep.json, rotating operands): 256 x 256 pair tiles in
// multicast clusters gain 3-4% on long-K shapes whose wave count the 33 co-resident 4-CTA clusters
// (132 SMs) do not raise, and lose ~2% at K = 2048 (fixed per-tile cost kMcFixed); the 512-wide
// multicast tile never measured best, so the heuristic leaves it to explicit requests.
double config_eff_mc(int bn) {
    static const double env = [] {
        const char* e = getenv("GE_MC_EFF");                // calibration override (tuning only)
        return e ? atof(e) : 0.0;
    }();
    if (env > 0) return env;
    return bn == 512 ? 1.166 : 1.144;       // 1.06 / 1.04 x the pair refit's 1.10
}
constexpr double kMcFixed = 1050.0;     // cycles per multicast tile (cluster-of-4 pipeline fill/drain)
constexpr double kDrain512 = 13600.0;   // cycles exposed per 256 x 512 pair tile (single accumulator)

// Refit (scripts/tune_sweep.py on 50 paper-sweep shapes in rc plus the default shape list in rr,
// profiles/r01_tune_rc50.json, r01_tune_rr_default.json) after the straight-line epilogue: the
// pick's geomean regret against the measured best configuration went 0.978 -> 0.993.
double config_eff(int bn, int cg) {
    if (cg == 2) return bn == 512 ? 1.32 : bn == 256 ? 1.10 : bn == 192 ? 0.87 : 0.59;
    return bn == 256 ? 0.92 : bn == 192 ? 0.82 : bn == 128 ? 0.60 : 0.29;
}
// Half-row pair tiles (128 x BN, 64 rows per CTA), relative to the same per-SM reference; GE_HR_EFF
// overrides (calibration only).
double config_eff_hr(int bn) {
    static const double env = [] {
        const char* e = getenv("GE_HR_EFF");
        return e ? atof(e) : 0.0;
    }();
    if (env > 0) return env;
    return bn == 256 ? 0.20 : 0.20;     // provisional (not picked by default until calibrated on B200)
}
// Cycles per tile column exposed once per launch by the last tile's drain (TMEM -> registers ->
// smem -> TMA store runs after the final MMA; wider tiles drain longer), same refit.
constexpr double kDrainPerCol = 4.0;

// Cost model: per-SM time ~ waves x per-SM tile area x
// (K + exposed epilogue) / eff, waves = ceil(#tiles / #concurrent tiles).  Small problems pick
// narrow tiles to fill the 148 SMs; large ones the CTA-pair tiles.
// Co-resident split-K clusters per (BN index, S) on each device, queried once (0 = unknown: the
// planner then uses its GPC estimate).
struct SplitCap {
    int cap[4][9];
    int mc[2];          // co-resident multicast clusters (two CTA pairs) for BN = 512, 256
};
std::mutex g_cap_mu;
SplitCap g_cap[64];
bool g_cap_done[64];
const SplitCap* split_capacity() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    std::lock_guard<std::mutex> lk(g_cap_mu);
    SplitCap& c = g_cap[dev & 63];
    if (!g_cap_done[dev & 63]) {
        const int bns[4] = {64, 128, 192, 256};
        for (int i = 0; i < 4; ++i)
            for (int S = 0; S <= 8; ++S) c.cap[i][S] = S >= 2 ? ge::clusters_cg1(bns[i], S) : 0;
        c.mc[0] = ge::clusters_mc(512);
        c.mc[1] = ge::clusters_mc(256);
        g_cap_done[dev & 63] = true;
        if (getenv("GE_PRINT_SPLIT_CAPACITY"))      // dev: calibration of the planner's fallback estimate
            for (int i = 0; i < 4; ++i)
                fprintf(stderr, "split capacity bn=%d: S=2..8: %d %d %d %d %d %d %d\n", bns[i], c.cap[i][2], c.cap[i][3],
                        c.cap[i][4], c.cap[i][5], c.cap[i][6], c.cap[i][7], c.cap[i][8]);
    }
    return &c;
}

// sk_allowed: a stream-K workspace is available (the caller passed one); without it the planner
// considers only data-parallel and split-K tiles (the library never allocates on the device entry points).
Plan make_plan(const Args& a, int sms, const SplitCap* cap, bool sk_allowed) {
    // Cost model in SM cycles, calibrated on B200:
    //   one 64-deep k-block of a 128 x BN per-SM tile: 128*BN*64*2 / (8192 flop/clk * eff);
    //   the single-buffered 256 x 512 tile exposes part of its accumulator drain per tile;
    //   a stream-K launch adds its partial traffic (write + read-back of a 128 x BN fp32 slot per
    //   CTA at ~16 B/clk, profiles/r01_stream_k.txt) plus a fixed handshake.
    static const double sk_fixed = [] {
        const char* e = getenv("GE_SK_FIXED_CYCLES");       // calibration override (tuning only)
        return e ? atof(e) : 12000.0;
    }();
    Plan best{};
    double best_cost = 0;
    const int cands[8][2] = {{512, 2}, {256, 2}, {192, 2}, {256, 1}, {192, 1}, {128, 2}, {128, 1}, {64, 1}};
    const int64_t nkb = std::max<int64_t>(1, cdiv(a.K, 64) + cdiv(a.K2, 64));
    for (const auto& c : cands) {
        const int bn = c[0], cg = c[1];
        if (a.o.tile_n && a.o.tile_n != bn) continue;
        if (a.o.cta_group && a.o.cta_group != cg) continue;
        if (a.o.tile_m && a.o.tile_m != 128 * cg) continue;             // (tile_m 128 with pairs: half-row, below)
        if (bn == 192 && cg == 2 && a.lb == GE_ROW_MAJOR) continue;     // pair tile needs a K-major B
        // Skinny M (<= 64 rows): most of every A stage is TMA zero-fill, the shape is HBM bound on B
        // and 128 x 128 tiles measure best (profiles/r01_tune_sweep.json); narrower tiles only add
        // A-stage traffic per useful byte.
        if (a.M <= 64 && !a.o.tile_n && !a.o.cta_group && !(bn == 128 && cg == 1)) continue;
        const int64_t tiles = a.batch * cdiv(a.M, 128 * cg) * cdiv(a.N, bn);
        const int64_t conc = std::max(1, sms / cg);
        double eff = config_eff(bn, cg);
        // The prologue transform rewrites each 16 KB A stage in smem: configurations with less MMA
        // time per stage than 256 x 512 pair tiles become shared-memory bound.
        if (a.o.prologue != GE_PRO_NONE && bn * cg < 1024) eff *= 0.55;
        const double t_kb = 128.0 * bn * 64 * 2 / (8192.0 * eff);
        // exposed per tile by the single 512-column accumulator (drain + refill), fitted with eff = 1.20
        // to the 256 x 256 / 256 x 512 ratios measured at 4096^3 and 8192^3 (profiles/r01_tune_sweep.json)
        const double drain = bn == 512 ? kDrain512 : 0.0;
        const double waves = static_cast<double>(cdiv(std::max<int64_t>(tiles, 1), conc));
        double cost = waves * (nkb * t_kb + drain) + kDrainPerCol * bn;
        int64_t sk = 0;
        // stream-K for the last partial wave (double-buffered accumulators only)
        const int64_t rem = tiles % conc;
        const bool sk_ok = sk_allowed && bn <= 256 && rem != 0 && nkb >= 2 && a.o.stream_k != 1;
        if (sk_ok) {
            const double share = static_cast<double>(tiles / conc) * nkb + static_cast<double>(rem) * nkb / conc;
            // measured: the owner reads one partial per contributor and every cluster's share ends at
            // about the same time, so partial write + wait + read-back adds 10-25K cycles whatever the
            // share (profiles/r01_stream_k.txt, r01_paper_sweep_stream_k.txt)
            const int64_t contributors = std::max<int64_t>(1, conc / std::max<int64_t>(rem, 1));
            const double partial = (1.0 + contributors) * 128.0 * bn * 4 / 16.0;
            const double sk_cost = share * t_kb + partial + sk_fixed + kDrainPerCol * bn;
            if (a.o.stream_k == 2 || sk_cost < cost) {
                cost = sk_cost;
                sk = rem;
            }
        }
        int splits = 0;
        // Split-K for few, long tiles, single-CTA tiles only: a cluster of S
        // CTAs per tile, one K-slice each, partials reduce-scattered over distributed shared
        // memory ((S-1)/S of a 128 x BN fp32 tile sent per CTA at ~9.5 B/clk, plus the handshake).
        // Co-resident clusters of S come from cudaOccupancyMaxActiveClusters (GPC-bound).
        if (cg == 1 && bn <= 256 && a.o.stream_k == 0 && nkb >= 8) {
            const int64_t smax = std::min<int64_t>(8, nkb / 4);
            for (int64_t S = 2; S <= smax; ++S) {
                const int64_t units = 4 * bn / 32;
                const int64_t recv = cdiv(units, S) * (S - 1) * 32 * 32 * 4;
                if (recv > static_cast<int64_t>(ge::stages_for(bn, 1, a.o.prologue == GE_PRO_HADAMARD)) * (128 + bn) * 64 * 2)
                    continue;
                const int bi = bn == 64 ? 0 : bn == 128 ? 1 : bn == 192 ? 2 : 3;
                // fallback (no device): cudaOccupancyMaxActiveClusters measured on B200, S = 2..8
                static const int kCap148[9] = {0, 0, 74, 45, 33, 26, 22, 15, 15};
                int64_t conc_s = (cap && cap->cap[bi][S] > 0) ? cap->cap[bi][S]
                                                              : static_cast<int64_t>(kCap148[S] * (sms / 148.0));
                conc_s = std::max<int64_t>(1, conc_s);
                // every CTA sends and receives (S-1)/S of its fp32 partial at once: ~9.5 B/clk each way
                // measured (DSMEM is ~17 B/clk bidirectional; debug counters on 640x1024x3840,
                // 2048x128x3456, 128x2176x3200: 8.6-10 B/clk effective)
                const double red = (S - 1.0) / S * 128.0 * bn * 4 / 9.5 + 1500.0;
                const double c_split = static_cast<double>(cdiv(tiles, conc_s)) *
                                       (static_cast<double>(cdiv(nkb, S)) * t_kb + red) + kDrainPerCol * bn;
                if (c_split < cost * (1 - 1e-9)) {
                    cost = c_split;
                    splits = static_cast<int>(S);
                    sk = 0;
                }
            }
        }
        if (a.o.multicast == 2) cost = 1e300;                      // forced multicast: pairs only below
        if (best.bn == 0 || cost < best_cost * (1 - 1e-9)) {
            best = Plan{bn, cg, ge::stages_for(bn, cg, a.o.prologue == GE_PRO_HADAMARD), false, tiles, sk,
                        sk ? conc : std::min<int64_t>(tiles, conc)};
            if (splits) {
                best.splits = splits;
                best.clusters = tiles * splits;
            }
            best_cost = cost;
        }
    }
    // Half-row CTA pairs: 128 x BN tiles with 64 rows per CTA
    // (cta_group::2, M = 128).  Per CTA and k-block the MMA reads a 64-row A slice and its half of B,
    // so narrow tiles keep the tensor pipe fed where 128-row single-CTA tiles re-read A from smem
    // for every N = 64..128 instruction.  Data-parallel tiles only.
    const bool hr_ok = a.o.multicast != 2 && a.o.stream_k != 2 && (!a.o.cta_group || a.o.cta_group == 2) &&
                       (!a.o.tile_m || a.o.tile_m == 128);
    if (hr_ok) {
        for (const int bn : {256, 128}) {
            if (a.o.tile_n && a.o.tile_n != bn) continue;
            const int64_t tiles = a.batch * cdiv(a.M, 128) * cdiv(a.N, bn);
            const int64_t conc = std::max(1, sms / 2);
            double eff = config_eff_hr(bn);
            if (a.o.prologue != GE_PRO_NONE) eff *= 0.55;
            const double t_kb = 64.0 * bn * 64 * 2 / (8192.0 * eff);
            const double waves = static_cast<double>(cdiv(std::max<int64_t>(tiles, 1), conc));
            const double cost = waves * nkb * t_kb + kDrainPerCol * bn / 2;
            if (best.bn == 0 || cost < best_cost * (1 - 1e-9)) {
                best = Plan{bn, 2, ge::stages_for(bn, 2, a.o.prologue == GE_PRO_HADAMARD, true), false, tiles, 0,
                            std::min<int64_t>(tiles, conc)};
                best.hr = true;
                best_cost = cost;
            }
        }
    }
    // Multicast clusters of two CTA pairs: data-parallel tiles of
    // 512 x BN, co-resident clusters from cudaOccupancyMaxActiveClusters (GPC-bound: 4-CTA clusters
    // leave some SMs idle, which the cost model charges through `conc`).
    const bool mc_ok = a.o.multicast != 1 && a.o.prologue == GE_PRO_NONE && a.o.stream_k != 2 &&
                       (!a.o.cta_group || a.o.cta_group == 2) && (a.M > 256 || a.o.multicast == 2) &&
                       a.o.tile_m != 128;
    if (mc_ok) {
        for (const int bn : {512, 256}) {
            if (a.o.tile_n && a.o.tile_n != bn) continue;
            if (bn == 512 && a.o.multicast != 2) continue;        // never measured best (see config_eff_mc)
            const int64_t tiles = a.batch * cdiv(a.M, 512) * cdiv(a.N, bn);
            int64_t conc = (cap && cap->mc[bn == 512 ? 0 : 1] > 0) ? cap->mc[bn == 512 ? 0 : 1]
                                                                    : static_cast<int64_t>(33 * (sms / 148.0));
            conc = std::max<int64_t>(1, conc);
            const double t_kb = 128.0 * bn * 64 * 2 / (8192.0 * config_eff_mc(bn));
            const double drain = bn == 512 ? kDrain512 : 0.0;
            const double cost = static_cast<double>(cdiv(tiles, conc)) * (nkb * t_kb + drain + kMcFixed) + kDrainPerCol * bn;
            if (a.o.multicast == 2 || cost < best_cost * (1 - 1e-9)) {
                if (a.o.multicast == 2 && best.mc && cost >= best_cost) continue;
                best = Plan{bn, 2, ge::stages_for(bn, 2), true, tiles, 0, std::min<int64_t>(tiles, conc)};
                best_cost = cost;
            }
        }
    }
    best.clusters = std::max<int64_t>(best.clusters, 1);
    return best;
}

// Stream-K workspace: one fp32 128 x BN slot per CTA plus one flag per CTA (flags must start at 0;
// every launch leaves them at 0).
size_t sk_workspace_bytes(const Plan& pl) {
    if (!pl.sk_tiles) return 0;
    const size_t ctas = static_cast<size_t>(pl.clusters * pl.cg);
    return pl.splits ? 0 : ctas * 128 * pl.bn * 4 + ctas * 4;       // split-K reduces in DSMEM
}

// Raster group: tiles are walked in groups of `group_m` tile-rows so the tiles in flight share
// A panels (along n) and B panels (along m) in L2.  GE_GROUP_M overrides (tuning only).
int group_m_for(const Plan& pl, const Args& a, int sms) {
    static int env = [] {
        const char* e = getenv("GE_GROUP_M");
        return e ? atoi(e) : 0;
    }();
    (void)pl; (void)a; (void)sms;
    if (env > 0) return env;
    return 16;
}

// Diagnostics timeline (debug build, ge_debug_set_timeline): a caller-owned device buffer that
// launches append %globaltimer stamps of CTA 0 to (no per-launch reset, so graph-replayed
// back-to-back launches keep their programmatic-dependent-launch overlap).
unsigned long long* g_timeline = nullptr;
// Diagnostics (env GE_DEBUG_STATS=1, debug build): a zeroed per-CTA counter buffer per device.
unsigned long long* g_dbg[64] = {};
int g_dbg_ctas[64] = {};
int g_dbg_last = -1;                    // device of the last launch (read by ge_debug_read)
#if GE_DBG
unsigned long long* debug_buffer(int sms) {
    static const bool on = getenv("GE_DEBUG_STATS") != nullptr;
    if (!on) return nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    dev &= 63;
    if (!g_dbg[dev]) {
        if (cudaMalloc(&g_dbg[dev], sizeof(unsigned long long) * ge::DBG_SLOTS * sms) != cudaSuccess) {
            cudaGetLastError();
            g_dbg[dev] = nullptr;
            return nullptr;
        }
        g_dbg_ctas[dev] = sms;
    }
    cudaMemset(g_dbg[dev], 0, sizeof(unsigned long long) * ge::DBG_SLOTS * g_dbg_ctas[dev]);
    g_dbg_last = dev;
    return g_dbg[dev];
}
#endif

// ------------------------------------------------------------------ tensor maps
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
        cudaGetLastError();
    });
    return fn;
}

// Tensor-map cache: an encoded CUtensorMap depends only on the encode
// arguments (address, dims, strides, box, swizzle, type), so maps are memoised in a small
// direct-mapped table keyed by exactly those; repeated calls on the same buffers skip
// cuTensorMapEncodeTiled.  Entries own nothing: a freed and re-allocated buffer at the same address
// with the same geometry encodes to the same bytes.  Guarded by a mutex (calls are thread-safe).
struct MapKey {
    uint64_t ptr, inner, outer, batch, ld, stride;
    uint32_t box_inner, box_outer, dt, es, swz, pad;
    bool operator==(const MapKey& o) const { return std::memcmp(this, &o, sizeof(MapKey)) == 0; }
};
struct MapEntry {
    bool valid = false;
    MapKey key;
    CUtensorMap map;
};
constexpr int kMapSlots = 256;
std::mutex g_map_mu;
MapEntry g_maps[kMapSlots];
std::atomic<uint64_t> g_map_hits{0}, g_map_misses{0};

uint64_t map_hash(const MapKey& k) {
    const uint64_t* w = reinterpret_cast<const uint64_t*>(&k);
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < sizeof(MapKey) / 8; ++i) {
        h ^= w[i];
        h *= 1099511628211ull;
        h ^= h >> 29;
    }
    return h;
}

// 3-D map {inner, outer, batch} with 128-B swizzle; OOB elements load as zero, stores clip.
bool encode3d(CUtensorMap* m, CUtensorMapDataType dt, int es, const void* ptr, int64_t inner, int64_t outer,
              int64_t batch, int64_t ld, int64_t stride, uint32_t box_inner, uint32_t box_outer,
              CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    MapKey key;
    std::memset(&key, 0, sizeof key);
    key.ptr = reinterpret_cast<uint64_t>(ptr);
    key.inner = static_cast<uint64_t>(inner);
    key.outer = static_cast<uint64_t>(outer);
    key.batch = static_cast<uint64_t>(batch);
    key.ld = static_cast<uint64_t>(ld);
    key.stride = static_cast<uint64_t>(batch > 1 ? stride : 0);
    key.box_inner = box_inner;
    key.box_outer = box_outer;
    key.dt = static_cast<uint32_t>(dt);
    key.es = static_cast<uint32_t>(es);
    key.swz = static_cast<uint32_t>(swz);
    MapEntry& slot = g_maps[map_hash(key) % kMapSlots];
    {
        std::lock_guard<std::mutex> lk(g_map_mu);
        if (slot.valid && slot.key == key) {
            *m = slot.map;
            g_map_hits.fetch_add(1, std::memory_order_relaxed);
            return true;
        }
    }
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)batch};
    // byte strides of dims 1 and 2; a 1-item batch gets a harmless non-zero stride
    int64_t s2 = batch > 1 ? stride * es : ld * es * std::max<int64_t>(outer, 1);
    cuuint64_t strides[2] = {(cuuint64_t)(ld * es), (cuuint64_t)s2};
    cuuint32_t box[3] = {box_inner, box_outer, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(m, dt, 3, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    g_map_misses.fetch_add(1, std::memory_order_relaxed);
    std::lock_guard<std::mutex> lk(g_map_mu);
    slot.valid = true;
    slot.key = key;
    slot.map = *m;
    return true;
}

// Swap-AB: C^T = B^T A^T.  Legal where the epilogue commutes with the
// transpose without new bias addressing (ROW <-> COL, no FULL bias), with no prologue on A (it would
// become the MMA's B operand) and no sum of matmuls.  Heuristic: skinny M (<= 64) against a long N,
// where the unswapped tile wastes most of every A stage on zero-filled rows and the 128-row MMA side
// would hold only M valid rows (a shallow ring of useful B bytes, a split-K reduction of mostly zeros).
bool swap_legal(const Args& a) {
    return a.o.prologue == GE_PRO_NONE && a.K2 == 0 && !(has_bias(a.op) && a.o.bias_mode == GE_BIAS_FULL) &&
           a.o.multicast != 2 && a.o.stream_k != 2 && a.o.cta_group != 2 && a.o.tile_n != 512 && a.o.tile_m != 256;
}
bool use_swap(const Args& a) {
    if (a.o.swap_ab == 1 || !swap_legal(a)) return false;
    if (a.o.swap_ab == 2) return true;
    return a.M <= 64 && a.N >= 1024 && !a.o.tile_n && !a.o.cta_group && !a.o.tile_m;
}
// The swapped problem: A' = B^T (M' = N), B' = A^T (N' = M); a transposed view flips the layout
// bit and keeps the leading dimension; the bias modes ROW (bias[j]) and COL (bias[i]) trade places.
Args swapped(const Args& a) {
    Args t = a;
    t.M = a.N;
    t.N = a.M;
    t.la = a.lb == GE_ROW_MAJOR ? GE_COL_MAJOR : GE_ROW_MAJOR;
    t.lb = a.la == GE_ROW_MAJOR ? GE_COL_MAJOR : GE_ROW_MAJOR;
    t.A = a.B;
    t.lda = a.ldb;
    t.sA = a.sB;
    t.B = a.A;
    t.ldb = a.lda;
    t.sB = a.sA;
    if (has_bias(a.op)) t.o.bias_mode = a.o.bias_mode == GE_BIAS_ROW ? GE_BIAS_COL : GE_BIAS_ROW;
    return t;
}

ge_status launch_impl(Args& a, cudaStream_t st, bool c_trans);

ge_status launch(Args& a, cudaStream_t st) {
    ge_status s = validate(a);
    if (s != GE_OK) return s;
    if (a.batch == 0 || a.M == 0 || a.N == 0) return GE_OK;
    if (use_swap(a)) {
        Args t = swapped(a);
        return launch_impl(t, st, true);
    }
    return launch_impl(a, st, false);
}

// Plan, encode and launch an already validated problem (c_trans: store C transposed, swap-AB).
ge_status launch_impl(Args& a, cudaStream_t st, bool c_trans) {
    ge_status s;
    int sms = 0;
    s = device_info(&sms);
    if (s != GE_OK) return s;
    // Stream-K needs the caller's workspace (header: no device allocation on this entry point)
    const bool have_ws = a.o.workspace != nullptr;
    if (a.o.stream_k == 2 && !have_ws)
        return fail(GE_ERR_INVALID_VALUE, "stream_k = 2 needs a workspace (size: ge_plan's workspace_bytes)");
    Plan pl = make_plan(a, sms, split_capacity(), have_ws);
    if (pl.sk_tiles && static_cast<size_t>(a.o.workspace_bytes) < sk_workspace_bytes(pl)) {
        if (a.o.stream_k == 2) return fail(GE_ERR_INVALID_VALUE, "workspace smaller than ge_plan's workspace_bytes");
        pl = make_plan(a, sms, split_capacity(), false);
    }
    const bool arow = a.la == GE_ROW_MAJOR, brow = a.lb == GE_ROW_MAJOR;
    const bool a_mn = !arow, b_mn = brow;          // row-major A is K-major; row-major B is N(MN)-major
    const bool f32 = a.o.out_dtype == GE_OUT_F32;
    // prologue kernel variant: 1 in-place op on A, 2 with the Hadamard S tile staged next to A
    const int pro = a.o.prologue == GE_PRO_NONE ? 0 : a.o.prologue == GE_PRO_HADAMARD ? 2 : 1;
    const int es = f32 ? 4 : 2;

    ge::Maps maps;
    std::memset(&maps, 0, sizeof maps);
    if (a.K > 0) {
        bool ok;
        const uint32_t arows = pl.hr ? 64 : 128;                       // A rows per CTA (the K-major box)
        if (!a_mn) ok = encode3d(&maps.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.A, a.K, a.M, a.batch, a.lda, a.sA, 64, arows);
        else ok = encode3d(&maps.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.A, a.M, a.K, a.batch, a.lda, a.sA, 64, 64);
        if (!ok) return fail(GE_ERR_CUDA, "cuTensorMapEncodeTiled failed for A");
        // B rows per MMA per CTA; multicast clusters load (and multicast) half of them per CTA
        const uint32_t brows = static_cast<uint32_t>(std::min(pl.bn, 256) / pl.cg / (pl.mc ? 2 : 1));
        if (!b_mn) ok = encode3d(&maps.b, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.B, a.K, a.N, a.batch, a.ldb, a.sB, 64, brows);
        else ok = encode3d(&maps.b, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.B, a.N, a.K, a.batch, a.ldb, a.sB, 64, 64);
        if (!ok) return fail(GE_ERR_CUDA, "cuTensorMapEncodeTiled failed for B");
    }
    if (a.K > 0 && pro == 2) {
        // Hadamard S: A's geometry and box (it lands at the same swizzled offsets as A); the P slot
        const int64_t sT = a.batch > 1 ? a.o.stride_prologue_tile : 0;
        bool ok;
        if (!a_mn) ok = encode3d(&maps.p, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.o.prologue_tile, a.K, a.M,
                                 sT ? a.batch : 1, a.o.ld_prologue_tile, sT, 64, pl.hr ? 64 : 128);
        else ok = encode3d(&maps.p, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.o.prologue_tile, a.M, a.K,
                           sT ? a.batch : 1, a.o.ld_prologue_tile, sT, 64, 64);
        if (!ok) return fail(GE_ERR_CUDA, "cuTensorMapEncodeTiled failed for the prologue tile");
    }
    if (a.K2 > 0) {
        bool ok;
        if (!a_mn) ok = encode3d(&maps.p, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.P, a.K2, a.M, 1, a.ldp, 0, 64, pl.hr ? 64 : 128);
        else ok = encode3d(&maps.p, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.P, a.M, a.K2, 1, a.ldp, 0, 64, 64);
        if (!ok) return fail(GE_ERR_CUDA, "cuTensorMapEncodeTiled failed for P");
        const uint32_t brows = static_cast<uint32_t>(std::min(pl.bn, 256) / pl.cg / (pl.mc ? 2 : 1));
        if (!b_mn) ok = encode3d(&maps.q, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.Q, a.K2, a.N, 1, a.ldq, 0, 64, brows);
        else ok = encode3d(&maps.q, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a.Q, a.N, a.K2, 1, a.ldq, 0, 64, 64);
        if (!ok) return fail(GE_ERR_CUDA, "cuTensorMapEncodeTiled failed for Q");
    }
    // swap-AB (c_trans): the map describes the caller's C (a.N rows of a.M columns); the kernel
    // stages each 32 x 32 block transposed and stores it with the coordinates swapped.  The TMA store
    // clips the inner dimension only at 16-B granularity (measured: a ragged width wrote into the
    // caller's padding), so the map's inner extent is the width rounded down to 16 B and the kernel
    // writes the ragged edge element-wise.
    const int64_t c_inner = c_trans ? a.M : a.N, c_outer = c_trans ? a.N : a.M;
    const int64_t c_ext = c_inner / (16 / es) * (16 / es);
    const bool c_tma = (reinterpret_cast<uintptr_t>(a.C) % 16 == 0) && ((a.ldc * es) % 16 == 0) &&
                       (a.batch == 1 || (a.sC * es) % 16 == 0) && c_ext > 0;
    if (c_tma) {
        if (!encode3d(&maps.c, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, es, a.C, c_ext,
                      c_outer, a.batch, a.ldc, a.sC, 32, 32, f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B))
            return fail(GE_ERR_CUDA, "cuTensorMapEncodeTiled failed for C");
    }

    ge::Params p{};
    p.M = static_cast<int>(a.M);
    p.N = static_cast<int>(a.N);
    p.K = static_cast<int>(a.K);
    p.batch = static_cast<int>(a.batch);
    p.num_m_tiles = static_cast<int>(cdiv(a.M, pl.hr ? 128 : 128 * pl.cg * (pl.mc ? 2 : 1)));
    p.num_n_tiles = static_cast<int>(cdiv(a.N, pl.bn));
    p.a_mn = a_mn ? 1 : 0;
    p.b_mn = b_mn ? 1 : 0;
    p.num_k_blocks1 = static_cast<int>(cdiv(a.K, ge::kBK));
    p.num_k_blocks = p.num_k_blocks1 + static_cast<int>(cdiv(a.K2, ge::kBK));
    p.group_m = group_m_for(pl, a, sms);
    {
        static int hints[3] = {-1, -1, -1};
        static std::once_flag once;
        std::call_once(once, [] {
            const char* e = getenv("GE_L2_HINTS");     // tuning only: "a,b,c" with 0 normal 1 first 2 last
            if (e) sscanf(e, "%d,%d,%d", &hints[0], &hints[1], &hints[2]);
        });
        p.hint_a = hints[0] >= 0 ? hints[0] : 0;
        p.hint_b = hints[1] >= 0 ? hints[1] : 0;
        p.hint_c = hints[2] >= 0 ? hints[2] : 0;
    }
    p.num_tiles = pl.tiles;
    p.bias = has_bias(a.op) ? static_cast<const __half*>(a.bias) : nullptr;
    p.bias_mode = has_bias(a.op) ? a.o.bias_mode : ge::BIAS_NONE;
    p.ldbias = a.o.ldbias;
    p.stride_bias = a.sBias;
    p.bias_vec = p.bias && (reinterpret_cast<uintptr_t>(p.bias) % 16 == 0) && (a.sBias % 8 == 0) &&
                 (a.o.bias_mode != GE_BIAS_FULL || a.o.ldbias % 8 == 0);
    p.act = act_of(a.op);
    p.bias_sign = (a.op & GE_EPI_SUB) ? -1.0f : 1.0f;
    p.literal = (a.op & GE_EPI_F16_INTERMEDIATE) ? 1 : 0;
    p.scale = a.o.prologue == GE_PRO_SCALE_K ? a.o.prologue_scale : nullptr;
    p.prologue = a.o.prologue;
    p.scale_vec = p.scale && (reinterpret_cast<uintptr_t>(p.scale) % 16 == 0);
    p.s_batched = (a.batch > 1 && a.o.stride_prologue_tile != 0) ? 1 : 0;

    p.C = a.C;
    p.ldc = a.ldc;
    p.stride_c = a.sC;
    p.c_tma = c_tma ? 1 : 0;
    p.c_vec = c_tma ? 1 : 0;                      // same alignment conditions as the TMA store
    p.c_trans = c_trans ? 1 : 0;
    p.c_ext = static_cast<int>(c_ext);

#if GE_DBG
    // diagnostics build only (libgemm_epilogue_dbg.so): counters and timing experiments
    p.dbg = debug_buffer(sms);
    p.tl = g_timeline;
    static const int noload = getenv("GE_DEBUG_NOLOAD") ? 1 : 0;   // timing experiment only
    p.dbg_noload = noload;
    static const int dflags = getenv("GE_DEBUG_FLAGS") ? atoi(getenv("GE_DEBUG_FLAGS")) : 0;   // experiments only
    p.dbg_flags = dflags;
    if (dflags & 4) p.c_tma = 0;                  // experiment: st.global epilogue instead of TMA stores
#endif

    // stream-K (last partial wave split across all clusters) in the caller's workspace
    Plan plan = pl;
    p.dp_tiles = plan.tiles;
    p.sk_units = 0;
    p.sk_ws = nullptr;
    p.sk_flags = nullptr;
    p.splits = plan.splits;
    if (plan.sk_tiles) {
        const size_t ctas = static_cast<size_t>(plan.clusters * plan.cg);
        p.sk_ws = static_cast<float*>(a.o.workspace);
        p.sk_flags = reinterpret_cast<unsigned int*>(static_cast<char*>(a.o.workspace) + ctas * 128 * plan.bn * 4);
        p.dp_tiles = plan.tiles - plan.sk_tiles;
        p.sk_units = plan.sk_tiles * p.num_k_blocks;
    }
    const int grid = static_cast<int>(std::max<int64_t>(plan.clusters, 1) * plan.cg * (plan.mc ? 2 : 1));
    cudaError_t e;
    if (pl.hr) {
        if (pl.bn == 128) e = ge::launch_cg2_bn128_hr(f32, pro, maps, p, grid, st);
        else e = ge::launch_cg2_bn256_hr(f32, pro, maps, p, grid, st);
    } else if (pl.mc) {
        if (pl.bn == 512) e = ge::launch_cg2_bn512_mc(f32, pro, maps, p, grid, st);
        else e = ge::launch_cg2_bn256_mc(f32, pro, maps, p, grid, st);
    } else if (pl.cg == 1) {
        if (pl.bn == 64) e = ge::launch_cg1_bn64(f32, pro, maps, p, grid, st);
        else if (pl.bn == 128) e = ge::launch_cg1_bn128(f32, pro, maps, p, grid, st);
        else if (pl.bn == 192) e = ge::launch_cg1_bn192(f32, pro, maps, p, grid, st);
        else e = ge::launch_cg1_bn256(f32, pro, maps, p, grid, st);
    } else {
        if (pl.bn == 128) e = ge::launch_cg2_bn128(f32, pro, maps, p, grid, st);
        else if (pl.bn == 192) e = ge::launch_cg2_bn192(f32, pro, maps, p, grid, st);
        else if (pl.bn == 256) e = ge::launch_cg2_bn256(f32, pro, maps, p, grid, st);
        else e = ge::launch_cg2_bn512(f32, pro, maps, p, grid, st);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(GE_ERR_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(e));
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return GE_OK;
}

Args make_args(int64_t batch, int64_t M, int64_t N, int64_t K, int32_t la, int32_t lb, const void* A, int64_t lda,
               int64_t sA, const void* B, int64_t ldb, int64_t sB, const void* bias, int64_t sBias, void* C,
               int64_t ldc, int64_t sC, int32_t op, const ge_options* opt) {
    Args a{batch, M, N, K, la, lb, A, lda, sA, B, ldb, sB, bias, sBias, C, ldc, sC, op, {}};
    if (opt) a.o = *opt;
    else a.o = ge_options{GE_BIAS_ROW, 0, GE_PRO_NONE, nullptr, GE_OUT_F16, 0, 0, 0, nullptr, 0, 0, nullptr, 0, 0, 0, 0};
    return a;
}

// ------------------------------------------------------------------ host-buffer workspace
struct Workspace {
    void* ptr = nullptr;
    size_t bytes = 0;
};
std::mutex g_ws_mu;
Workspace g_ws[64];

// Copy/compute streams and events of the pipelined host-buffer path, one set per device
// (used under g_ws_mu).
constexpr int kPipeBlocks = 8;
struct PipeStreams {
    bool init = false, ok = false;
    cudaStream_t h2d = nullptr, cmp = nullptr, d2h = nullptr;
    cudaEvent_t ev_start = nullptr, ev_end = nullptr, ev_in[kPipeBlocks] = {}, ev_out[kPipeBlocks] = {};
};
PipeStreams g_pipe[64];
PipeStreams& pipe_streams(int dev) {
    PipeStreams& p = g_pipe[dev & 63];
    if (!p.init) {
        p.init = true;
        bool ok = cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaStreamCreateWithFlags(&p.cmp, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaEventCreateWithFlags(&p.ev_start, cudaEventDisableTiming) == cudaSuccess &&
                  cudaEventCreateWithFlags(&p.ev_end, cudaEventDisableTiming) == cudaSuccess;
        for (int i = 0; ok && i < kPipeBlocks; ++i)
            ok = cudaEventCreateWithFlags(&p.ev_in[i], cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&p.ev_out[i], cudaEventDisableTiming) == cudaSuccess;
        if (!ok) cudaGetLastError();
        p.ok = ok;
    }
    return p;
}

}  // namespace

namespace ge {
int clusters_cg1(int bn, int cluster) {
    return bn == 64 ? clusters_cg1_bn64(cluster) : bn == 128 ? clusters_cg1_bn128(cluster)
         : bn == 192 ? clusters_cg1_bn192(cluster) : clusters_cg1_bn256(cluster);
}
template <bool SX>
int smem_bytes_t(int bn, int cg, bool hr) {
    if (hr) return bn == 128 ? Cfg<128, 2, SX, true>::kSmemBytes : Cfg<256, 2, SX, true>::kSmemBytes;
    if (cg == 1)
        return bn == 64 ? Cfg<64, 1, SX>::kSmemBytes : bn == 128 ? Cfg<128, 1, SX>::kSmemBytes
             : bn == 192 ? Cfg<192, 1, SX>::kSmemBytes : Cfg<256, 1, SX>::kSmemBytes;
    return bn == 128 ? Cfg<128, 2, SX>::kSmemBytes : bn == 192 ? Cfg<192, 2, SX>::kSmemBytes
         : bn == 256 ? Cfg<256, 2, SX>::kSmemBytes : Cfg<512, 2, SX>::kSmemBytes;
}
template <bool SX>
int stages_t(int bn, int cg, bool hr) {
    if (hr) return bn == 128 ? Cfg<128, 2, SX, true>::kStages : Cfg<256, 2, SX, true>::kStages;
    if (cg == 1)
        return bn == 64 ? Cfg<64, 1, SX>::kStages : bn == 128 ? Cfg<128, 1, SX>::kStages
             : bn == 192 ? Cfg<192, 1, SX>::kStages : Cfg<256, 1, SX>::kStages;
    return bn == 128 ? Cfg<128, 2, SX>::kStages : bn == 192 ? Cfg<192, 2, SX>::kStages
         : bn == 256 ? Cfg<256, 2, SX>::kStages : Cfg<512, 2, SX>::kStages;
}
int smem_bytes_for(int bn, int cg, bool sx, bool hr) {
    return sx ? smem_bytes_t<true>(bn, cg, hr) : smem_bytes_t<false>(bn, cg, hr);
}
int stages_for(int bn, int cg, bool sx, bool hr) { return sx ? stages_t<true>(bn, cg, hr) : stages_t<false>(bn, cg, hr); }
}  // namespace ge

extern "C" {

ge_status gemm_epilogue(int64_t M, int64_t N, int64_t K, int32_t layoutA, int32_t layoutB, const void* A, int64_t lda,
                        const void* B, int64_t ldb, const void* bias, void* C, int64_t ldc, int32_t op,
                        const ge_options* opt, void* stream) {
    Args a = make_args(1, M, N, K, layoutA, layoutB, A, lda, 0, B, ldb, 0, bias, 0, C, ldc, 0, op, opt);
    g_detail.clear();
    return launch(a, static_cast<cudaStream_t>(stream));
}

ge_status gemm_epilogue_batched(int64_t batch, int64_t M, int64_t N, int64_t K, int32_t layoutA, int32_t layoutB,
                                const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb,
                                int64_t strideB, const void* bias, int64_t strideBias, void* C, int64_t ldc,
                                int64_t strideC, int32_t op, const ge_options* opt, void* stream) {
    Args a = make_args(batch, M, N, K, layoutA, layoutB, A, lda, strideA, B, ldb, strideB, bias, strideBias, C, ldc,
                       strideC, op, opt);
    g_detail.clear();
    return launch(a, static_cast<cudaStream_t>(stream));
}

ge_status gemm2_epilogue(int64_t M, int64_t N, int64_t K1, int64_t K2, int32_t layoutA, int32_t layoutB,
                         const void* A, int64_t lda, const void* B, int64_t ldb, const void* P, int64_t ldp,
                         const void* Q, int64_t ldq, const void* bias, void* C, int64_t ldc, int32_t op,
                         const ge_options* opt, void* stream) {
    Args a = make_args(1, M, N, K1, layoutA, layoutB, A, lda, 0, B, ldb, 0, bias, 0, C, ldc, 0, op, opt);
    a.K2 = K2;
    a.P = P;
    a.ldp = ldp;
    a.Q = Q;
    a.ldq = ldq;
    g_detail.clear();
    return launch(a, static_cast<cudaStream_t>(stream));
}

ge_status ge_validate(int64_t batch, int64_t M, int64_t N, int64_t K, int32_t layoutA, int32_t layoutB, const void* A,
                      int64_t lda, int64_t strideA, const void* B, int64_t ldb, int64_t strideB, const void* bias,
                      int64_t strideBias, void* C, int64_t ldc, int64_t strideC, int32_t op, const ge_options* opt) {
    Args a = make_args(batch, M, N, K, layoutA, layoutB, A, lda, strideA, B, ldb, strideB, bias, strideBias, C, ldc,
                       strideC, op, opt);
    g_detail.clear();
    return validate(a);
}

ge_status gemm_epilogue_host(int64_t batch, int64_t M, int64_t N, int64_t K, int32_t layoutA, int32_t layoutB,
                             const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb, int64_t strideB,
                             const void* bias, int64_t strideBias, void* C, int64_t ldc, int64_t strideC, int32_t op,
                             const ge_options* opt, void* stream) {
    g_detail.clear();
    Args a = make_args(batch, M, N, K, layoutA, layoutB, A, lda, strideA, B, ldb, strideB, bias, strideBias, C, ldc,
                       strideC, op, opt);
    ge_status s = validate(a);
    if (s != GE_OK) return s;
    if (a.batch == 0 || a.M == 0 || a.N == 0) return GE_OK;
    int sms = 0;
    s = device_info(&sms);
    if (s != GE_OK) return s;
    const bool arow = a.la == GE_ROW_MAJOR, brow = a.lb == GE_ROW_MAJOR;
    const int es = a.o.out_dtype == GE_OUT_F32 ? 4 : 2;
    const int64_t nA = a.K ? extent_bytes(a.batch, arow ? a.M : a.K, arow ? a.K : a.M, a.lda, a.sA, 2) : 0;
    const int64_t nB = a.K ? extent_bytes(a.batch, brow ? a.K : a.N, brow ? a.N : a.K, a.ldb, a.sB, 2) : 0;
    int64_t nBias = 0;
    if (has_bias(a.op)) {
        if (a.o.bias_mode == GE_BIAS_ROW) nBias = ((a.batch - 1) * a.sBias + a.N) * 2;
        else if (a.o.bias_mode == GE_BIAS_COL) nBias = ((a.batch - 1) * a.sBias + a.M) * 2;
        else nBias = extent_bytes(a.batch, a.M, a.N, a.o.ldbias, a.sBias, 2);
    }
    const int64_t nS = (a.o.prologue == GE_PRO_SCALE_K && a.K) ? a.K * 4 : 0;
    // Hadamard prologue tile S (A's layout): copied whole, up front like B
    const int64_t nT = (a.o.prologue == GE_PRO_HADAMARD && a.K)
                           ? extent_bytes(a.o.stride_prologue_tile ? a.batch : 1, arow ? a.M : a.K, arow ? a.K : a.M,
                                          a.o.ld_prologue_tile, a.o.stride_prologue_tile, 2)
                           : 0;
    const int64_t nC = extent_bytes(a.batch, a.M, a.N, a.ldc, a.sC, es);
    auto up = [](int64_t x) { return (x + 255) / 256 * 256; };
    // stream-K workspace of the launches below (one fp32 128 x 256 slot and one flag per CTA,
    // zero-filled once when allocated; every launch leaves the flags at zero)
    const int64_t nSK = up(static_cast<int64_t>(sms) * (128 * 256 * 4 + 4));
    const size_t need = nSK + up(nA) + up(nB) + up(nBias) + up(nS) + up(nT) + up(nC);
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_ws_mu);
    Workspace& ws = g_ws[dev & 63];
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (ws.bytes < need) {
        if (ws.ptr) {
            cudaStreamSynchronize(st);
            cudaFree(ws.ptr);
        }
        ws.ptr = nullptr;
        ws.bytes = 0;
        if (cudaMalloc(&ws.ptr, need) != cudaSuccess) {
            cudaGetLastError();
            return fail(GE_ERR_CUDA, "workspace cudaMalloc failed");
        }
        ws.bytes = need;
        if (cudaMemsetAsync(ws.ptr, 0, nSK, st) != cudaSuccess) {
            cudaGetLastError();
            return fail(GE_ERR_CUDA, "workspace memset failed");
        }
    }
    char* base = static_cast<char*>(ws.ptr);
    char* dSK = base;
    char* dA = base + nSK;
    char* dB = dA + up(nA);
    char* dBias = dB + up(nB);
    char* dS = dBias + up(nBias);
    char* dT = dS + up(nS);
    char* dC = dT + up(nT);
    // Pipelined end-to-end path: B, bias and scale go first, then A and C
    // move in blocks (rows of A / C, or whole batch items) so that the GEMM and the C read-back of
    // one block overlap the host->device copy of the next (separate copy engines per direction).
    PipeStreams& ps = pipe_streams(dev);
    if (!ps.ok) return fail(GE_ERR_CUDA, "could not create the copy/compute streams");
    auto chk = [&](cudaError_t e, const char* what) {
        if (e == cudaSuccess) return true;
        cudaGetLastError();
        fail(GE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
        return false;
    };
    if (!chk(cudaEventRecord(ps.ev_start, st), "event")) return GE_ERR_CUDA;
    if (!chk(cudaStreamWaitEvent(ps.h2d, ps.ev_start, 0), "event")) return GE_ERR_CUDA;
    if (nB && !chk(cudaMemcpyAsync(dB, a.B, nB, cudaMemcpyHostToDevice, ps.h2d), "H2D B")) return GE_ERR_CUDA;
    if (nBias && !chk(cudaMemcpyAsync(dBias, a.bias, nBias, cudaMemcpyHostToDevice, ps.h2d), "H2D bias"))
        return GE_ERR_CUDA;
    if (nS && !chk(cudaMemcpyAsync(dS, a.o.prologue_scale, nS, cudaMemcpyHostToDevice, ps.h2d), "H2D scale"))
        return GE_ERR_CUDA;
    if (nT && !chk(cudaMemcpyAsync(dT, a.o.prologue_tile, nT, cudaMemcpyHostToDevice, ps.h2d), "H2D prologue tile"))
        return GE_ERR_CUDA;
    // blocks: batch items when batched, else row blocks (multiples of the 256-row pair tile)
    const bool by_item = a.batch > 1;
    const int64_t units = by_item ? a.batch : a.M;
    int64_t nblk = by_item ? std::min<int64_t>(a.batch, kPipeBlocks) : std::min<int64_t>(kPipeBlocks, a.M / 1024);
    nblk = std::max<int64_t>(nblk, 1);
    int64_t per = cdiv(units, nblk);
    if (!by_item) per = cdiv(per, 256) * 256;
    nblk = cdiv(units, per);
    for (int64_t blk = 0; blk < nblk; ++blk) {
        const int64_t u0 = blk * per, u1 = std::min(units, u0 + per);
        // host -> device: this block of A
        if (nA) {
            cudaError_t e;
            if (by_item) {
                const int64_t item = extent_bytes(1, arow ? a.M : a.K, arow ? a.K : a.M, a.lda, 0, 2);
                const int64_t off = u0 * a.sA * 2, bytes = (u1 - u0 - 1) * a.sA * 2 + item;
                e = cudaMemcpyAsync(dA + off, static_cast<const char*>(a.A) + off, bytes, cudaMemcpyHostToDevice,
                                    ps.h2d);
            } else if (arow) {
                const int64_t off = u0 * a.lda * 2, bytes = ((u1 - u0 - 1) * a.lda + a.K) * 2;
                e = cudaMemcpyAsync(dA + off, static_cast<const char*>(a.A) + off, bytes, cudaMemcpyHostToDevice,
                                    ps.h2d);
            } else {
                e = cudaMemcpy2DAsync(dA + u0 * 2, a.lda * 2, static_cast<const char*>(a.A) + u0 * 2, a.lda * 2,
                                      (u1 - u0) * 2, a.K, cudaMemcpyHostToDevice, ps.h2d);
            }
            if (!chk(e, "H2D A")) return GE_ERR_CUDA;
        }
        if (!chk(cudaEventRecord(ps.ev_in[blk], ps.h2d), "event")) return GE_ERR_CUDA;
        if (!chk(cudaStreamWaitEvent(ps.cmp, ps.ev_in[blk], 0), "event")) return GE_ERR_CUDA;
        // the fused kernel on this block
        Args d = a;
        d.o.workspace = dSK;
        d.o.workspace_bytes = nSK;
        d.B = nB ? dB : nullptr;
        d.o.prologue_scale = nS ? reinterpret_cast<const float*>(dS) : nullptr;
        d.o.prologue_tile = nT ? dT : nullptr;
        if (by_item) {
            d.batch = u1 - u0;
            if (nT && a.o.stride_prologue_tile) d.o.prologue_tile = dT + u0 * a.o.stride_prologue_tile * 2;
            d.A = nA ? dA + u0 * a.sA * 2 : nullptr;
            d.B = nB ? dB + u0 * a.sB * 2 : nullptr;
            d.C = dC + u0 * a.sC * es;
            d.bias = nBias ? dBias + u0 * a.sBias * 2 : nullptr;
        } else {
            d.M = u1 - u0;
            d.A = nA ? dA + (arow ? u0 * a.lda : u0) * 2 : nullptr;
            if (nT) d.o.prologue_tile = dT + (arow ? u0 * a.o.ld_prologue_tile : u0) * 2;
            d.C = dC + u0 * a.ldc * es;
            d.bias = nullptr;
            if (nBias) {
                const int64_t boff = a.o.bias_mode == GE_BIAS_ROW ? 0 : a.o.bias_mode == GE_BIAS_COL ? u0 : u0 * a.o.ldbias;
                d.bias = dBias + boff * 2;
            }
        }
        if (d.K > 0 && !d.A) d.A = dA;
        s = launch(d, ps.cmp);
        if (s != GE_OK) return s;
        if (!chk(cudaEventRecord(ps.ev_out[blk], ps.cmp), "event")) return GE_ERR_CUDA;
        if (!chk(cudaStreamWaitEvent(ps.d2h, ps.ev_out[blk], 0), "event")) return GE_ERR_CUDA;
        // device -> host: the block's M x N window of C (the caller's padding is left untouched)
        cudaError_t e = cudaSuccess;
        if (by_item) {
            for (int64_t b = u0; b < u1 && e == cudaSuccess; ++b)
                e = cudaMemcpy2DAsync(static_cast<char*>(a.C) + b * a.sC * es, a.ldc * es, dC + b * a.sC * es,
                                      a.ldc * es, a.N * es, a.M, cudaMemcpyDeviceToHost, ps.d2h);
        } else {
            e = cudaMemcpy2DAsync(static_cast<char*>(a.C) + u0 * a.ldc * es, a.ldc * es, dC + u0 * a.ldc * es,
                                  a.ldc * es, a.N * es, u1 - u0, cudaMemcpyDeviceToHost, ps.d2h);
        }
        if (!chk(e, "D2H C")) return GE_ERR_CUDA;
    }
    if (!chk(cudaEventRecord(ps.ev_end, ps.d2h), "event")) return GE_ERR_CUDA;
    if (!chk(cudaStreamWaitEvent(st, ps.ev_end, 0), "event")) return GE_ERR_CUDA;
    if (!chk(cudaStreamSynchronize(st), "host path")) return GE_ERR_CUDA;
    return GE_OK;
}

ge_status ge_release_workspace(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return fail(GE_ERR_UNSUPPORTED_DEVICE, "no CUDA device");
    }
    std::lock_guard<std::mutex> lk(g_ws_mu);
    Workspace& ws = g_ws[dev & 63];
    if (ws.ptr) {
        cudaDeviceSynchronize();
        cudaFree(ws.ptr);
    }
    ws.ptr = nullptr;
    ws.bytes = 0;
    return GE_OK;
}

const char* ge_status_string(ge_status s) {
    switch (s) {
    case GE_OK: return "GE_OK";
    case GE_ERR_INVALID_VALUE: return "GE_ERR_INVALID_VALUE: invalid argument";
    case GE_ERR_MISALIGNED: return "GE_ERR_MISALIGNED: operand breaks the 16-byte TMA alignment rules";
    case GE_ERR_ALIASING: return "GE_ERR_ALIASING: output overlaps an input";
    case GE_ERR_UNSUPPORTED_DEVICE: return "GE_ERR_UNSUPPORTED_DEVICE: needs an sm_100 (B200) device";
    case GE_ERR_CUDA: return "GE_ERR_CUDA: CUDA call failed";
    }
    return "unknown ge_status";
}

const char* ge_last_error_detail(void) { return g_detail.c_str(); }

ge_status ge_plan(int64_t batch, int64_t M, int64_t N, int64_t K, int32_t layoutA, int32_t layoutB,
                  const ge_options* opt, int32_t num_sms, int32_t* tile_m, int32_t* tile_n, int32_t* cta_group,
                  int32_t* stages, int64_t* num_tiles, int64_t* stream_k_tiles, int64_t* workspace_bytes,
                  int32_t* split_k) {
    g_detail.clear();
    Args a = make_args(batch, M, N, K, layoutA, layoutB, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0, nullptr, 0, 0,
                       GE_EPI_NONE, opt);
    if (batch < 0 || M < 0 || N < 0 || K < 0 || num_sms <= 0) return fail(GE_ERR_INVALID_VALUE, "bad plan arguments");
    {
        const ge_status so = validate_options(a);
        if (so != GE_OK) return so;
    }
    // descriptive: assumes the caller will pass a workspace of *workspace_bytes when stream-K is planned
    const Plan p = make_plan(a, num_sms, split_capacity(), true);     // (nullptr without a device)
    if (tile_m) *tile_m = p.hr ? 128 : 128 * p.cg * (p.mc ? 2 : 1);
    if (tile_n) *tile_n = p.bn;
    if (cta_group) *cta_group = p.cg;
    if (stages) *stages = p.stages;
    if (num_tiles) *num_tiles = p.tiles;
    if (stream_k_tiles) *stream_k_tiles = p.sk_tiles;
    if (workspace_bytes) *workspace_bytes = static_cast<int64_t>(sk_workspace_bytes(p));
    if (split_k) *split_k = p.splits > 1 ? p.splits : 1;
    return GE_OK;
}

ge_status ge_plan_ex(int64_t batch, int64_t M, int64_t N, int64_t K, int32_t layoutA, int32_t layoutB, int32_t op,
                     const ge_options* opt, int32_t num_sms, ge_plan_info* out) {
    g_detail.clear();
    Args a = make_args(batch, M, N, K, layoutA, layoutB, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0, nullptr, 0, 0, op,
                       opt);
    if (batch < 0 || M < 0 || N < 0 || K < 0 || num_sms <= 0 || !out) return fail(GE_ERR_INVALID_VALUE, "bad plan arguments");
    if (!op_valid(op)) return fail(GE_ERR_INVALID_VALUE, "bad epilogue op (see ge_epilogue_op flags)");
    {
        const ge_status so = validate_options(a);
        if (so != GE_OK) return so;
    }
    const bool sw = use_swap(a);
    const Args t = sw ? swapped(a) : a;
    const Plan p = make_plan(t, num_sms, split_capacity(), true);
    out->tile_m = p.hr ? 128 : 128 * p.cg * (p.mc ? 2 : 1);
    out->tile_n = p.bn;
    out->cta_group = p.cg;
    out->stages = p.stages;
    out->num_tiles = p.tiles;
    out->stream_k_tiles = p.sk_tiles;
    out->workspace_bytes = static_cast<int64_t>(sk_workspace_bytes(p));
    out->split_k = p.splits > 1 ? p.splits : 1;
    out->multicast = p.mc ? 1 : 0;
    out->swap_ab = sw ? 1 : 0;
    return GE_OK;
}

uint64_t ge_launch_count(void) { return g_launches.load(); }

void ge_tensor_map_cache_stats(uint64_t* hits, uint64_t* misses) {
    if (hits) *hits = g_map_hits.load();
    if (misses) *misses = g_map_misses.load();
}

int32_t ge_debug_read(uint64_t* out, int32_t max_ctas) {
    if (g_dbg_last < 0 || !g_dbg[g_dbg_last] || !out) return 0;
    const int n = std::min(max_ctas, g_dbg_ctas[g_dbg_last]);
    if (cudaMemcpy(out, g_dbg[g_dbg_last], sizeof(uint64_t) * ge::DBG_SLOTS * n, cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// Debug build only (not in the header): set the timeline buffer (nullptr: off).  Layout: word 0 =
// launch counter, then 24 words per launch (see ge_kernel.cuh TL_*).
void ge_debug_set_timeline(unsigned long long* dev_buf) { g_timeline = dev_buf; }

const char* ge_version(void) { return "gemm_epilogue-b200 0.1.0 (sm_100a, tcgen05/TMA/TMEM)"; }

}  // extern "C"
