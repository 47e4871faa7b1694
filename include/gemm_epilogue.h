/*
 * gemm_epilogue.h -- C ABI of the B200 (sm_100a) fused fp16 GEMM + bias + ReLU library.
 *
 * The operation is the epilogue-fusion idiom of "Automatic Kernel Generation for
 * Volta Tensor Cores" (arXiv 2006.12645), Listing 1:
 *
 *     S1: C[i,j] = sum_k A[i,k] * B[k,j]            fp16 inputs, fp32 accumulation
 *     S2: E[i,j] = relu_add(C[i,j], bias[.])         ReLU at the root
 *
 * computed in ONE kernel with no global write of the intermediate C
 * (Sec. VII-A "Avoiding Intermediate Writes To Global Memory"),
 * optionally with a pointwise prologue on A (Sec. VII-C, Listing 5).
 * Readings of the paper that this interface fixes are listed in DESIGN.md (R-C1..R-C16).
 *
 * Conventions common to every entry point
 * ---------------------------------------
 * Element addressing (leading dimension ld counted in ELEMENTS; 0 = packed):
 *     A row-major: a(i,k) = A[i*lda + k], lda >= K      A col-major: a(i,k) = A[k*lda + i], lda >= M
 *     B row-major: b(k,j) = B[k*ldb + j], ldb >= N      B col-major: b(k,j) = B[j*ldb + k], ldb >= K
 *     C is always row-major: c(i,j) = C[i*ldc + j], ldc >= N (PAPER.md:869 stores row-major)
 * Layout pair names: rr, rc, cr, cc = (layout of A, layout of B).  rc is the paper's Listing 2
 * case (A row x B col).  In PyTorch terms rr is `A @ B`.
 * Types: A, B, bias are IEEE binary16; prologue_scale is fp32; C is fp16 (the paper's,
 * PAPER.md:844, 896-897) or fp32 (GE_OUT_F32).  Accumulation is fp32 in Tensor Memory.
 * Epilogue arithmetic is fp32 (acc + bias, then ReLU y = v > 0 ? v : +0), rounded once
 * with round-to-nearest-even at the store (DESIGN.md R-C3, R-C5, R-C6).
 * Ownership: the caller owns every buffer.  The library never allocates device memory on
 * the device-pointer entry points and never retains a pointer after the call returns
 * (the kernel may still be reading it until the stream reaches that point).
 * Streams: device-pointer entry points are asynchronous on `stream` (a cudaStream_t,
 * NULL = legacy default stream) and never synchronize the device.  Results are valid
 * once the caller synchronizes the stream.  Calls are thread-safe.
 * Errors: argument errors are returned synchronously BEFORE any launch, with nothing
 * written.  GE_ERR_CUDA reports a launch failure (detail: ge_last_error_detail()).
 * Asynchronous device faults surface at the caller's next synchronization.
 * Alignment (Tensor Memory Accelerator rules): A and B base pointers must be 16-byte
 * aligned and lda*2, ldb*2 (and batch strides *2) multiples of 16 bytes, else
 * GE_ERR_MISALIGNED.  C, bias and scale have no alignment requirement: a C whose base or
 * ldc is not 16-byte compatible is written by a st.global epilogue instead of TMA stores.
 * Only the M x N window of C is written: elements past column N-1 of a row (the padding of
 * ldc > N) keep their contents, also when N*sizeof(C) is not a multiple of 16 bytes (the TMA
 * store covers the 16-byte-aligned part of each row, the ragged edge is stored element-wise).
 * Aliasing: C must not overlap A, B, bias, scale or the prologue tile (`__restrict__`), else
 * GE_ERR_ALIASING.
 * Degenerate sizes: M == 0 or N == 0 (or batch == 0) is a no-op returning GE_OK.
 * K == 0 gives C = op(bias) (DESIGN.md R-C9).
 */
#ifndef GEMM_EPILOGUE_H
#define GEMM_EPILOGUE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { GE_ROW_MAJOR = 0, GE_COL_MAJOR = 1 } ge_layout;

typedef enum { GE_OUT_F16 = 0, GE_OUT_F32 = 1 } ge_out_dtype;

/* The pointwise epilogue (S2 of Listing 1), bit flags over the paper's op set "add, subtract,
 * ReLU, Sigmoid, Tanh": optionally add (or, with GE_EPI_SUB,
 * subtract) the bias, then at most one activation at the root.  Values 0-3 are the original
 * ops.  Any op with GE_EPI_BIAS needs a non-NULL bias pointer. */
typedef enum {
    GE_EPI_NONE = 0,        /* C = A.B                         (Listing 2, plain GEMM)       */
    GE_EPI_BIAS = 1,        /* C = A.B + beta                                               */
    GE_EPI_RELU = 2,        /* C = relu(A.B)                                                 */
    GE_EPI_BIAS_RELU = 3,   /* C = relu(A.B + beta)            (Listing 1, relu_add)         */
    GE_EPI_SIGMOID = 4,     /* activation flag: 1 / (1 + exp(-v))                            */
    GE_EPI_BIAS_SIGMOID = 5,
    GE_EPI_TANH = 8,        /* activation flag: tanh(v)                                      */
    GE_EPI_BIAS_TANH = 9,
    GE_EPI_SUB = 16,        /* modifier: subtract the bias (v = A.B - beta); needs GE_EPI_BIAS */
    GE_EPI_F16_INTERMEDIATE = 32 /* modifier: the paper-literal rounding point (PAPER.md:1109-1112,
                               1119-1122; DESIGN.md R-C3): the fp32 accumulator is rounded to fp16
                               (RNE) before the pointwise op and acc16 +- beta is rounded to fp16
                               again before the activation, i.e. act(fp16(fp16(acc) +- beta)).
                               Default (flag clear): fp32 throughout, one rounding at the store. */
} ge_epilogue_op;

/* Shape of the bias operand beta (DESIGN.md R-C2). */
typedef enum {
    GE_BIAS_ROW = 0,        /* beta(i,j) = bias[j], length N (default; the DL idiom)          */
    GE_BIAS_COL = 1,        /* beta(i,j) = bias[i], length M                                  */
    GE_BIAS_FULL = 2        /* beta(i,j) = bias[i*ldbias + j], M x N (paper-literal) */
} ge_bias_mode;

/* Pointwise prologue applied to A before the contraction (Sec. VII-C, DESIGN.md R-C12). */
typedef enum {
    GE_PRO_NONE = 0,
    GE_PRO_SCALE_K = 1,     /* a'(i,k) = fp16_rne(s[k] * a(i,k)), s = prologue_scale, fp32, length K */
    GE_PRO_RELU = 2,        /* a'(i,k) = max(a(i,k), +0)  (Listing 5)          */
    GE_PRO_HADAMARD = 3     /* a'(i,k) = fp16_rne(s(i,k) * a(i,k)): a full-tile elementwise scale, a
                               second input dataspace of the prologue's compound op (
                               DESIGN.md R-C18).  S = prologue_tile, fp16, M x K in A's layout
                               (row-major: s(i,k) = S[i*lds + k]; col-major: S[k*lds + i]). */
} ge_prologue_op;

typedef struct {
    int32_t bias_mode;              /* ge_bias_mode */
    int64_t ldbias;                 /* FULL only: row stride of bias in elements (0 = N) */
    int32_t prologue;               /* ge_prologue_op */
    const float* prologue_scale;    /* SCALE_K only: device pointer (host pointer for *_host), length K */
    int32_t out_dtype;              /* ge_out_dtype */
    int32_t tile_n;                 /* 0 = heuristic; else force the N tile (64, 128, 192, 256; 512 with
                                       cta_group 2; 192 with cta_group 2 needs a column-major B) */
    int32_t cta_group;              /* 0 = heuristic; 1 = single-CTA tiles; 2 = CTA-pair tiles */
    int32_t stream_k;               /* 0 = heuristic (stream-K tail or split-K); 1 = off (data-parallel
                                       tiles only); 2 = stream-K (never split-K) whenever the last
                                       wave is partial */
    void* workspace;                /* optional device workspace for stream-K partials (size: ge_plan's
                                       workspace_bytes); 16-byte aligned, ZERO-FILLED before its first
                                       use and left zero-filled by every launch; must not be shared by
                                       launches that may run concurrently.  NULL (or smaller than the
                                       planned size) = no stream-K: the heuristic then plans data-parallel
                                       or split-K tiles only (the library never allocates device memory
                                       on the device-pointer entry points); stream_k = 2 with no or too
                                       small a workspace is GE_ERR_INVALID_VALUE. */
    int64_t workspace_bytes;
    int32_t multicast;              /* 0 = heuristic; 1 = off; 2 = force clusters of two CTA pairs stacked
                                       along M (512 x tile_n tiles) whose B tiles are loaded once and
                                       TMA-multicast to both pairs (a third less L2->SM traffic per flop;
                                       needs no prologue and stream_k != 2; data-parallel tiles only) */
    const void* prologue_tile;      /* HADAMARD only: S (device pointer; host pointer for *_host), fp16,
                                       M x K in A's layout; 16-byte aligned, ld_prologue_tile * 2 and
                                       stride_prologue_tile * 2 multiples of 16 (else GE_ERR_MISALIGNED) */
    int64_t ld_prologue_tile;       /* leading dimension of S in elements (0 = packed: K row-major, M col-major) */
    int64_t stride_prologue_tile;   /* batched: element stride between items' S (0 = one S shared by all) */
    int32_t tile_m;                 /* 0 = heuristic; 128 = 128-row tiles (with cta_group 2: HALF-ROW CTA
                                       pairs, cta_group::2 with M = 128, 64 rows per CTA, tile_n 128/256);
                                       256 = CTA-pair tiles of 256 rows */
    int32_t swap_ab;                /* 0 = heuristic; 1 = never; 2 = always where legal.  Swap-AB computes
                                       C^T = B^T A^T (the long N side becomes the 128-row MMA side, the
                                       skinny M side the MMA N) and stores C transposed; used for skinny
                                       M (<= 64) with ROW/COL/no bias, no prologue, no sum of matmuls
                                       (DESIGN.md "Skinny shapes").  Results stay within the bound; the
                                       summation order may differ from the unswapped launch. */
} ge_options;                       /* NULL options = {ROW, 0, NONE, NULL, F16, 0, 0, 0, NULL, 0, 0, NULL, 0, 0, 0, 0} */

typedef enum {
    GE_OK = 0,
    GE_ERR_INVALID_VALUE = 1,       /* negative size, ld too small, NULL pointer that is needed, bad enum */
    GE_ERR_MISALIGNED = 2,          /* A/B base or stride breaks the 16-byte TMA rules */
    GE_ERR_ALIASING = 3,            /* C overlaps an input */
    GE_ERR_UNSUPPORTED_DEVICE = 4,  /* current device is not sm_100 or no device */
    GE_ERR_CUDA = 5                 /* a CUDA runtime/driver call failed */
} ge_status;

/*
 * Single GEMM: C = epilogue(prologue(A) . B).  All pointers are device pointers on the
 * current device; `stream` is a cudaStream_t.  See conventions above.
 */
ge_status gemm_epilogue(int64_t M, int64_t N, int64_t K,
                        int32_t layoutA, int32_t layoutB,
                        const void* A, int64_t lda,
                        const void* B, int64_t ldb,
                        const void* bias,
                        void* C, int64_t ldc,
                        int32_t op, const ge_options* opt, void* stream);

/*
 * Strided-batched GEMM (DESIGN.md R-C14): item b uses A + b*strideA, B + b*strideB,
 * C + b*strideC and bias + b*strideBias (strides in ELEMENTS; strideBias = 0 shares one
 * bias).  All items share M, N, K, layouts and options.  One persistent launch covers the
 * whole batch (the batch index is the slowest coordinate of the tile id).
 */
ge_status gemm_epilogue_batched(int64_t batch, int64_t M, int64_t N, int64_t K,
                                int32_t layoutA, int32_t layoutB,
                                const void* A, int64_t lda, int64_t strideA,
                                const void* B, int64_t ldb, int64_t strideB,
                                const void* bias, int64_t strideBias,
                                void* C, int64_t ldc, int64_t strideC,
                                int32_t op, const ge_options* opt, void* stream);

/*
 * Sum of matmuls, Listing 4: C = epilogue(prologue-free A.B + P.Q), with
 * A (M x K1), B (K1 x N), P (M x K2), Q (K2 x N); P takes A's layout and Q takes B's layout
 * (ldp/ldq their leading dimensions, 0 = packed).  Both products accumulate into the same fp32
 * Tensor Memory accumulator (one operand stream after the other), then bias/activation are
 * applied once.  K1 and K2 may differ.  opt->prologue must be NONE.
 * Alignment/aliasing rules of A/B apply to P/Q.  Asynchronous on `stream`.
 */
ge_status gemm2_epilogue(int64_t M, int64_t N, int64_t K1, int64_t K2,
                         int32_t layoutA, int32_t layoutB,
                         const void* A, int64_t lda, const void* B, int64_t ldb,
                         const void* P, int64_t ldp, const void* Q, int64_t ldq,
                         const void* bias, void* C, int64_t ldc,
                         int32_t op, const ge_options* opt, void* stream);

/*
 * Host-buffer variant (end-to-end path): same arguments as gemm_epilogue_batched but
 * A, B, bias, prologue_scale and C are HOST pointers (pinned memory gives full PCIe
 * bandwidth and copy/compute overlap; pageable works).  The call copies B (and bias, scale) to
 * a library-owned device workspace, then streams A and C in blocks (row blocks, or batch items)
 * on library copy/compute streams so each block's kernel and C read-back overlap the next
 * block's upload; it is ordered after prior work on `stream` and synchronizes before returning.
 * This entry point (only) allocates: the workspace (operands, C and a stream-K area) grows on
 * demand, is kept per device for reuse and is released by ge_release_workspace().  Operand
 * alignment rules apply to ld/strides only.
 */
ge_status gemm_epilogue_host(int64_t batch, int64_t M, int64_t N, int64_t K,
                             int32_t layoutA, int32_t layoutB,
                             const void* A, int64_t lda, int64_t strideA,
                             const void* B, int64_t ldb, int64_t strideB,
                             const void* bias, int64_t strideBias,
                             void* C, int64_t ldc, int64_t strideC,
                             int32_t op, const ge_options* opt, void* stream);

/* Frees the workspace of gemm_epilogue_host on the current device. */
ge_status ge_release_workspace(void);

/*
 * Argument validation only (no device access, no launch): returns what the batched entry
 * point would return for these arguments before touching the GPU.  Pointers are only
 * compared and alignment-checked, never dereferenced.
 */
ge_status ge_validate(int64_t batch, int64_t M, int64_t N, int64_t K,
                      int32_t layoutA, int32_t layoutB,
                      const void* A, int64_t lda, int64_t strideA,
                      const void* B, int64_t ldb, int64_t strideB,
                      const void* bias, int64_t strideBias,
                      void* C, int64_t ldc, int64_t strideC,
                      int32_t op, const ge_options* opt);

/* Static, never-NULL description of a status code. */
const char* ge_status_string(ge_status status);

/* Thread-local detail of the last non-OK status on this thread ("" if none). */
const char* ge_last_error_detail(void);

/*
 * Describes the configuration the heuristic picks for a shape (no device access): tile_m,
 * tile_n, cta_group, pipeline stages, the number of output tiles, how many of them run
 * stream-K (the last partial wave's tiles, whose K range is split evenly across all clusters;
 * partial sums are reduced in fixed order, so results stay run-to-run deterministic), the
 * split-K factor (split_k > 1: every tile is computed by a cluster of split_k CTAs, one K-slice
 * each, and the fp32 partials are reduce-scattered through distributed shared memory in fixed
 * order -- no workspace; only for few, long tiles) and the stream-K workspace bytes.  The plan is
 * the one a launch of the UNSWAPPED problem makes when given opt->workspace of at least
 * *workspace_bytes (without one, a launch re-plans with stream-K off); ge_plan_ex below also
 * reports multicast and the swap-AB decision (which depends on the op's bias).  The option checks
 * of the launch entry points apply (GE_ERR_INVALID_VALUE for invalid combinations).  Any output
 * pointer may be NULL.
 */
ge_status ge_plan(int64_t batch, int64_t M, int64_t N, int64_t K, int32_t layoutA, int32_t layoutB,
                  const ge_options* opt, int32_t num_sms,
                  int32_t* tile_m, int32_t* tile_n, int32_t* cta_group, int32_t* stages,
                  int64_t* num_tiles, int64_t* stream_k_tiles, int64_t* workspace_bytes, int32_t* split_k);

/* The launch configuration ge_plan_ex reports (see ge_plan); swap_ab = 1 when the launch computes
 * C^T = B^T A^T (tile_m / tile_n / num_tiles then describe the swapped problem: N x M). */
typedef struct {
    int32_t tile_m, tile_n, cta_group, stages;
    int64_t num_tiles, stream_k_tiles, workspace_bytes;
    int32_t split_k, multicast, swap_ab;
} ge_plan_info;

/* ge_plan with every planning decision a launch makes, including multicast clusters, half-row
 * pairs and swap-AB (which depends on the op's bias flag and opt->bias_mode / prologue). */
ge_status ge_plan_ex(int64_t batch, int64_t M, int64_t N, int64_t K, int32_t layoutA, int32_t layoutB,
                     int32_t op, const ge_options* opt, int32_t num_sms, ge_plan_info* out);

/* Number of fused kernels this library has launched in this process (for launch accounting). */
uint64_t ge_launch_count(void);

/* Tensor-map cache counters of this process: maps reused / encoded with
 * cuTensorMapEncodeTiled.  The cache memoises encodings by (address, dims, strides, box, swizzle,
 * type) and owns nothing.  Either pointer may be NULL. */
void ge_tensor_map_cache_stats(uint64_t* hits, uint64_t* misses);

/*
 * Diagnostics: when the process runs with GE_DEBUG_STATS=1 (diagnostics build), every launch
 * records per-CTA counters (30 x uint64 per CTA: total cycles, producer cycles blocked on free
 * stages, MMA cycles blocked on loaded stages, MMA cycles blocked on a drained accumulator,
 * epilogue cycles blocked on a full accumulator, epilogue phase timings, and %globaltimer
 * stamps (ns) of kernel entry, end of setup, end of the epilogue and exit, then the prologue
 * transform warps' cycles blocked on landed stages and spent rewriting them, and the MMA warp's
 * cycles issuing k-block MMAs and committing, the TMA producer's cycles issuing loads and its loop
 * total, and the split-K owner's TMEM-load / partial-add / math / store cycles).  Copies the last launch's counters of up to
 * max_ctas CTAs into out (synchronizing) and returns how many were copied (0 when disabled).
 */
int32_t ge_debug_read(uint64_t* out, int32_t max_ctas);

/* Library version string. */
const char* ge_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GEMM_EPILOGUE_H */
