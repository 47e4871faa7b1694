/*
 * ge_oracle.c -- CPU oracle for the fused GEMM + bias + ReLU hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2006_12645_b200/) never links, imports or calls it.
 * It shares no code, header or constant with the CUDA path.
 *
 * What it computes: the plain definition of the paper's fused idioms, in fp64,
 * on exactly-widened fp16 inputs, with no tiling, fusion or reordering:
 *
 *   Listing 1 (Sec. III "Problem Statement"):
 *       S1: C[i,j] = sum_k A[i,k] * B[k,j]
 *       S2: E[i,j] = relu_add(C[i,j], bias[i,j])   (ReLU at the root)
 *   generalised to the paper's pointwise op set: add or subtract the
 *   bias, then ReLU, Sigmoid or Tanh at the root.
 *   Listing 5 (Sec. VII-C "Pointwise Operations in Prologue"):
 *       C[i,j] = sum_k relu(A[i,k]) * B[k,j]
 *   plus the SCALE_K prologue reading of DESIGN.md (R-C12): a'(i,k) = s_k * a(i,k), and the
 *   full-tile Hadamard prologue (DESIGN.md R-C18; "the compound operation in statement S1 could have
 *   multiple input dataspaces"): a'(i,k) = s(i,k) * a(i,k), S an M x K fp16
 *   dataspace stored in A's layout.
 *
 *   a'(i,k)  = a(i,k) | s_k * a(i,k) | max(a(i,k), 0) | s(i,k) * a(i,k)
 *                                                       (prologue NONE|SCALE_K|RELU|HADAMARD)
 *   pre(i,j) = sum_{k<K} a'(i,k) * b(k,j) +- beta(i,j)        (beta = 0|bias[j]|bias[i]|bias[i,j])
 *   out(i,j) = act(pre): identity | relu (pre > 0 ? pre : +0) | sigmoid 1/(1+e^-pre) | tanh(pre)
 *   mag(i,j) = sum_{k<K} |a'(i,k) * b(k,j)|                    (scale of the rounding error)
 *
 * The sum runs k = 0, 1, ..., K-1 in that order (Listing 1's loop order).
 * Inputs are read through index formulas restated here, written independently
 * of the CUDA path:
 *   A row-major: a(i,k) = A[i*lda + k]      A col-major: a(i,k) = A[k*lda + i]
 *   B row-major: b(k,j) = B[k*ldb + j]      B col-major: b(k,j) = B[j*ldb + k]
 *
 * Parity pins (tests/test_oracle_pins.py): fp16 codec vs numpy over all 65536
 * patterns; hand-computed golden cases (tests/golden/); exact rational brute
 * force on tiny shapes; numpy fp64 matmul cross-check; closed forms (identity,
 * zeros, all-ones, diagonal, rank-1, K=0); layout invariance; ReLU invariant.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- fp16 codec
 * IEEE 754 binary16: 1 sign, 5 exponent (bias 15), 10 fraction bits.
 * Decoding is exact into fp64.  Encoding is round-to-nearest-even with
 * overflow to +-inf and gradual underflow (subnormals kept).
 */
double oracle_f16_to_f64(uint16_t h) {
    int sign = (h >> 15) & 1;
    int e = (h >> 10) & 0x1f;
    int f = h & 0x3ff;
    double v;
    if (e == 0) {
        v = ldexp((double)f, -24);                 /* subnormal: f * 2^-24 */
    } else if (e == 31) {
        v = f ? NAN : INFINITY;
    } else {
        v = ldexp((double)(1024 + f), e - 25);     /* (1 + f/1024) * 2^(e-15) */
    }
    return sign ? -v : v;
}

uint16_t oracle_f64_to_f16_rne(double x) {
    uint16_t sign = signbit(x) ? 0x8000 : 0;
    double a = fabs(x);
    if (isnan(x)) return 0x7e00;
    if (isinf(a)) return sign | 0x7c00;
    if (a == 0.0) return sign;
    /* Values >= 65520 (halfway between 65504 and 2^16) round to inf. */
    if (a >= 65520.0) return sign | 0x7c00;
    int e;
    (void)frexp(a, &e);                 /* a = m * 2^e, m in [0.5, 1) */
    int exp16 = e - 1;                  /* a = 1.xxx * 2^exp16 */
    double quantum;                     /* spacing of fp16 values near a */
    if (exp16 < -14) quantum = ldexp(1.0, -24);          /* subnormal range */
    else quantum = ldexp(1.0, exp16 - 10);
    double q = a / quantum;             /* exact: quantum is a power of two */
    double fl = floor(q);
    double rem = q - fl;
    double n;
    if (rem > 0.5) n = fl + 1.0;
    else if (rem < 0.5) n = fl;
    else n = (fmod(fl, 2.0) == 0.0) ? fl : fl + 1.0;     /* tie -> even */
    double r = n * quantum;             /* the rounded magnitude, exact */
    if (r >= 65520.0) return sign | 0x7c00;
    /* Re-encode r (exactly representable in fp16). */
    if (r < ldexp(1.0, -14)) {
        return sign | (uint16_t)(r / ldexp(1.0, -24));   /* subnormal (or 2^-14 exactly handled below) */
    }
    int er;
    double mr = frexp(r, &er);          /* r = mr * 2^er */
    int biased = (er - 1) + 15;
    uint16_t frac = (uint16_t)((mr * 2.0 - 1.0) * 1024.0);
    return sign | (uint16_t)(biased << 10) | frac;
}

/* ------------------------------------------------------------ definitions */
enum { OR_ROW = 0, OR_COL = 1 };
enum { OR_BIAS_NONE = -1, OR_BIAS_ROW = 0, OR_BIAS_COL = 1, OR_BIAS_FULL = 2 };
enum { OR_PRO_NONE = 0, OR_PRO_SCALE_K = 1, OR_PRO_RELU = 2, OR_PRO_HADAMARD = 3 };

typedef struct {
    int64_t M, N, K;
    int layoutA, layoutB;
    const uint16_t *A; int64_t lda;
    const uint16_t *B; int64_t ldb;
    const uint16_t *bias; int bias_mode; int64_t ldbias;
    int act;                /* 0 identity, 1 relu, 2 sigmoid, 3 tanh */
    int bias_sign;          /* +1 add, -1 subtract */
    int prologue; const float *scale;
    const uint16_t *S; int64_t lds;     /* HADAMARD: s(i,k), A's layout */
    int literal_round;      /* DESIGN.md R-C3 paper-literal variant: relu(f16(f16(acc)+bias)) */
    /* the evaluated rows I and columns J (the output is out[r*nJ + c] for i=I[r], j=J[c]) */
    const int64_t *I; int64_t nI;
    const int64_t *J; int64_t nJ;
    /* logical operands for those rows/columns, widened once: a data-layout step,
     * no arithmetic is reordered */
    double *ap;             /* a'(I[r],k) at ap[r*K + k] */
    double *bt;             /* b(k,J[c])  at bt[c*K + k] */
    double *out, *mag;
    int nthreads, tid;
} job_t;

static int64_t row_of(const job_t *T, int64_t r) { return T->I ? T->I[r] : r; }
static int64_t col_of(const job_t *T, int64_t c) { return T->J ? T->J[c] : c; }

static double a_elem(const job_t *T, int64_t i, int64_t k) {
    uint16_t h = (T->layoutA == OR_ROW) ? T->A[i * T->lda + k] : T->A[k * T->lda + i];
    return oracle_f16_to_f64(h);
}
static double b_elem(const job_t *T, int64_t k, int64_t j) {
    uint16_t h = (T->layoutB == OR_ROW) ? T->B[k * T->ldb + j] : T->B[j * T->ldb + k];
    return oracle_f16_to_f64(h);
}
/* s(i,k) of the Hadamard prologue, read through A's layout formula */
static double s_elem(const job_t *T, int64_t i, int64_t k) {
    uint16_t h = (T->layoutA == OR_ROW) ? T->S[i * T->lds + k] : T->S[k * T->lds + i];
    return oracle_f16_to_f64(h);
}
/* prologue a'(i,k): PAPER.md:1201-1206 (ReLU), DESIGN.md R-C12 (SCALE_K) and R-C18 (HADAMARD,
 * PAPER.md:1222-1224) */
static double a_prime(const job_t *T, int64_t i, int64_t k) {
    double a = a_elem(T, i, k);
    if (T->prologue == OR_PRO_SCALE_K) return (double)T->scale[k] * a;
    if (T->prologue == OR_PRO_RELU) return a > 0.0 ? a : 0.0;
    if (T->prologue == OR_PRO_HADAMARD) return s_elem(T, i, k) * a;
    return a;
}
/* beta(i,j): DESIGN.md R-C2 (ROW default, COL, FULL = PAPER.md:363 literal) */
static double beta(const job_t *T, int64_t i, int64_t j) {
    switch (T->bias_mode) {
    case OR_BIAS_ROW: return oracle_f16_to_f64(T->bias[j]);
    case OR_BIAS_COL: return oracle_f16_to_f64(T->bias[i]);
    case OR_BIAS_FULL: return oracle_f16_to_f64(T->bias[i * T->ldbias + j]);
    default: return 0.0;
    }
}

/* One output element, Listing 1's S1 then S2. */
static void element(const job_t *T, int64_t r, int64_t c, double *res, double *m) {
    const double *ar = T->ap + r * T->K;
    const double *bc = T->bt + c * T->K;
    double acc = 0.0, mg = 0.0;
    for (int64_t k = 0; k < T->K; ++k) {           /* S1: C[i,j] = mul_acc(C[i,j], A[i,k], B[k,j]) */
        double p = ar[k] * bc[k];
        acc += p;
        mg += fabs(p);
    }
    int64_t i = row_of(T, r), j = col_of(T, c);
    double pre;
    if (T->literal_round) {
        /* R-C3 literal reading: accumulator converted to fp16 before the pointwise op
         * (PAPER.md:1109-1112), relu_add on fp16 fragments. */
        double c16 = oracle_f16_to_f64(oracle_f64_to_f16_rne(acc));
        pre = oracle_f16_to_f64(oracle_f64_to_f16_rne(c16 + T->bias_sign * beta(T, i, j)));
    } else {
        pre = acc + T->bias_sign * beta(T, i, j);   /* S2: add (or subtract) */
    }
    double o;                                       /* S2: activation at the root */
    switch (T->act) {
    case 1: o = pre > 0.0 ? pre : 0.0; break;
    case 2: o = 1.0 / (1.0 + exp(-pre)); break;
    case 3: o = tanh(pre); break;
    default: o = pre;
    }
    *res = o;
    *m = mg;
}

static void *worker(void *arg) {
    job_t *T = (job_t *)arg;
    for (int64_t r = T->tid; r < T->nI; r += T->nthreads)
        for (int64_t c = 0; c < T->nJ; ++c)
            element(T, r, c, &T->out[r * T->nJ + c], &T->mag[r * T->nJ + c]);
    return NULL;
}

static void *widen_worker(void *arg) {
    job_t *T = (job_t *)arg;
    for (int64_t r = T->tid; r < T->nI; r += T->nthreads)
        for (int64_t k = 0; k < T->K; ++k) T->ap[r * T->K + k] = a_prime(T, row_of(T, r), k);
    for (int64_t c = T->tid; c < T->nJ; c += T->nthreads)
        for (int64_t k = 0; k < T->K; ++k) T->bt[c * T->K + k] = b_elem(T, k, col_of(T, c));
    return NULL;
}

static int run_threads(job_t *base, void *(*fn)(void *)) {
    int nt = base->nthreads < 1 ? 1 : base->nthreads;
    if (nt > 256) nt = 256;
    job_t jobs[256];
    pthread_t th[256];
    for (int t = 0; t < nt; ++t) {
        jobs[t] = *base;
        jobs[t].tid = t;
        jobs[t].nthreads = nt;
    }
    for (int t = 1; t < nt; ++t)
        if (pthread_create(&th[t], NULL, fn, &jobs[t]) != 0) return -2;
    fn(&jobs[0]);
    for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
    return 0;
}

/*
 * Evaluate out/mag (fp64, unrounded) on the cross product of rows I x columns J.
 * I == NULL means all M rows (nI ignored), J == NULL all N columns.
 * out[r*nJ + c] is element (I[r], J[c]).  Returns 0, or <0 on bad arguments.
 * bias_mode: -1 none, 0 ROW bias[j], 1 COL bias[i], 2 FULL bias[i*ldbias+j]; bias_sign +1/-1.
 * act: 0 identity, 1 relu, 2 sigmoid, 3 tanh.  prologue: 0 none, 1 SCALE_K (scale[k], fp32), 2 RELU,
 * 3 HADAMARD (S: fp16 M x K in A's layout with leading dimension lds).
 */
int oracle_gemm_epilogue(int64_t M, int64_t N, int64_t K, int layoutA, int layoutB,
                         const uint16_t *A, int64_t lda, const uint16_t *B, int64_t ldb,
                         const uint16_t *bias, int bias_mode, int bias_sign, int64_t ldbias, int act,
                         int prologue, const float *scale, const uint16_t *S, int64_t lds, int literal_round,
                         const int64_t *I, int64_t nI, const int64_t *J, int64_t nJ,
                         double *out, double *mag, int nthreads) {
    if (M < 0 || N < 0 || K < 0) return -1;
    if (act < 0 || act > 3 || (bias_sign != 1 && bias_sign != -1)) return -1;
    if (bias_mode != OR_BIAS_NONE && !bias) return -1;
    if (prologue == OR_PRO_SCALE_K && !scale) return -1;
    if (prologue == OR_PRO_HADAMARD && K > 0 && !S) return -1;
    if (prologue < OR_PRO_NONE || prologue > OR_PRO_HADAMARD) return -1;
    job_t T;
    memset(&T, 0, sizeof T);
    T.M = M; T.N = N; T.K = K;
    T.layoutA = layoutA; T.layoutB = layoutB;
    T.A = A; T.lda = lda; T.B = B; T.ldb = ldb;
    T.bias = bias; T.bias_mode = bias_mode; T.ldbias = ldbias;
    T.act = act; T.bias_sign = bias_sign; T.prologue = prologue; T.scale = scale;
    T.S = S; T.lds = lds;
    T.literal_round = literal_round;
    T.I = I; T.nI = I ? nI : M;
    T.J = J; T.nJ = J ? nJ : N;
    for (int64_t r = 0; I && r < nI; ++r) if (I[r] < 0 || I[r] >= M) return -1;
    for (int64_t c = 0; J && c < nJ; ++c) if (J[c] < 0 || J[c] >= N) return -1;
    T.out = out; T.mag = mag;
    T.nthreads = nthreads;
    size_t na = (size_t)(T.nI * K), nb = (size_t)(T.nJ * K);
    T.ap = (double *)malloc((na ? na : 1) * sizeof(double));
    T.bt = (double *)malloc((nb ? nb : 1) * sizeof(double));
    if (!T.ap || !T.bt) { free(T.ap); free(T.bt); return -3; }
    int rc = run_threads(&T, widen_worker);
    if (rc == 0) rc = run_threads(&T, worker);
    free(T.ap);
    free(T.bt);
    return rc;
}

/* Array forms of the codec (one ctypes call instead of one per element). */
void oracle_f16_decode_array(const uint16_t *h, double *out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_f16_to_f64(h[i]);
}
void oracle_f16_encode_array(const double *x, uint16_t *out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_f64_to_f16_rne(x[i]);
}

/*
 * Sum of matmuls, Listing 4 (Sec. VII-B "Matmuls with Pointwise Epilogue"):
 *     S1: C[i,j] = sum_k A[i,k] B[k,j]      (k < K1)
 *     S2: R[i,j] = sum_k P[i,k] Q[k,j]      (k < K2)
 *     S3: Z[i,j] = add(C[i,j], R[i,j])      then the same bias / activation as above
 * K1 and K2 may differ (the outputs share the shape).  P and Q use the
 * layouts of A and B.  Evaluated by two plain oracle passes (no bias / activation) and the S3
 * add, then S2-of-Listing-1 bias and activation; mag = sum|ab| + sum|pq|.
 */
int oracle_gemm2_epilogue(int64_t M, int64_t N, int64_t K1, int64_t K2, int layoutA, int layoutB,
                          const uint16_t *A, int64_t lda, const uint16_t *B, int64_t ldb,
                          const uint16_t *P, int64_t ldp, const uint16_t *Q, int64_t ldq,
                          const uint16_t *bias, int bias_mode, int bias_sign, int64_t ldbias, int act,
                          const int64_t *I, int64_t nI, const int64_t *J, int64_t nJ,
                          double *out, double *mag, int nthreads) {
    const int64_t nr = I ? nI : M, nc = J ? nJ : N;
    const size_t n = (size_t)(nr * nc);
    double *c = (double *)malloc((n ? n : 1) * sizeof(double));
    double *cm = (double *)malloc((n ? n : 1) * sizeof(double));
    double *r = (double *)malloc((n ? n : 1) * sizeof(double));
    double *rm = (double *)malloc((n ? n : 1) * sizeof(double));
    int rc = (c && cm && r && rm) ? 0 : -3;
    if (rc == 0)
        rc = oracle_gemm_epilogue(M, N, K1, layoutA, layoutB, A, lda, B, ldb, NULL, OR_BIAS_NONE, 1, 0, 0,
                                  OR_PRO_NONE, NULL, NULL, 0, 0, I, nI, J, nJ, c, cm, nthreads);
    if (rc == 0)
        rc = oracle_gemm_epilogue(M, N, K2, layoutA, layoutB, P, ldp, Q, ldq, NULL, OR_BIAS_NONE, 1, 0, 0,
                                  OR_PRO_NONE, NULL, NULL, 0, 0, I, nI, J, nJ, r, rm, nthreads);
    if (rc == 0) {
        job_t T;
        memset(&T, 0, sizeof T);
        T.bias = bias; T.bias_mode = bias ? bias_mode : OR_BIAS_NONE; T.ldbias = ldbias;
        for (int64_t a = 0; a < nr; ++a)
            for (int64_t b = 0; b < nc; ++b) {
                const size_t x = (size_t)(a * nc + b);
                const int64_t i = I ? I[a] : a, j = J ? J[b] : b;
                const double pre = (c[x] + r[x]) + bias_sign * beta(&T, i, j);       /* S3, then bias */
                double o;
                switch (act) {
                case 1: o = pre > 0.0 ? pre : 0.0; break;
                case 2: o = 1.0 / (1.0 + exp(-pre)); break;
                case 3: o = tanh(pre); break;
                default: o = pre;
                }
                out[x] = o;
                mag[x] = cm[x] + rm[x];
            }
    }
    free(c); free(cm); free(r); free(rm);
    return rc;
}
