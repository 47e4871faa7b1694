// TMA ingest probe: bytes per SM per ns that one CTA per SM pulls through cp.async.bulk.tensor into
// an S-stage smem ring (a consumer thread frees each stage as soon as it lands; no MMA), for box
// shapes {64 fp16 inner (128 B, SWIZZLE_128B), R rows}, L2-resident or HBM-streamed operands, one or
// two issuing warps.  Question it answers: is ~40 B/clk/SM (what the fused kernel's producer
// sustains) a TMA / L2->SM limit, and does the box size change it?
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_bw tma_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
    asm volatile(
        "{\n\t.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}" ::"r"(su32(b)),
        "r"(ph)
        : "memory");
}
__device__ __forceinline__ void bar_wait_mode(uint64_t* b, uint32_t ph, int mode) {
    if (mode == 1) {            // test_wait spin (never suspends)
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred P;\n\tmbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                         : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
    } else if (mode == 2) {     // try_wait with a long suspend-time hint (the fused kernel's form)
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, 0x989680;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                         : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
    } else {
        bar_wait(b, ph);
    }
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            su32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(su32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// nbox boxes of R rows per stage (stage = nbox * R * 128 B), S stages, `iters` stages per CTA.
// rows_span: the CTA's row window (L2-resident when small), cols: K extent (8192).
__global__ void __launch_bounds__(128, 1) k_tma(const __grid_constant__ CUtensorMap map, int R, int nbox, int S, int iters,
                                                int rows_span, int two_warps, unsigned long long* out, int wmode) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* ring = sm + ((1024 - (su32(sm) & 1023)) & 1023);
    __shared__ uint64_t full[16], empty[16];
    const int stage_bytes = nbox * R * 128;
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
        for (int s = 0; s < S; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned long long t0 = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int row0 = (blockIdx.x * R * nbox) % rows_span;
    if (two_warps >= 2) {
        // single thread: refill slot s as soon as its previous load landed (no consumer thread);
        // two_warps - 1 = slots waited for and refilled per batch
        const int G = two_warps - 1;
        if (threadIdx.x == 0) {
            for (int i = 0; i < iters; ++i) {
                const int s = i % S;
                if (i >= S && (i % G) == 0)
                    for (int g = 0; g < G; ++g) bar_wait_mode(&full[(i + g) % S], (((i + g) / S) - 1) & 1, wmode);
                bar_expect(&full[s], stage_bytes);
                const int kc = (i * 64) % 8192;
                const int rr = (row0 + (i / 128) * R * nbox) % rows_span;
                for (int j = 0; j < nbox; ++j) tma2d(ring + s * stage_bytes + j * R * 128, &map, &full[s], kc, rr + j * R);
            }
            for (int i = iters; i < iters + S; ++i) bar_wait_mode(&full[i % S], ((i / S) - 1) & 1, wmode);
            unsigned long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            out[blockIdx.x] = t1 - t0;
        }
    } else if ((warp == 0 || (two_warps && warp == 2)) && lane == 0) {
        for (int i = 0; i < iters; ++i) {
            const int s = i % S;
            if (i >= S) bar_wait_mode(&empty[s], ((i / S) - 1) & 1, wmode);
            if (warp == 0) bar_expect(&full[s], stage_bytes);
            const int kc = (i * 64) % 8192;
            const int rr = (row0 + (i / 128) * R * nbox) % rows_span;
            for (int j = 0; j < nbox; ++j) {
                if (two_warps && (j & 1) != (warp == 2 ? 1 : 0)) continue;
                tma2d(ring + s * stage_bytes + j * R * 128, &map, &full[s], kc, rr + j * R);
            }
        }
    } else if (warp == 1 && lane == 0) {
        for (int i = 0; i < iters; ++i) {
            const int s = i % S;
            bar_wait_mode(&full[s], (i / S) & 1, wmode);
            bar_arrive(&empty[s]);
        }
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        out[blockIdx.x] = t1 - t0;
    }
}

// Burst variant: one barrier per round expecting N boxes, N boxes issued back to back, then one wait
// (no per-stage ring protocol): pure TMA issue + transfer throughput with N boxes in flight.
__global__ void __launch_bounds__(128, 1) k_burst(const __grid_constant__ CUtensorMap map, int R, int N, int rounds,
                                                  int rows_span, unsigned long long* out, int multi) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* ring = sm + ((1024 - (su32(sm) & 1023)) & 1023);
    __shared__ uint64_t fulls[16];
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
        for (int j = 0; j < 16; ++j) bar_init(&fulls[j], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t0, t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        const int row0 = (blockIdx.x * R) % rows_span;
        if (multi == 4) {
            // lean refill: incremental coordinates and slot index (no divisions), per-slot barriers
            const int total = rounds * N;
            int j = 0, kc = 0, rr = row0, cnt = 0;
            uint32_t ph = 0;
            for (int i = 0; i < total; ++i) {
                if (i >= N) bar_wait(&fulls[j], ph ^ 1);
                bar_expect(&fulls[j], R * 128);
                tma2d(ring + j * R * 128, &map, &fulls[j], kc, rr);
                kc += 64;
                if (kc == 8192) { kc = 0; rr += R; if (rr >= rows_span) rr -= rows_span; }
                if (++j == N) { j = 0; ph ^= 1; }
                ++cnt;
            }
            for (int g = 0; g < N; ++g) { bar_wait(&fulls[j], ph ^ 1); if (++j == N) { j = 0; ph ^= 1; } }
        } else if (multi >= 2) {
            // pipelined refill with this kernel's code: N loads in flight, slot j refilled once its
            // previous load landed; multi == 3 waits for and refills the N slots as one group
            const int total = rounds * N;
            for (int i = 0; i < total; ++i) {
                const int j = i % N;
                if (i >= N && (multi == 2 || j == 0)) {
                    if (multi == 2) bar_wait(&fulls[j], ((i / N) - 1) & 1);
                    else for (int g = 0; g < N; ++g) bar_wait(&fulls[g], ((i / N) - 1) & 1);
                }
                bar_expect(&fulls[j], R * 128);
                tma2d(ring + j * R * 128, &map, &fulls[j], (i * 64) % 8192, (row0 + (i / 128) * R) % rows_span);
            }
            for (int j = 0; j < N; ++j) bar_wait(&fulls[j], ((total / N) - 1) & 1);
        }
        for (int r = 0; r < rounds && multi < 2; ++r) {
            if (multi) {
                for (int j = 0; j < N; ++j) {
                    bar_expect(&fulls[j], R * 128);
                    tma2d(ring + j * R * 128, &map, &fulls[j], ((r * N + j) * 64) % 8192, (row0 + ((r * N + j) / 128) * R) % rows_span);
                }
                for (int j = 0; j < N; ++j) bar_wait(&fulls[j], r & 1);
            } else {
                bar_expect(&fulls[0], N * R * 128);
                for (int j = 0; j < N; ++j)
                    tma2d(ring + j * R * 128, &map, &fulls[0], ((r * N + j) * 64) % 8192, (row0 + ((r * N + j) / 128) * R) % rows_span);
                bar_wait(&fulls[0], r & 1);
            }
        }
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        out[blockIdx.x] = t1 - t0;
    }
}

int main(int argc, char** argv) {
    typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fp, 12000, cudaEnableDefault, &q);
    Enc enc = reinterpret_cast<Enc>(fp);
    const int ROWS = 8192, COLS = 8192;
    void* buf;
    cudaMalloc(&buf, (size_t)ROWS * COLS * 2);
    cudaMemset(buf, 0, (size_t)ROWS * COLS * 2);
    unsigned long long* d_out;
    cudaMalloc(&d_out, 148 * 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Case { int R, nbox, span, two, grid; const char* name; int S = 0; int wmode = 0; };
    const Case cases[] = {
        {128, 1, 1024, 2, 148, "box 64x128, S=8, single thread refill", 8, 0},
        {128, 1, 1024, 3, 148, "box 64x128, S=8, refill in batches of 2", 8, 0},
        {128, 1, 1024, 5, 148, "box 64x128, S=8, refill in batches of 4", 8, 0},
        {128, 1, 1024, 9, 148, "box 64x128, S=8, refill in batches of 8", 8, 0},
        {128, 1, 1024, 5, 148, "box 64x128, S=12, refill in batches of 4", 12, 0},
        {128, 1, 1024, 0, 148, "box 64x128, S=8, test_wait spin", 8, 1},
        {128, 1, 1024, 0, 148, "box 64x128, S=8, try_wait hint 10ms", 8, 2},
        {128, 2, 1024, 0, 148, "2 boxes 64x128, S=6, test_wait spin", 6, 1},
        {256, 1, 1024, 0, 148, "box 64x256, S=6, test_wait spin", 6, 1},
        {128, 1, 1024, 0, 148, "box 64x128, S=1", 1},
        {128, 1, 1024, 0, 148, "box 64x128, S=2", 2},
        {128, 1, 1024, 0, 148, "box 64x128, S=4", 4},
        {128, 1, 1024, 0, 148, "box 64x128, S=8", 8},
        {128, 1, 1024, 0, 148, "box 64x128, S=12", 12},
        {128, 1, 1024, 0, 148, "box 64x128 (16 KB), L2-resident"},
        {64, 1, 1024, 0, 148, "box 64x64 (8 KB), L2-resident"},
        {256, 1, 1024, 0, 148, "box 64x256 (32 KB), L2-resident"},
        {128, 2, 1024, 0, 148, "2 boxes 64x128 per stage (32 KB), L2-resident"},
        {128, 2, 1024, 1, 148, "2 boxes 64x128, two issuing warps, L2-resident"},
        {64, 4, 1024, 0, 148, "4 boxes 64x64 per stage (32 KB), L2-resident"},
        {32, 4, 1024, 0, 148, "4 boxes 64x32 per stage (16 KB), L2-resident"},
        {128, 1, 8192, 0, 148, "box 64x128, streamed from HBM (128 MB)"},
        {256, 1, 8192, 0, 148, "box 64x256, streamed from HBM"},
        {128, 1, 1024, 0, 16, "box 64x128, 16 CTAs, L2-resident"},
        {256, 1, 1024, 0, 16, "box 64x256, 16 CTAs, L2-resident"},
    };
    for (const Case& c : cases) {
        CUtensorMap m;
        cuuint64_t dims[2] = {(cuuint64_t)COLS, (cuuint64_t)ROWS};
        cuuint64_t strides[1] = {(cuuint64_t)COLS * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)c.R};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
        const int stage = c.nbox * c.R * 128;
        const int S = c.S ? c.S : std::min(8, (192 * 1024) / stage);
        const int iters = 2000;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int w = 0; w < 2; ++w) k_tma<<<c.grid, 128, S * stage + 1024>>>(m, c.R, c.nbox, S, 50, c.span, c.two, d_out, c.wmode);
        cudaEventRecord(e0);
        k_tma<<<c.grid, 128, S * stage + 1024>>>(m, c.R, c.nbox, S, iters, c.span, c.two, d_out, c.wmode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long h[148];
        cudaMemcpy(h, d_out, 148 * 8, cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < c.grid; ++i) mx = h[i] > mx ? h[i] : mx;
        const double bytes = (double)iters * stage;
        printf("%-52s S=%d  per SM %6.1f B/ns  chip %7.1f GB/s (kernel %.3f ms)  err=%s\n", c.name, S, bytes / mx,
               bytes * c.grid / (ms * 1e6), ms, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFuncSetAttribute(k_burst, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int bursts[][3] = {{128, 8, 1}, {128, 8, 2}, {128, 8, 4}, {128, 4, 4}, {128, 12, 4}, {64, 8, 4}, {256, 6, 4}};
    for (auto& bc : bursts) {
        const int R = bc[0], N = bc[1], multi = bc[2];
        CUtensorMap m;
        cuuint64_t dims[2] = {(cuuint64_t)COLS, (cuuint64_t)ROWS};
        cuuint64_t strides[1] = {(cuuint64_t)COLS * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)R};
        cuuint32_t es[2] = {1, 1};
        enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int rounds = 400;
        const int smem = N * R * 128 + 1024;
        k_burst<<<148, 128, smem>>>(m, R, N, 20, 1024, d_out, multi);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_burst<<<148, 128, smem>>>(m, R, N, rounds, 1024, d_out, multi);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long h[148];
        cudaMemcpy(h, d_out, 148 * 8, cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        const double bytes = (double)rounds * N * R * 128;
        printf("burst%s: %2d boxes of 64x%-3d per round  %7.1f ns/round  per SM %6.1f B/ns  chip %7.1f GB/s  err=%s\n", multi == 4 ? "(lean refill)      " : multi == 3 ? "(refill by group)  " : multi == 2 ? "(refill per slot)  " : multi ? "(1 barrier per box)" : "(1 barrier)       ", N, R,
               mx / rounds, bytes / mx, bytes * 148 / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
