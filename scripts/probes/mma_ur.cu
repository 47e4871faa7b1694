// Dev probe: can the MMA descriptors live in uniform registers?  Descriptors passed as kernel
// parameters (constant bank -> LDCU into UR) and used with compile-time stage/k indices, vs the
// production form (computed from the smem base in registers).  usage: mma_ur mode
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include "../../paper_2006_12645_b200/csrc/ge_ptx.cuh"
using namespace ge;

struct Descs { uint64_t a[4], b[4]; };

template <int N>
__global__ void probe(int reps, int mode, const __grid_constant__ Descs dd, unsigned long long* out) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t bar_end, bars[8], never;
    __shared__ volatile int done;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar_end, 1);
        for (int i = 0; i < 8; ++i) ptx::mbar_init(&bars[i], 1);
        ptx::mbar_init(&never, 1);
        done = 0;
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc<1>(&slot, 256);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    constexpr uint32_t IDESC = ptx::make_idesc_f16(128, N, false, false);
    long long t0 = 0;
    if (warp == 1) {
        const uint32_t a = (ptx::smem_u32(smem_raw) + 1023) & ~1023u, b = a + 16384 * 4;
        const uint64_t ad0 = ptx::make_sw128_desc(a, 0, 1024), bd0 = ptx::make_sw128_desc(b, 0, 1024);
        for (int r = -2; r < reps; ++r) {
            if (r == 0) t0 = clock64();
#pragma unroll
            for (int st = 0; st < 4; ++st) {
                if (mode != 1) ptx::mma_kblock<1, 2, 2>(tmem, ad0 + st * 1024, bd0 + st * 1024, IDESC, 1);
                else ptx::mma_kblock<1, 2, 2>(tmem, dd.a[st], dd.b[st], IDESC, 1);
                if (st & 1) ptx::mma_commit_elect<1>(&bars[st]);
            }
        }
        ptx::mma_commit_elect<1>(&bar_end);
        ptx::mbar_wait(&bar_end, 0);
        if (threadIdx.x == 32) { out[0] = clock64() - t0; done = 1; }
    } else if (mode >= 2 && (warp == 2 || (mode == 3 && warp == 3))) {
        // pollers: try_wait on a barrier that never completes (like idle producer / epilogue waiters)
        if ((threadIdx.x & 31) == 0 || mode == 3)
            while (!done) { ptx::mbar_try_wait(ptx::smem_u32(&never), 0); }
    }
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<1>(tmem, 256);
}

int main(int argc, char** argv) {
    const int mode = atoi(argv[1]);
    unsigned long long* d; cudaMalloc(&d, 8);
    const int smem = 16384 * 8 + 2048;
    cudaFuncSetAttribute(probe<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    // dynamic smem starts at a fixed shared-window offset; the kernel aligns it to 1 KB the same way
    Descs dd;
    // the shared address is only known on the device: mode 1 uses offsets from address 0x400-aligned
    // base 0x400 (reserved system smem precedes dynamic smem on sm_90+); correctness is irrelevant
    // for an issue-rate probe as long as the addresses stay inside the allocation
    for (int st = 0; st < 4; ++st) {
        auto mk = [](uint32_t addr) { return (uint64_t)((addr >> 4) & 0x3FFF) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61); };
        dd.a[st] = mk(0x400 + st * 16384); dd.b[st] = mk(0x400 + 65536 + st * 16384);
    }
    const int reps = 200;
    probe<64><<<1, 128, smem>>>(reps, mode, dd, d);
    unsigned long long h = 0;
    cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("N=64 mode=%d: %s %.1f cycles/MMA, %.1f cycles/k-block\n", mode, cudaGetErrorString(e), double(h) / (reps * 16), double(h) / (reps * 4));
    return 0;
}
