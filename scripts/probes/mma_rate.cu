// Dev probe: back-to-back tcgen05.mma (cta_group::1, kind::f16, M=128, K=16) issue rate from one
// CTA, operands in smem (contents irrelevant).  usage: mma_rate N mode per_commit
//   mode 0: whole warp, elect.sync inside each MMA's asm (production form)
//   mode 1: one lane (threadIdx 32) issues, descriptors recomputed per MMA
//   mode 2: one lane, descriptors precomputed outside the timed loop
//   mode 3: whole warp, elect once per k-block group (if elect) { 4 MMAs }
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_rate mma_rate.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include "../../paper_2006_12645_b200/csrc/ge_ptx.cuh"
using namespace ge;

__device__ __forceinline__ bool elect_one() {
    uint32_t e;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(e));
    return e != 0;
}

template <int N, int PC>
__global__ void probe(int reps, int per_commit, int mode, unsigned long long* out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t bar_end, bars[8];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar_end, 1);
        for (int i = 0; i < 8; ++i) ptx::mbar_init(&bars[i], 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc<1>(&slot, 256);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    constexpr uint32_t IDESC = ptx::make_idesc_f16(128, N, false, false);
    const uint32_t a = ptx::smem_u32(smem), b = a + 16384 * 4;
    long long t0 = 0;
    if (warp == 1) {
        if (mode >= 6) {
            // k-block loop like the kernel: [wait on a completed barrier] [fence] 4 MMAs (one asm) + commit
            const uint64_t ad0 = ptx::make_sw128_desc(a, 0, 1024), bd0 = ptx::make_sw128_desc(b, 0, 1024);
            if (threadIdx.x == 32) ptx::mbar_arrive(&bars[7]);            // completes phase 0 of bars[7]
            __syncwarp();
            for (int r = -2; r < reps; ++r) {
                if (r == 0) t0 = clock64();
                for (int i = 0; i < per_commit; i += 4) {
                    const int st = (i >> 2) & 3;
                    if (mode == 9 || mode == 10) {
                        // early test of the next stage, consumed after this stage's MMAs
                        const bool ok = ptx::mbar_test(&bars[7], 0);
                        ptx::tc_fence_after();
                        ptx::mma_kblock<1, 2, 2>(tmem, ad0 + st * 1024, bd0 + st * 1024, IDESC, 1);
                        if (mode == 9 || (st & 1)) ptx::mma_commit_elect<1>(&bars[st]);
                        if (!ok) ptx::mbar_wait(&bars[7], 0);
                        continue;
                    }
                    if (mode >= 7) ptx::mbar_wait(&bars[7], 0);
                    if (mode >= 8) ptx::tc_fence_after();
                    ptx::mma_kblock<1, 2, 2>(tmem, ad0 + st * 1024, bd0 + st * 1024, IDESC, 1);
                    ptx::mma_commit_elect<1>(&bars[st]);
                }
            }
            ptx::mma_commit_elect<1>(&bar_end);
        } else if (mode == 0 || mode == 3) {
            for (int r = -2; r < reps; ++r) {
                if (r == 0) t0 = clock64();
                for (int i = 0; i < per_commit; i += 4) {
                    const int st = (i >> 2) & 3;
                    if (mode == 0) {
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            ptx::mma_f16_elect<1>(tmem, ptx::make_sw128_desc(a + st * 16384 + k * 32, 0, 1024),
                                                  ptx::make_sw128_desc(b + st * 16384 + k * 32, 0, 1024), IDESC, 1);
                    } else if (elect_one()) {
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            ptx::mma_f16<1>(tmem, ptx::make_sw128_desc(a + st * 16384 + k * 32, 0, 1024),
                                            ptx::make_sw128_desc(b + st * 16384 + k * 32, 0, 1024), IDESC, 1);
                    }
                    __syncwarp();
                }
            }
            ptx::mma_commit_elect<1>(&bar_end);
        } else if (threadIdx.x == 32) {
            uint64_t ad[16], bd[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                ad[i] = ptx::make_sw128_desc(a + (i >> 2) * 16384 + (i & 3) * 32, 0, 1024);
                bd[i] = ptx::make_sw128_desc(b + (i >> 2) * 16384 + (i & 3) * 32, 0, 1024);
            }
            for (int r = -2; r < reps; ++r) {
                if (r == 0) t0 = clock64();
                if (mode == 1) {
                    for (int i = 0; i < per_commit; ++i)
                        ptx::mma_f16<1>(tmem, ptx::make_sw128_desc(a + ((i >> 2) & 3) * 16384 + (i & 3) * 32, 0, 1024),
                                        ptx::make_sw128_desc(b + ((i >> 2) & 3) * 16384 + (i & 3) * 32, 0, 1024), IDESC, 1);
                } else if (mode == 2) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) ptx::mma_f16<1>(tmem, ad[i], bd[i], IDESC, 1);
                } else {
                    // mode 4: commit (to a rotating barrier) after every per_commit MMAs
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        ptx::mma_f16<1>(tmem, ad[i], bd[i], IDESC, 1);
                        if ((i + 1) % PC == 0) {
                            if (mode == 4) ptx::mma_commit<1>(&bars[(i / PC) & 7]);
                            else ptx::mma_commit<1>(&bars[0]);
                        }
                    }
                }
            }
            ptx::mma_commit<1>(&bar_end);
        }
        ptx::mbar_wait(&bar_end, 0);
        if (threadIdx.x == 32) out[0] = clock64() - t0;
    }
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<1>(tmem, 256);
}

template <int N, int PC>
void run(int mode, int per_commit) {
    unsigned long long* d; cudaMalloc(&d, 8);
    const int smem = 16384 * 8 + 1024 + 65536;
    cudaFuncSetAttribute(probe<N, PC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int reps = 200;
    probe<N, PC><<<1, 128, smem>>>(reps, per_commit, mode, d);
    unsigned long long h = 0;
    cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const int pcp = per_commit;
    if (mode >= 2) per_commit = 16;
    printf("N=%3d mode=%d (commit every %2d) per_loop=%2d: %s %.1f cycles/MMA (floor %d)\n", N, mode, pcp, per_commit,
           cudaGetErrorString(e), double(h) / (reps * per_commit), N / 2);
    cudaFree(d);
}

int main(int argc, char** argv) {
    const int n = atoi(argv[1]), mode = atoi(argv[2]), pc = atoi(argv[3]);
#define R(NN) if (n == NN) { if (pc == 1) run<NN, 1>(mode, pc); if (pc == 4) run<NN, 4>(mode, pc); if (pc == 16) run<NN, 16>(mode, pc); }
    R(64) R(128) R(256)
    return 0;
}
