// Launch-cost probe: per-launch time of a near-empty kernel in a CUDA graph of R back-to-back
// launches, varying what our fused kernel's launch carries: dynamic smem size, cluster dims, PDL,
// block size, TMEM allocation.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o
// launch_cost launch_cost.cu ; run: ./launch_cost
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_empty(int* out) {
    if (out && threadIdx.x == 0 && blockIdx.x == 100000) out[0] = 1;
}

template <int CG>
__global__ void k_tmem(int* out) {
    __shared__ uint32_t slot;
    extern __shared__ uint8_t dyn[];
    if (threadIdx.x / 32 == 2) {
        uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&slot));
        if (CG == 1) asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(a));
        else asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(a));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if (CG == 2) {
        asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    if (out && threadIdx.x == 0 && blockIdx.x == 100000) out[0] = dyn[0];
    __syncthreads();
    if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
    if (threadIdx.x / 32 == 2) {
        if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
        else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(slot));
    }
}

static float run(void (*kern)(int*), int grid, int block, int smem, int cluster, bool pdl, int R = 40) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaStream_t st;
    cudaStreamCreate(&st);
    auto launch = [&]() {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(block);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        int n = 0;
        at[n].id = cudaLaunchAttributeClusterDimension;
        at[n].val.clusterDim.x = cluster;
        at[n].val.clusterDim.y = 1;
        at[n].val.clusterDim.z = 1;
        ++n;
        if (pdl) {
            at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[n].val.programmaticStreamSerializationAllowed = 1;
            ++n;
        }
        cfg.attrs = at;
        cfg.numAttrs = n;
        cudaLaunchKernelEx(&cfg, kern, (int*)nullptr);
    };
    launch();
    cudaStreamSynchronize(st);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < R; ++i) launch();
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    for (int i = 0; i < 5; ++i) cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("  error %s\n", cudaGetErrorString(e));
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(st);
    return ms * 1000.f / (5 * R);
}

int main() {
    const int big = 227 * 1024 - 1024;
    struct C { const char* name; void (*k)(int*); int grid, block, smem, cluster; bool pdl; };
    C cs[] = {
        {"empty 8x128 smem0", k_empty, 8, 128, 0, 1, false},
        {"empty 8x384 smem0", k_empty, 8, 384, 0, 1, false},
        {"empty 8x384 smem226K", k_empty, 8, 384, big, 1, false},
        {"empty 8x384 smem226K pdl", k_empty, 8, 384, big, 1, true},
        {"empty 8x384 smem226K cl2", k_empty, 8, 384, big, 2, false},
        {"empty 148x384 smem226K cl2 pdl", k_empty, 148, 384, big, 2, true},
        {"tmem1 8x384 smem226K", k_tmem<1>, 8, 384, big, 1, false},
        {"tmem1 8x384 smem226K pdl", k_tmem<1>, 8, 384, big, 1, true},
        {"tmem2 8x384 smem226K cl2", k_tmem<2>, 8, 384, big, 2, false},
        {"tmem2 8x384 smem226K cl2 pdl", k_tmem<2>, 8, 384, big, 2, true},
        {"tmem2 148x384 smem226K cl2 pdl", k_tmem<2>, 148, 384, big, 2, true},
        {"tmem1 148x384 smem100K pdl", k_tmem<1>, 148, 384, 100 * 1024, 1, true},
    };
    for (auto& c : cs) printf("%-36s %7.2f us/launch\n", c.name, run(c.k, c.grid, c.block, c.smem, c.cluster, c.pdl));
    return 0;
}
