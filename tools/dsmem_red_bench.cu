// Shared-memory OR-reduction throughput, local vs a cluster peer's shared memory (DSMEM):
// the measurement behind DESIGN.md §9's note on cluster tiles for the bitmap fill.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dsmem_red_bench tools/dsmem_red_bench.cu
//   tools/dsmem_red_bench        (one B200; prints G reductions/s per mode)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kWords = 50000;  // 200 KB of shared memory per CTA (like the fill's tile)
constexpr int kIters = 4096;

// mode 0: every reduction to this CTA's shared memory; 1: every one to the peer CTA's;
// 2: a random half to the peer (a tile split across two SMs).
template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(1024) red_kernel(unsigned seed, unsigned* sink) {
    extern __shared__ uint32_t tile[];
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) tile[i] = 0;
    unsigned rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    const uint32_t local = (uint32_t)__cvta_generic_to_shared(tile);
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank ^ 1u));
    unsigned x = seed ^ (blockIdx.x * 1024u + threadIdx.x) * 2654435761u;
    for (int it = 0; it < kIters; ++it) {
        x = x * 1664525u + 1013904223u;
        const uint32_t w = (x >> 8) % kWords;
        const uint32_t bit = 1u << (x & 31);
        if (MODE == 0) {
            asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(local + 4 * w), "r"(bit) : "memory");
        } else {
            const bool far = MODE == 1 || (x >> 31);
            const uint32_t a = (far ? remote : local) + 4 * w;
            asm volatile("red.shared::cluster.or.b32 [%0], %1;" ::"r"(a), "r"(bit) : "memory");
        }
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0) sink[blockIdx.x] = tile[seed % kWords];
}

template <int MODE>
double run(int blocks, unsigned* sink) {
    const size_t smem = kWords * 4;
    cudaFuncSetAttribute(red_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    red_kernel<MODE><<<blocks, 1024, smem>>>(1u, sink);  // warm-up
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) red_kernel<MODE><<<blocks, 1024, smem>>>(r + 2u, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 0; }
    return (double)blocks * 1024 * kIters * reps / (ms * 1e-3) / 1e9;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms & ~1;  // one CTA per SM, 2 per cluster
    unsigned* sink;
    cudaMalloc(&sink, blocks * sizeof(unsigned));
    printf("{\"sms\": %d, \"blocks\": %d, \"threads\": 1024, \"reductions_per_thread\": %d,\n", sms, blocks, kIters);
    printf(" \"local_G_per_s\": %.1f,\n", run<0>(blocks, sink));
    printf(" \"peer_G_per_s\": %.1f,\n", run<1>(blocks, sink));
    printf(" \"half_peer_G_per_s\": %.1f}\n", run<2>(blocks, sink));
    return 0;
}
