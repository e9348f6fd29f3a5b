// microbench_fp64.cu -- issue-rate probes for the per-sample arithmetic of the emit kernels on
// sm_100a: DMUL/DADD, the llround lowering (DADD.RZ + F2I.F64.TRUNC), a magic-number rounding
// alternative (two DADDs + integer ops, no F2I), and I2F.F64 for k -> double.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_fp64 microbench_fp64.cu
//   ./microbench_fp64        (prints ops per SM per clock for each probe)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int ILP = 8;

__global__ void k_dadd(double* out, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = a + threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = __dadd_rn(x[i], b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dmul(double* out, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = a + threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = __dmul_rn(x[i], b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// llround lowering: DADD.RZ + F2I.S32.F64.TRUNC (one "round" = 2 instructions)
__global__ void k_round_f2i(int* out, double a, double b) {
    double x[ILP];
    int acc[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
        x[i] = a + threadIdx.x + i * 0.37;
        acc[i] = 0;
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            acc[i] += __double2int_rz(__dadd_rz(x[i], copysign(0.5, x[i])));
            x[i] = __dadd_rn(x[i], b);
        }
    }
    int s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// magic-number rounding: RZ(x + copysign(0.5)) then RZ(h + copysign(2^52)) -> low word
__global__ void k_round_magic(int* out, double a, double b) {
    double x[ILP];
    int acc[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
        x[i] = a + threadIdx.x + i * 0.37;
        acc[i] = 0;
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            const double h = __dadd_rz(x[i], copysign(0.5, x[i]));
            const double t = __dadd_rz(h, copysign(4503599627370496.0, h));
            const int lo = __double2loint(t);
            const int sg = __double2hiint(t) >> 31;
            acc[i] += (lo ^ sg) - sg;
            x[i] = __dadd_rn(x[i], b);
        }
    }
    int s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_i2f(double* out, long long a) {
    long long k[ILP];
    double acc[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
        k[i] = a + threadIdx.x + i;
        acc[i] = 0;
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            acc[i] = __dadd_rn(acc[i], __ll2double_rn(k[i]));
            k[i] += 3;
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_i2f32(double* out, int a) {
    int k[ILP];
    double acc[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
        k[i] = a + threadIdx.x + i;
        acc[i] = 0;
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            acc[i] = __dadd_rn(acc[i], __int2double_rn(k[i]));
            k[i] += 3;
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// same-address atomicAdd claims (lane 0 of every warp), as a persistent-kernel work queue does
__global__ void k_claim(unsigned long long* ctr, unsigned long long* out, int iters) {
    unsigned long long acc = 0;
    for (int i = 0; i < iters; ++i) {
        unsigned long long g = 0;
        if ((threadIdx.x & 31) == 0) g = atomicAdd(ctr, 1ull);
        acc += __shfl_sync(0xffffffffu, g, 0);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    const int blocks = sms * 8, threads = 256;
    double* d;
    cudaMalloc(&d, sizeof(double) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch, double ops_per_inner) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 5.0 * blocks * threads * (double)ITERS * ILP * ops_per_inner;
        const double per_s = ops / (ms / 1e3);
        printf("%-14s %8.3f ms  %10.1f Gop/s  %7.2f op/clk/SM (at %d MHz nominal)\n", name, ms,
               per_s / 1e9, per_s / (sms * clk_khz * 1e3), clk_khz / 1000);
    };
    run("dadd", [&] { k_dadd<<<blocks, threads>>>(d, 1.0, 1e-7); }, 1);
    run("dmul", [&] { k_dmul<<<blocks, threads>>>(d, 1.0, 1.0000001); }, 1);
    run("round_f2i", [&] { k_round_f2i<<<blocks, threads>>>((int*)d, 1.0, 0.3); }, 1);
    run("round_magic", [&] { k_round_magic<<<blocks, threads>>>((int*)d, 1.0, 0.3); }, 1);
    run("i2f_s64", [&] { k_i2f<<<blocks, threads>>>(d, 1); }, 1);
    run("i2f_s32", [&] { k_i2f32<<<blocks, threads>>>(d, 1); }, 1);
    {
        unsigned long long *ctr, *o;
        cudaMalloc(&ctr, 8);
        cudaMalloc(&o, sizeof(unsigned long long) * sms * 4 * 128);
        const int iters = 256;
        k_claim<<<sms * 4, 128>>>(ctr, o, iters);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        k_claim<<<sms * 4, 128>>>(ctr, o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double claims = (double)sms * 4 * 4 * iters;
        printf("%-14s %8.3f ms  %10.1f Mclaims/s (one global counter, %d warps)\n", "claim_atomic",
               ms, claims / (ms / 1e3) / 1e6, sms * 16);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
