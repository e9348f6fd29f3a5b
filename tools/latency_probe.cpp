// Host-side latency of the small-batch API path (device-resident inputs): where does a small
// create + emit spend its time? Build: see tools/gpu_session.sh. Prints mean us per call sequence.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#include "../include/voxgpu.h"

using Clock = std::chrono::steady_clock;

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 1;
    const int64_t len = argc > 2 ? atoll(argv[2]) : 1000;
    vxg_context* ctx = nullptr;
    if (vxg_create(0, &ctx)) return 1;
    void *d_segs, *d_out, *d_off;
    cudaMalloc(&d_segs, 48 * n);
    vxg_gen_segments(ctx, n, nullptr, nullptr, len, 0, 0, 7, (vxg_segment*)d_segs, VXG_MEM_DEVICE);
    vxg_batch* b0 = nullptr;
    vxg_batch_create(ctx, (vxg_segment*)d_segs, n, VXG_MEM_DEVICE, &b0);
    int64_t nn, mx, cap;
    vxg_batch_info(b0, &nn, &mx, &cap);
    vxg_batch_destroy(b0);
    cudaMalloc(&d_out, 12 * cap + 64);
    cudaMalloc(&d_off, 8 * (n + 1));
    const int iters = 500;
    auto run = [&](const char* name, auto&& body) {
        for (int i = 0; i < 20; ++i) body();
        vxg_synchronize(ctx);
        const auto t0 = Clock::now();
        for (int i = 0; i < iters; ++i) body();
        vxg_synchronize(ctx);
        const double us = std::chrono::duration<double, std::micro>(Clock::now() - t0).count() / iters;
        std::printf("%-40s %8.2f us\n", name, us);
    };
    run("create+destroy (no readback)", [&] {
        vxg_batch* b;
        vxg_batch_create(ctx, (vxg_segment*)d_segs, n, VXG_MEM_DEVICE, &b);
        vxg_batch_destroy(b);
    });
    run("create+info (plan readback)", [&] {
        vxg_batch* b;
        vxg_batch_create(ctx, (vxg_segment*)d_segs, n, VXG_MEM_DEVICE, &b);
        vxg_batch_info(b, &nn, &mx, &cap);
        vxg_batch_destroy(b);
    });
    run("create+emit_list(device)", [&] {
        vxg_batch* b;
        int64_t t;
        vxg_batch_create(ctx, (vxg_segment*)d_segs, n, VXG_MEM_DEVICE, &b);
        vxg_batch_emit_list(b, (vxg_voxel*)d_out, cap, (int64_t*)d_off, &t, VXG_MEM_DEVICE);
        vxg_batch_destroy(b);
    });
    run("create+emit_list+timing", [&] {
        vxg_batch* b;
        int64_t t;
        vxg_timing tm;
        vxg_batch_create(ctx, (vxg_segment*)d_segs, n, VXG_MEM_DEVICE, &b);
        vxg_batch_emit_list(b, (vxg_voxel*)d_out, cap, (int64_t*)d_off, &t, VXG_MEM_DEVICE);
        vxg_batch_timing(b, &tm);
        vxg_batch_destroy(b);
    });
    {
        vxg_batch* b;
        vxg_batch_create(ctx, (vxg_segment*)d_segs, n, VXG_MEM_DEVICE, &b);
        vxg_batch_info(b, &nn, &mx, &cap);
        run("emit_list only (resolved batch)", [&] {
            int64_t t;
            vxg_batch_emit_list(b, (vxg_voxel*)d_out, cap, (int64_t*)d_off, &t, VXG_MEM_DEVICE);
        });
        vxg_timing tm;
        vxg_batch_timing(b, &tm);
        std::printf("gpu: plan %.2f us, emit %.2f us, count+scan %.2f us\n", tm.preprocess_ns / 1e3,
                    tm.kernel_ns / 1e3, tm.assemble_ns / 1e3);
        vxg_batch_destroy(b);
    }
    {
        std::vector<vxg_voxel> chain(len + 8);
        vxg_segment seg;
        cudaMemcpy(&seg, d_segs, 48, cudaMemcpyDeviceToHost);
        run("voxelize_parametric (host)", [&] {
            int64_t c;
            vxg_voxelize_parametric(ctx, &seg, chain.data(), (int64_t)chain.size(), &c);
        });
    }
    cudaStream_t st = (cudaStream_t)vxg_get_stream(ctx);
    void* h;
    cudaHostAlloc(&h, 64, 0);
    run("bare memcpy D2H 8B + sync", [&] {
        cudaMemcpyAsync(h, d_off, 8, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
    });
    vxg_destroy(ctx);
    return 0;
}
