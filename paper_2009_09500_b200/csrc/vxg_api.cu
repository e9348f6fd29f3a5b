// vxg_api.cu -- host side of libvoxgpu.so: the C ABI declared in include/voxgpu.h.
//
// Owns contexts (device, stream, events, caching device allocator) and batches (device-resident
// segments + plan == a voxline::BatchPlan). Every entry point validates arguments the way the
// reference does before touching the GPU and maps failures onto the reference's exception
// classes. There is no CPU fallback: every voxel is produced by a kernel in
// vxg_kernels.cu; if no CUDA device is usable, vxg_create fails with VXG_CUDA_ERROR.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "vxg_device.cuh"
#include "vxg_internal.h"

using vxg::Control;
using vxg::SegRec;

namespace {

using Clock = std::chrono::steady_clock;
int64_t ns_since(Clock::time_point a) {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - a).count();
}

// ---------------------------------------------------------------- caching device allocator
// cudaMalloc/cudaFree of multi-GB buffers cost milliseconds and cudaFree synchronises the
// device, so batches draw from a per-context cache (best fit, never shrinks unless an allocation
// fails, in which case the cache is released and the allocation retried once).
class DeviceCache {
   public:
    ~DeviceCache() { release(); }
    void* get(size_t bytes) {
        if (bytes == 0) bytes = 256;
        bytes = (bytes + 255) & ~size_t(255);
        std::lock_guard<std::mutex> g(mu_);
        auto it = free_.lower_bound(bytes);
        if (it != free_.end() && it->first <= bytes + bytes / 4 + (64u << 20)) {
            void* p = it->second;
            sizes_[p] = it->first;
            free_.erase(it);
            return p;
        }
        void* p = nullptr;
        if (cudaMalloc(&p, bytes) != cudaSuccess) {
            cudaGetLastError();
            release_locked();
            if (cudaMalloc(&p, bytes) != cudaSuccess) {
                cudaGetLastError();
                return nullptr;
            }
        }
        sizes_[p] = bytes;
        return p;
    }
    void put(void* p) {
        if (!p) return;
        std::lock_guard<std::mutex> g(mu_);
        auto it = sizes_.find(p);
        if (it == sizes_.end()) return;
        free_.emplace(it->second, p);
        sizes_.erase(it);
    }
    void release() {
        std::lock_guard<std::mutex> g(mu_);
        release_locked();
    }

   private:
    void release_locked() {
        if (!free_.empty()) cudaDeviceSynchronize();
        for (auto& kv : free_) cudaFree(kv.second);
        free_.clear();
    }
    std::mutex mu_;
    std::multimap<size_t, void*> free_;
    std::map<void*, size_t> sizes_;
};

// error key: ((2^59 - 1 - seg) << 3) | kind; atomicMax keeps the lowest segment.
constexpr long long kSegMax = (1ll << 59) - 1;

}  // namespace

struct vxg_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // streamed bitmap readback (created on first use)
    unsigned* h_layers = nullptr;        // mapped: per-z-layer done flags (streamed readback)
    int64_t h_layers_cap = 0;
    bool own_stream = false;
    std::string err;
    int64_t err_seg = -1;
    int64_t launches = 0;
    int num_sms = 148;
    DeviceCache cache;
    Control* h_ctl = nullptr;  // pinned readback slots (2)
    // single-chain path: mapped pinned chain buffer + control block (allocated on first use)
    int32_t* h_single = nullptr;
    Control* h_single_ctl = nullptr;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t lev[2] = {nullptr, nullptr};  // the last long_chain_kernel launch (created on use)
    bool lev_set = false;
    // one-launch small-batch path (vxg_run_batch_device): look-back words, control block, the
    // last asynchronous call's arguments (re-routed to the multi-pass path if needed)
    struct SmallState;
    SmallState* small = nullptr;

    vxg_status fail(vxg_status s, int64_t seg, const char* fmt, ...) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        err = buf;
        err_seg = seg;
        return s;
    }
    vxg_status cuda_fail(cudaError_t e, const char* where) {
        if (e == cudaErrorMemoryAllocation)
            return fail(VXG_OUT_OF_MEMORY, -1, "%s: %s", where, cudaGetErrorString(e));
        return fail(VXG_CUDA_ERROR, -1, "%s: %s", where, cudaGetErrorString(e));
    }
    void ok() {
        err.clear();
        err_seg = -1;
    }
};

// A device buffer drawn from the context cache.
struct DBuf {
    vxg_context* ctx = nullptr;
    void* p = nullptr;
    size_t bytes = 0;
    bool ensure(vxg_context* c, size_t b) {
        if (p && bytes >= b) return true;
        release();
        ctx = c;
        p = c->cache.get(b);
        bytes = p ? b : 0;
        return p != nullptr;
    }
    void release() {
        if (p && ctx) ctx->cache.put(p);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
    ~DBuf() { release(); }
};

struct vxg_context::SmallState {
    DBuf status, ctl;  // look-back words, control block
    Control* h_ctl = nullptr;  // pinned readback
    bool pending = false;
    int64_t calls = 0;  // asynchronous calls since the last result
    const vxg_segment* segs = nullptr;
    int64_t n = 0, out_cap = 0;
    vxg_voxel* out = nullptr;
    int64_t* chain = nullptr;
};

struct vxg_batch {
    vxg_context* ctx = nullptr;
    int64_t n = 0;
    const double* d_segs = nullptr;  // owned (segs) or borrowed device pointer
    DBuf segs, rec, off, status, status2, tile_seg, out, chain, entries, ent_off, ctl, ranges;
    DBuf prec;  // bitmap tile path: the records in walk order (+ their N)
    int64_t max_steps = 0, capacity = 0;
    int64_t slab_lo = 0, slab_hi = -1;  // vxg_batch_set_slab: every segment may reach this slab
    // The plan's scalars (N_max, capacity) and errors are read back lazily: batch_create only
    // enqueues the plan kernel; the first call that needs them (or the emit's own readback for a
    // small list batch) resolves the plan, so a small batch costs one host round trip, not two.
    bool plan_pending = false;
    vxg_status plan_status = VXG_OK;  // a resolved plan's error, re-reported by every later call
    std::string plan_err;
    int64_t plan_err_seg = -1;
    cudaEvent_t pev[2] = {nullptr, nullptr};  // plan kernel start / end (this batch's own)
    float plan_ms = 0.f, emit_ms = 0.f, aux_ms = 0.f;  // plan kernel / emit kernel / tile index + clip
    vxg_timing timing{0, 0, 0};
    ~vxg_batch() {
        for (cudaEvent_t e : pev)
            if (e) cudaEventDestroy(e);
    }
};

namespace {

constexpr int kMaxCtlSlots = 4;

vxg_status check_launch(vxg_context* ctx, const char* where) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return ctx->cuda_fail(e, where);
    return VXG_OK;
}

vxg_status ctl_status(vxg_context* ctx, const Control& out, const char* phase);

// Read back a Control block (synchronises the stream) and convert a recorded error.
vxg_status read_ctl(vxg_context* ctx, Control* d_ctl, Control& out, const char* phase) {
    cudaError_t e = cudaMemcpyAsync(ctx->h_ctl, d_ctl, sizeof(Control), cudaMemcpyDeviceToHost,
                                    ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, phase);
    out = *ctx->h_ctl;
    return ctl_status(ctx, out, phase);
}

vxg_status ctl_status(vxg_context* ctx, const Control& out, const char* phase) {
    if (out.abort)
        return ctx->fail(VXG_LOGIC_ERROR, -1, "%s: look-back watchdog fired (internal error)", phase);
    if (out.err_seg != 0) {
        const long long key = out.err_seg;
        const int kind = (int)(key & 7);
        const long long seg = kSegMax - (key >> 3);
        switch (kind) {
            case VXG_RANGE_ERROR:
                return ctx->fail(VXG_RANGE_ERROR, seg,
                                 "round_point: coordinate outside the 32-bit lattice or "
                                 "non-finite (segment %lld, %s)",
                                 seg, phase);
            case VXG_INVALID_ARGUMENT:
                return ctx->fail(VXG_INVALID_ARGUMENT, seg, "%s: invalid argument (item %lld)",
                                 phase, seg);
            default:
                return ctx->fail((vxg_status)kind, seg, "%s: logic error at segment %lld", phase,
                                 seg);
        }
    }
    return VXG_OK;
}

bool is_aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Pointer attributes: is `p` device-accessible memory?
bool is_device_ptr(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

vxg_status upload_segments(vxg_batch* b, const vxg_segment* segs, int64_t n, vxg_mem where) {
    vxg_context* ctx = b->ctx;
    const size_t bytes = sizeof(vxg_segment) * (size_t)n;
    if (where == VXG_MEM_DEVICE && is_aligned16(segs)) {
        b->d_segs = reinterpret_cast<const double*>(segs);
        return VXG_OK;
    }
    if (!b->segs.ensure(ctx, bytes)) return ctx->fail(VXG_OUT_OF_MEMORY, -1, "segments: out of device memory");
    const cudaError_t e =
        cudaMemcpyAsync(b->segs.p, segs, bytes,
                        where == VXG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                        ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "segments upload");
    b->d_segs = b->segs.as<double>();
    return VXG_OK;
}

Control* ctl_slot(vxg_batch* b, int i) { return b->ctl.as<Control>() + i; }

// VXG_LIST_FX=0: the list walker's fast runs evaluate every sample in FP64 (tests, A/B)
int list_fx_off() {
    const char* e = std::getenv("VXG_LIST_FX");
    return e && e[0] == '0' ? 1 : 0;
}

// Plan kernel + look-back scan (batch_preprocess).
vxg_status run_plan(vxg_batch* b) {
    vxg_context* ctx = b->ctx;
    const int64_t n = b->n;
    const int tiles = vxg::plan_tile_count(n);
    if (!b->rec.ensure(ctx, sizeof(SegRec) * (size_t)n) ||
        !b->off.ensure(ctx, sizeof(long long) * (size_t)(n + 1)) ||
        !b->status.ensure(ctx, sizeof(unsigned long long) * (size_t)tiles))
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "batch_preprocess: out of device memory");
    cudaMemsetAsync(ctl_slot(b, 0), 0, sizeof(Control), ctx->stream);
    cudaMemsetAsync(b->status.p, 0, sizeof(unsigned long long) * (size_t)tiles, ctx->stream);
    vxg::PlanArgs a{b->d_segs, n, b->rec.as<SegRec>(), b->off.as<long long>(),
                    b->status.as<unsigned long long>(), ctl_slot(b, 0)};
    cudaEventRecord(b->pev[0], ctx->stream);
    vxg::launch_plan(a, ctx->stream);
    ctx->launches++;
    cudaEventRecord(b->pev[1], ctx->stream);
    b->plan_pending = true;
    return check_launch(ctx, "plan_kernel");
}

// The plan's readback (slot 0) once it is on the host: N_max, capacity, plan errors.
vxg_status plan_resolved(vxg_batch* b, const Control& c) {
    b->plan_pending = false;
    cudaEventElapsedTime(&b->plan_ms, b->pev[0], b->pev[1]);
    const vxg_status s = ctl_status(b->ctx, c, "batch_preprocess");
    if (s) {
        b->plan_status = s;
        b->plan_err = b->ctx->err;
        b->plan_err_seg = b->ctx->err_seg;
        return s;
    }
    b->max_steps = (int64_t)c.max_steps;
    b->capacity = c.total;
    return VXG_OK;
}

// Resolve a pending plan (one readback). Every entry point that needs N_max / capacity calls it.
vxg_status plan_ready(vxg_batch* b) {
    vxg_context* ctx = b->ctx;
    if (!b->plan_pending) {
        if (b->plan_status) {
            ctx->err = b->plan_err;
            ctx->err_seg = b->plan_err_seg;
        }
        return b->plan_status;
    }
    cudaError_t e = cudaMemcpyAsync(ctx->h_ctl, ctl_slot(b, 0), sizeof(Control),
                                    cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
        b->plan_pending = false;
        return ctx->cuda_fail(e, "batch_preprocess");
    }
    return plan_resolved(b, ctx->h_ctl[0]);
}

vxg_status new_batch(vxg_context* ctx, vxg_batch** out) {
    vxg_batch* b = new (std::nothrow) vxg_batch();
    if (!b) return ctx->fail(VXG_OUT_OF_MEMORY, -1, "batch: out of host memory");
    b->ctx = ctx;
    if (!b->ctl.ensure(ctx, sizeof(Control) * kMaxCtlSlots) ||
        cudaEventCreate(&b->pev[0]) != cudaSuccess || cudaEventCreate(&b->pev[1]) != cudaSuccess) {
        delete b;
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "batch: out of device memory");
    }
    *out = b;
    return VXG_OK;
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Batches below this many segments may emit a list before their plan is read back.
constexpr int64_t kDeferredMaxSegments = 1 << 18;

// Emit the voxel list into device buffers (out: >= out_cap voxels, chain: n+1): count pass, range
// scan, emit pass.
vxg_status emit_list_device(vxg_batch* b, int32_t* d_out, int64_t out_cap, long long* d_chain,
                            int64_t* total) {
    vxg_context* ctx = b->ctx;
    const int64_t blk = vxg::list_block_samples();
    const int64_t warps = vxg::list_resident_warps(ctx->num_sms);
    const char* mode_env = std::getenv("VXG_LIST_MODE");  // (read per call: tests toggle it)
    // A small batch whose plan is still pending goes straight to the count pass: the kernels
    // derive the range geometry from the capacity the plan kernel left in off[n], and the plan's
    // and the emit's control blocks come back in ONE readback.
    const bool deferred = b->plan_pending && b->n < kDeferredMaxSegments &&
                          !(mode_env && std::strcmp(mode_env, "fused") == 0);
    if (!deferred) {
        const vxg_status s = plan_ready(b);
        if (s) return s;
    }
    // Large batches: the fused kernel over 32 ranges per resident warp (count and emit tasks
    // overlap); small ones: one range per warp, count pass + scan + emit pass.
    const bool fused = !deferred && (mode_env ? std::strcmp(mode_env, "fused") == 0
                                              : b->capacity >= (int64_t)warps * 4 * 4 * blk);
    static const int rpw_env = std::getenv("VXG_FUSED_RPW") ? std::atoi(std::getenv("VXG_FUSED_RPW")) : 32;
    static const double la_env = std::getenv("VXG_FUSED_LA") ? std::atof(std::getenv("VXG_FUSED_LA")) : 1.0;
    // (two-pass: 2/3 of the emit pass's resident warps, so the count pass -- kCountSplit warps per
    // range, 4 CTAs per SM -- runs in one wave: cfg1 0.167 -> 0.162 ms)
    int64_t nranges = fused ? rpw_env * warps : std::max<int64_t>(1, warps * 2 / 3);
    const int64_t rblk = fused ? vxg::list_fused_block_samples() : blk;
    int64_t range_len = rblk;  // deferred: the kernels scale it by the capacity they read
    if (!deferred) {
        const int64_t blocks = ceil_div(b->capacity, rblk);
        range_len = ceil_div(blocks, nranges) * rblk;
        nranges = ceil_div(b->capacity, range_len);
    }
    if (!b->ranges.ensure(ctx, sizeof(long long) * (size_t)(4 * nranges + 1)))
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "batch_voxelize: out of device memory");
    if (fused && !b->status.ensure(ctx, sizeof(unsigned long long) *
                                            (size_t)std::max<int64_t>(nranges, vxg::plan_tile_count(b->n))))
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "batch_voxelize: out of device memory");
    if ((reinterpret_cast<uintptr_t>(d_out) & 3u) != 0)
        return ctx->fail(VXG_INVALID_ARGUMENT, -1, "batch_voxelize: output must be 4-byte aligned");
    cudaMemsetAsync(ctl_slot(b, 1), 0, sizeof(Control), ctx->stream);
    long long* rc = b->ranges.as<long long>();
    vxg::ListArgs a{b->rec.as<SegRec>(), b->off.as<long long>(), b->n,
                    deferred ? -1 : b->capacity, nranges,
                    range_len, rc, rc + 3 * nranges, d_out, out_cap, d_chain, ctl_slot(b, 1),
                    fused ? b->status.as<unsigned long long>() : nullptr,
                    std::max<int64_t>(1, (int64_t)(la_env * (double)warps)),
                    deferred ? ctl_slot(b, 0) : nullptr, list_fx_off()};
    cudaError_t e;
    if (fused) {
        cudaMemsetAsync(b->status.p, 0, sizeof(unsigned long long) * (size_t)nranges, ctx->stream);
        cudaEventRecord(ctx->ev[2], ctx->stream);
        cudaEventRecord(ctx->ev[3], ctx->stream);
        e = vxg::launch_list_fused(a, ctx->num_sms, ctx->stream);
        ctx->launches += 1;
    } else {
        cudaEventRecord(ctx->ev[2], ctx->stream);
        e = vxg::launch_list_count(a, ctx->stream);
        cudaEventRecord(ctx->ev[3], ctx->stream);
        if (e == cudaSuccess) e = vxg::launch_list_emit(a, ctx->stream);
        ctx->launches += 3;
    }
    cudaEventRecord(ctx->ev[4], ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "list emit");
    Control c;
    vxg_status s;
    if (deferred) {  // slots 0 (plan) and 1 (emit) in one readback
        e = cudaMemcpyAsync(ctx->h_ctl, ctl_slot(b, 0), 2 * sizeof(Control), cudaMemcpyDeviceToHost,
                            ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) {
            b->plan_pending = false;
            return ctx->cuda_fail(e, "batch_voxelize");
        }
        c = ctx->h_ctl[1];
        s = plan_resolved(b, ctx->h_ctl[0]);
        if (!s) s = ctl_status(ctx, c, "batch_voxelize");
    } else {
        s = read_ctl(ctx, ctl_slot(b, 1), c, "batch_voxelize");
    }
    cudaEventElapsedTime(&b->aux_ms, ctx->ev[2], ctx->ev[3]);   // count pass + range scan
    cudaEventElapsedTime(&b->emit_ms, ctx->ev[3], ctx->ev[4]);  // emit pass (fused: both)
    if (s) return s;
    *total = c.total;
    return VXG_OK;
}

// BatchResult.total_voxels without the list: count pass + range scan, one readback.
vxg_status count_voxels_device(vxg_batch* b, int64_t* total) {
    vxg_context* ctx = b->ctx;
    if (const vxg_status s = plan_ready(b)) return s;
    const int64_t blk = vxg::list_block_samples();
    const int64_t warps = vxg::list_resident_warps(ctx->num_sms);
    int64_t nranges = std::max<int64_t>(1, warps * 2 / 3);
    const int64_t blocks = ceil_div(std::max<int64_t>(b->capacity, 1), blk);
    const int64_t range_len = ceil_div(blocks, nranges) * blk;
    nranges = ceil_div(std::max<int64_t>(b->capacity, 1), range_len);
    if (!b->ranges.ensure(ctx, sizeof(long long) * (size_t)(4 * nranges + 1)))
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "count_voxels: out of device memory");
    cudaMemsetAsync(ctl_slot(b, 1), 0, sizeof(Control), ctx->stream);
    long long* rc = b->ranges.as<long long>();
    vxg::ListArgs a{b->rec.as<SegRec>(), b->off.as<long long>(), b->n, b->capacity, nranges,
                    range_len, rc, rc + 3 * nranges, nullptr, 0, nullptr, ctl_slot(b, 1),
                    nullptr, 1, nullptr, list_fx_off()};
    cudaEventRecord(ctx->ev[2], ctx->stream);
    const cudaError_t e = vxg::launch_list_count(a, ctx->stream);
    ctx->launches += 2;
    cudaEventRecord(ctx->ev[3], ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "count_voxels");
    Control c;
    const vxg_status s = read_ctl(ctx, ctl_slot(b, 1), c, "count_voxels");
    cudaEventElapsedTime(&b->aux_ms, ctx->ev[2], ctx->ev[3]);
    if (s) return s;
    *total = c.total;
    return VXG_OK;
}

// Clip every segment to [z_lo, z_hi): entries + offsets; returns entries/samples.
vxg_status run_clip(vxg_batch* b, int64_t z_lo, int64_t z_hi, int64_t* n_entries,
                    int64_t* samples) {
    vxg_context* ctx = b->ctx;
    const int64_t n = b->n;
    const int tiles = vxg::clip_tile_count(n);
    if (!b->entries.ensure(ctx, sizeof(vxg::ClipEntry) * (size_t)n) ||
        !b->ent_off.ensure(ctx, sizeof(long long) * (size_t)(n + 1)) ||
        !b->status.ensure(ctx, sizeof(unsigned long long) * (size_t)std::max<int64_t>(tiles, vxg::plan_tile_count(n))) ||
        !b->status2.ensure(ctx, sizeof(unsigned long long) * (size_t)tiles))
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "clip: out of device memory");
    cudaMemsetAsync(ctl_slot(b, 2), 0, sizeof(Control), ctx->stream);
    cudaMemsetAsync(b->status.p, 0, sizeof(unsigned long long) * (size_t)tiles, ctx->stream);
    cudaMemsetAsync(b->status2.p, 0, sizeof(unsigned long long) * (size_t)tiles, ctx->stream);
    vxg::ClipArgs a{b->rec.as<SegRec>(), b->off.as<long long>(), n, z_lo, z_hi,
                    b->entries.as<vxg::ClipEntry>(), b->ent_off.as<long long>(),
                    b->status.as<unsigned long long>(), b->status2.as<unsigned long long>(),
                    ctl_slot(b, 2)};
    vxg::launch_clip(a, ctx->stream);
    ctx->launches++;
    vxg_status s = check_launch(ctx, "clip_kernel");
    if (s) return s;
    Control c;
    s = read_ctl(ctx, ctl_slot(b, 2), c, "clip");
    if (s) return s;
    *n_entries = c.n_entries;
    *samples = c.total;
    return VXG_OK;
}

// Generic path (any V): every sample ORs its bit into the bitmap with a global atomic.
vxg_status emit_bitmap_atomic(vxg_batch* b, unsigned long long* d_words, int64_t V, int64_t z_lo,
                              int64_t z_hi, int clip, int64_t* outside) {
    vxg_context* ctx = b->ctx;
    const int ts_log2 = vxg::bitmap_tile_log2();
    int64_t n_entries = b->n, samples = b->capacity;
    const long long* off = b->off.as<long long>();
    cudaEventRecord(ctx->ev[2], ctx->stream);
    if (clip) {
        vxg_status s = run_clip(b, z_lo, z_hi, &n_entries, &samples);
        if (s) return s;
        off = b->ent_off.as<long long>();
    }
    if (samples == 0) {
        if (outside) *outside = 0;
        b->emit_ms = b->aux_ms = 0.f;
        return VXG_OK;
    }
    const int64_t ntiles = ceil_div(samples, 1ll << ts_log2);
    if (!b->tile_seg.ensure(ctx, sizeof(long long) * (size_t)ntiles))
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "bitmap: out of device memory");
    cudaMemsetAsync(ctl_slot(b, 3), 0, sizeof(Control), ctx->stream);
    vxg::launch_tile_index(off, n_entries, ts_log2, b->tile_seg.as<long long>(), ctx->stream);
    cudaEventRecord(ctx->ev[3], ctx->stream);
    vxg::BitmapArgs a{b->rec.as<SegRec>(), clip ? b->entries.as<vxg::ClipEntry>() : nullptr, off,
                      b->tile_seg.as<long long>(), n_entries, samples, ntiles, d_words, V, z_lo,
                      z_hi, ctl_slot(b, 3)};
    cudaError_t e = vxg::launch_emit_bitmap(a, clip != 0, ctx->stream);
    ctx->launches += 2;
    cudaEventRecord(ctx->ev[4], ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "emit_bitmap_kernel");
    Control c;
    vxg_status s = read_ctl(ctx, ctl_slot(b, 3), c, "bitmap");
    cudaEventElapsedTime(&b->aux_ms, ctx->ev[2], ctx->ev[3]);
    cudaEventElapsedTime(&b->emit_ms, ctx->ev[3], ctx->ev[4]);
    if (s) return s;
    if (outside) *outside = (int64_t)c.outside;
    return VXG_OK;
}


// Tile-binned path (vxg_bitmap.cu): V a multiple of 128, every N_i < 2^31.
// Streamed readback of a host bitmap: while the fill kernel runs, every z-layer of tiles it has
// finished (counted in mapped memory by the kernel) is copied to the host on the copy stream, so
// the PCIe transfer overlaps the fill instead of following it.
struct LayerStream {
    uint64_t* host_words;
    unsigned* flags;  // mapped, one per z-layer: 1 once every tile of the layer is final
};

bool layer_stream_setup(vxg_context* ctx, int64_t ntz, LayerStream& ls) {
    if (!ctx->copy_stream &&
        cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (ctx->h_layers_cap < ntz) {
        if (ctx->h_layers) cudaFreeHost(ctx->h_layers);
        ctx->h_layers = nullptr;
        ctx->h_layers_cap = 0;
        void* p = nullptr;
        if (cudaHostAlloc(&p, sizeof(unsigned) * (size_t)ntz, cudaHostAllocMapped) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        ctx->h_layers = static_cast<unsigned*>(p);
        ctx->h_layers_cap = ntz;
    }
    std::memset(ctx->h_layers, 0, sizeof(unsigned) * (size_t)ntz);
    ls.flags = ctx->h_layers;
    return true;
}

vxg_status emit_bitmap_tiles(vxg_batch* b, unsigned long long* d_words, int64_t V, int64_t z_lo,
                             int64_t z_hi, int64_t* outside, uint64_t* host_words = nullptr,
                             bool overwrite = false) {
    vxg_context* ctx = b->ctx;
    vxg::TileArgs g{};
    g.overwrite = overwrite ? 1 : 0;
    g.rec = b->rec.as<SegRec>();
    g.off = b->off.as<long long>();
    g.n = b->n;
    g.V = V;
    g.z_lo = z_lo;
    g.z_hi = z_hi;
    vxg::tile_dims(V, z_hi - z_lo, g.tx, g.ty, g.tz);
    g.ntx = ceil_div(V, g.tx);
    g.nty = ceil_div(V, g.ty);
    g.ntz = ceil_div(z_hi - z_lo, g.tz);
    g.ntiles = g.ntx * g.nty * g.ntz;
    const long long nbins = g.ntiles * vxg::tile_len_classes();
    if (!b->tile_seg.ensure(ctx, sizeof(long long) * (size_t)(2 * nbins + 1) + 4 * (size_t)nbins))
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "bitmap: out of device memory");
    g.tile_cnt = b->tile_seg.as<long long>();
    g.tile_off = g.tile_cnt + nbins;
    g.tile_cur = reinterpret_cast<unsigned*>(g.tile_off + nbins + 1);
    g.words = d_words;
    g.ctl = ctl_slot(b, 3);
    LayerStream ls{host_words, nullptr};
    DBuf layer_cnt;
    // (if the streamed readback cannot be set up, the words are read back after the fill)
    if (host_words && (!layer_stream_setup(ctx, g.ntz, ls) ||
                       !layer_cnt.ensure(ctx, sizeof(unsigned) * (size_t)g.ntz)))
        ls.host_words = nullptr;
    const size_t slab_bytes = 8 * (size_t)(((V * V * (z_hi - z_lo)) + 63) / 64);
    auto plain_readback = [&]() -> vxg_status {
        cudaError_t ce = cudaMemcpyAsync(host_words, d_words, slab_bytes, cudaMemcpyDeviceToHost,
                                         ctx->stream);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(ctx->stream);
        return ce == cudaSuccess ? VXG_OK : ctx->cuda_fail(ce, "bitmap readback");
    };
    if (ls.host_words) {
        cudaMemsetAsync(layer_cnt.p, 0, sizeof(unsigned) * (size_t)g.ntz, ctx->stream);
        g.layer_cnt = layer_cnt.as<unsigned>();
        g.layer_done = ls.flags;
    }
    cudaEventRecord(ctx->ev[2], ctx->stream);
    cudaMemsetAsync(g.ctl, 0, sizeof(Control), ctx->stream);
    cudaMemsetAsync(g.tile_cnt, 0, sizeof(long long) * (size_t)nbins, ctx->stream);
    DBuf scan_status;  // the bin scan's look-back words
    const int scan_tiles = vxg::tile_scan_tiles(nbins);
    if (scan_status.ensure(ctx, sizeof(unsigned long long) * (size_t)scan_tiles)) {
        cudaMemsetAsync(scan_status.p, 0, sizeof(unsigned long long) * (size_t)scan_tiles, ctx->stream);
        g.scan_status = scan_status.as<unsigned long long>();
    }
    // A thin slab (one rank's share): the passes walk only the segments that reach it.
    const bool select = b->n >= (1 << 16) && b->n < (1ll << 31) && z_hi - z_lo < V &&
                        !(b->slab_lo <= z_lo && z_hi <= b->slab_hi) &&  // (filtered already)
                        !std::getenv("VXG_BITMAP_NO_SELECT");
    // Walk order grouped by segment length and start cell (pays off when lengths vary). Thin
    // slabs (below a quarter of the volume) only with the record copy (N < 2^28): as an index
    // permutation the sort cost them about what it saved (one rank of 8 on cfg5: 18.00 ->
    // 17.84 ms); with the copy and the in-slab length key (perm_key) it pays: cfg5 rank steps
    // N = 4 25.90 -> 24.31 ms, N = 8 14.79 -> 14.22 (tools/slab_probe.py,
    // profiles/r2_multigpu_s6/).
    const bool copyable = b->max_steps < (1ll << (32 - vxg::kRecNShift)) &&
                          !std::getenv("VXG_BITMAP_PERM_INDEX");
    const bool perm = b->n >= (1 << 16) && b->n < (1ll << 31) && b->max_steps >= 256 &&
                      (4 * (z_hi - z_lo) >= V || copyable || std::getenv("VXG_BITMAP_PERM")) &&
                      !std::getenv("VXG_BITMAP_NO_PERM");
    if (select || perm) {
        const size_t keys = (size_t)vxg::tile_perm_keys();
        if (!b->ent_off.ensure(ctx, keys * sizeof(long long) + sizeof(unsigned long long) +
                                        2 * sizeof(int) * (size_t)b->n))
            return ctx->fail(VXG_OUT_OF_MEMORY, -1, "bitmap: out of device memory");
        long long* perm_cur = b->ent_off.as<long long>();
        auto* nsel = reinterpret_cast<unsigned long long*>(perm_cur + keys);
        int* sel = reinterpret_cast<int*>(nsel + 1);
        int* order = sel + b->n;
        if (select) {
            cudaMemsetAsync(nsel, 0, sizeof(unsigned long long), ctx->stream);
            vxg::launch_slab_select(g, sel, nsel, ctx->stream);
            ctx->launches++;
            unsigned long long ns = 0;
            cudaError_t e = cudaMemcpyAsync(ctx->h_ctl, nsel, sizeof(ns), cudaMemcpyDeviceToHost,
                                            ctx->stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
            if (e != cudaSuccess) return ctx->cuda_fail(e, "bitmap: slab selection");
            std::memcpy(&ns, ctx->h_ctl, sizeof(ns));
            g.sel = sel;
            g.n = (long long)ns;
            g.perm = sel;  // (walk order = the selection's, unless sorted below)
        }
        if (perm && g.n > 0) {
            g.perm_cur = perm_cur;
            g.perm = order;
            // Copy the records into walk order when the memory is there: the count and scatter
            // passes then read them sequentially instead of gathering 64 B per segment (whole
            // 128-B lines come from DRAM for each gather).
            // (N rides in the copy's flag word: N < 2^28)
            const bool copy = copyable && b->prec.ensure(ctx, sizeof(SegRec) * (size_t)g.n);
            if (copy) g.prec = b->prec.as<SegRec>();
            cudaMemsetAsync(perm_cur, 0, keys * sizeof(long long), ctx->stream);
            vxg::launch_tiles_perm(g, ctx->stream);
            ctx->launches += 3;
            if (copy) {  // from here on segment ids are positions in the copy
                g.rec = g.prec;
                g.rec_n = 1;
                g.perm = nullptr;
                g.sel = nullptr;
                g.prec = nullptr;
            }
        }
    }
    vxg::launch_tiles_count(g, ctx->stream);
    vxg::launch_tiles_scan(g, ctx->stream);
    ctx->launches += 2;
    Control c;
    vxg_status s = read_ctl(ctx, g.ctl, c, "bitmap");
    if (s) return s;
    const long long npieces = c.n_entries;
    const long long in_box = (long long)c.outside;  // samples inside the slab box
    if (outside) *outside = b->capacity - c.total;
    if (npieces == 0) {
        b->emit_ms = b->aux_ms = 0.f;
        // nothing to fill: the device words (zeroed or uploaded) go back as they are
        if (overwrite) cudaMemsetAsync(d_words, 0, slab_bytes, ctx->stream);
        return host_words ? plain_readback() : VXG_OK;
    }
    // More pieces than the 32-bit bin cursors count, or than the device holds as 32-B records:
    // the slab is done as two thinner slabs (each a contiguous run of the words), recursively.
    // The outside count is a property of the whole volume: the first half reports it.
    long long max_pieces = 1ll << 32;
    if (const char* e = std::getenv("VXG_BITMAP_MAX_PIECES")) max_pieces = std::atoll(e);  // tests
    const bool fits = npieces < max_pieces &&
                      b->entries.ensure(ctx, 2 * sizeof(uint4) * (size_t)npieces);
    if (!fits) {
        if (g.ntz < 2)
            return ctx->fail(VXG_OUT_OF_MEMORY, -1,
                             "bitmap: %lld pieces in one layer of tiles exceed the device", npieces);
        const int64_t zm = z_lo + (g.ntz / 2) * g.tz;
        const int64_t plane_words = V * V / 64;  // (V is a multiple of the tile width)
        ls = LayerStream{};
        s = emit_bitmap_tiles(b, d_words, V, z_lo, zm, nullptr, host_words, overwrite);
        if (s) return s;
        return emit_bitmap_tiles(b, d_words + (zm - z_lo) * plane_words, V, zm, z_hi, nullptr,
                                 host_words ? host_words + (zm - z_lo) * plane_words : nullptr,
                                 overwrite);
    }
    g.pieces = b->entries.as<uint4>();
    vxg::launch_tiles_scatter(g, ctx->stream);
    cudaEventRecord(ctx->ev[3], ctx->stream);
    const cudaError_t e = vxg::launch_tiles_fill(g, ctx->num_sms, (double)in_box / (double)npieces,
                                                ctx->stream);
    ctx->launches += 2;
    cudaEventRecord(ctx->ev[4], ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "tiles_fill_kernel");
    cudaError_t qe = cudaSuccess;
    if (ls.host_words) {  // copy each finished layer while the fill goes on
        const int64_t plane_words = V * V / 64;
        std::vector<char> copied((size_t)g.ntz, 0);
        int64_t left = g.ntz;
        bool done = false;
        while (left > 0) {
            bool any = false;
            for (int64_t l = 0; l < g.ntz; ++l) {
                if (copied[(size_t)l]) continue;
                if (!done && reinterpret_cast<volatile unsigned*>(ls.flags)[l] == 0u) continue;
                const int64_t za = z_lo + l * g.tz, zb = std::min<int64_t>(za + g.tz, z_hi);
                const int64_t w0 = (za - z_lo) * plane_words;
                cudaMemcpyAsync(ls.host_words + w0, d_words + w0, 8 * (size_t)((zb - za) * plane_words),
                                cudaMemcpyDeviceToHost, ctx->copy_stream);
                copied[(size_t)l] = 1;
                --left;
                any = true;
            }
            if (left == 0) break;
            if (!done) {
                qe = cudaStreamQuery(ctx->stream);
                if (qe == cudaSuccess) {
                    done = true;  // the fill is over: copy whatever is left
                    continue;
                }
                if (qe != cudaErrorNotReady) break;
                qe = cudaSuccess;
            }
            if (!any) std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
    }
    s = read_ctl(ctx, g.ctl, c, "bitmap");
    if (ls.host_words) {
        const cudaError_t ce = cudaStreamSynchronize(ctx->copy_stream);
        if (!s && qe != cudaSuccess) s = ctx->cuda_fail(qe, "tiles_fill_kernel");
        if (!s && ce != cudaSuccess) s = ctx->cuda_fail(ce, "bitmap readback");
    }
    cudaEventElapsedTime(&b->aux_ms, ctx->ev[2], ctx->ev[3]);
    cudaEventElapsedTime(&b->emit_ms, ctx->ev[3], ctx->ev[4]);
    if (!s && host_words && !ls.host_words) s = plain_readback();  // (streaming was unavailable)
    return s;
}

bool use_tiles(const vxg_batch* b, int64_t V, int64_t z_lo, int64_t z_hi) {
    return V % 128 == 0 && b->max_steps < (1ll << 31) && z_hi > z_lo &&
           !std::getenv("VXG_BITMAP_ATOMIC");
}

vxg_status emit_bitmap_device(vxg_batch* b, unsigned long long* d_words, int64_t V, int64_t z_lo,
                              int64_t z_hi, int clip, int64_t* outside, bool overwrite = false) {
    // overwrite: the tile path stores every word of the slab itself (no memset, no read of the
    // old words); the global-atomic path ORs into a zeroed buffer
    if (use_tiles(b, V, z_lo, z_hi))
        return emit_bitmap_tiles(b, d_words, V, z_lo, z_hi, outside, nullptr, overwrite);
    if (overwrite) {
        const size_t nwords = (size_t)((V * V * (z_hi - z_lo) + 63) / 64);
        cudaMemsetAsync(d_words, 0, 8 * nwords, b->ctx->stream);
    }
    return emit_bitmap_atomic(b, d_words, V, z_lo, z_hi, clip, outside);
}

}  // namespace

// =============================================================================== C ABI
extern "C" {

VXG_API int vxg_abi_version(void) { return VXG_ABI_VERSION; }

VXG_API vxg_status vxg_create(int device, vxg_context** out) {
    if (!out) return VXG_INVALID_ARGUMENT;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return VXG_CUDA_ERROR;
    }
    if (device < 0 || device >= count) return VXG_INVALID_ARGUMENT;
    if (cudaSetDevice(device) != cudaSuccess) return VXG_CUDA_ERROR;
    vxg_context* ctx = new (std::nothrow) vxg_context();
    if (!ctx) return VXG_OUT_OF_MEMORY;
    ctx->device = device;
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_ctl), 2 * sizeof(Control), cudaHostAllocDefault) !=
            cudaSuccess ||
        cudaEventCreate(&ctx->ev[0]) != cudaSuccess || cudaEventCreate(&ctx->ev[1]) != cudaSuccess ||
        cudaEventCreate(&ctx->ev[2]) != cudaSuccess || cudaEventCreate(&ctx->ev[3]) != cudaSuccess ||
        cudaEventCreate(&ctx->ev[4]) != cudaSuccess) {
        delete ctx;
        return VXG_CUDA_ERROR;
    }
    ctx->own_stream = true;
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    *out = ctx;
    return VXG_OK;
}

VXG_API void vxg_destroy(vxg_context* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->copy_stream) {
        cudaStreamSynchronize(ctx->copy_stream);
        cudaStreamDestroy(ctx->copy_stream);
    }
    if (ctx->h_layers) cudaFreeHost(ctx->h_layers);
    if (ctx->small) {
        if (ctx->small->h_ctl) cudaFreeHost(ctx->small->h_ctl);
        delete ctx->small;  // (its buffers go back to the cache, released next)
    }
    ctx->cache.release();
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    if (ctx->h_ctl) cudaFreeHost(ctx->h_ctl);
    if (ctx->h_single) cudaFreeHost(ctx->h_single);
    for (cudaEvent_t e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ctx->lev)
        if (e) cudaEventDestroy(e);
    delete ctx;
}

VXG_API vxg_status vxg_set_stream(vxg_context* ctx, void* stream) {
    if (!ctx) return VXG_INVALID_ARGUMENT;
    cudaStreamSynchronize(ctx->stream);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    if (stream) {
        ctx->stream = static_cast<cudaStream_t>(stream);
        ctx->own_stream = false;
    } else {
        if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess)
            return VXG_CUDA_ERROR;
        ctx->own_stream = true;
    }
    return VXG_OK;
}

VXG_API void* vxg_get_stream(vxg_context* ctx) { return ctx ? ctx->stream : nullptr; }
VXG_API const char* vxg_last_error(const vxg_context* ctx) { return ctx ? ctx->err.c_str() : "no context"; }
VXG_API int64_t vxg_last_error_segment(const vxg_context* ctx) { return ctx ? ctx->err_seg : -1; }
VXG_API int64_t vxg_launch_count(const vxg_context* ctx) { return ctx ? ctx->launches : 0; }

VXG_API vxg_status vxg_synchronize(vxg_context* ctx) {
    if (!ctx) return VXG_INVALID_ARGUMENT;
    const cudaError_t e = cudaStreamSynchronize(ctx->stream);
    return e == cudaSuccess ? VXG_OK : ctx->cuda_fail(e, "synchronize");
}

VXG_API void* vxg_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}
VXG_API void vxg_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

// ------------------------------------------------------------------------------- geometry
VXG_API vxg_status vxg_round_points(vxg_context* ctx, const double* pts, int64_t n, int32_t* out) {
    if (!ctx || n < 0 || (n && (!pts || !out))) return VXG_INVALID_ARGUMENT;
    ctx->ok();
    if (n == 0) return VXG_OK;
    cudaSetDevice(ctx->device);
    DBuf dp, dout, dctl;
    if (!dp.ensure(ctx, 24 * (size_t)n) || !dout.ensure(ctx, 12 * (size_t)n) ||
        !dctl.ensure(ctx, sizeof(Control)))
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "round_point: out of device memory");
    cudaMemcpyAsync(dp.p, pts, 24 * (size_t)n, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemsetAsync(dctl.p, 0, sizeof(Control), ctx->stream);
    vxg::launch_round_points(dp.as<double>(), n, dout.as<int32_t>(), dctl.as<Control>(), ctx->stream);
    ctx->launches++;
    cudaMemcpyAsync(out, dout.p, 12 * (size_t)n, cudaMemcpyDeviceToHost, ctx->stream);
    Control c;
    return read_ctl(ctx, dctl.as<Control>(), c, "round_point");
}

VXG_API vxg_status vxg_segment_lengths(vxg_context* ctx, const vxg_segment* segs, int64_t n,
                                       double* out) {
    if (!ctx || n < 0 || (n && (!segs || !out))) return VXG_INVALID_ARGUMENT;
    ctx->ok();
    if (n == 0) return VXG_OK;
    cudaSetDevice(ctx->device);
    DBuf ds, dout;
    if (!ds.ensure(ctx, 48 * (size_t)n) || !dout.ensure(ctx, 8 * (size_t)n))
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "segment_length: out of device memory");
    cudaMemcpyAsync(ds.p, segs, 48 * (size_t)n, cudaMemcpyHostToDevice, ctx->stream);
    vxg::launch_segment_lengths(ds.as<double>(), n, dout.as<double>(), ctx->stream);
    ctx->launches++;
    cudaMemcpyAsync(out, dout.p, 8 * (size_t)n, cudaMemcpyDeviceToHost, ctx->stream);
    const cudaError_t e = cudaStreamSynchronize(ctx->stream);
    return e == cudaSuccess ? VXG_OK : ctx->cuda_fail(e, "segment_length");
}

VXG_API vxg_status vxg_make_plans(vxg_context* ctx, const vxg_segment* segs, int64_t n,
                                  int64_t* steps, double* w3) {
    if (!ctx || n <= 0 || !segs) return ctx ? ctx->fail(VXG_INVALID_ARGUMENT, -1, "make_plan: no segments") : VXG_INVALID_ARGUMENT;
    vxg_batch* b = nullptr;
    vxg_status s = vxg_batch_create(ctx, segs, n, VXG_MEM_HOST, &b);
    if (s) return s;
    std::vector<vxg_segment_plan> plans((size_t)n);
    s = vxg_batch_plans(b, plans.data());
    vxg_batch_destroy(b);
    if (s) return s;
    for (int64_t i = 0; i < n; ++i) {
        if (steps) steps[i] = plans[(size_t)i].step_count;
        if (w3) {
            w3[3 * i + 0] = plans[(size_t)i].wx;
            w3[3 * i + 1] = plans[(size_t)i].wy;
            w3[3 * i + 2] = plans[(size_t)i].wz;
        }
    }
    return VXG_OK;
}

// Chains up to this many samples take the one-launch single_chain_kernel (one CTA: ~2.5 us per
// 1024 samples on top of a ~12 us launch + synchronisation; longer chains are faster through the
// batch path's full-GPU passes).
constexpr int64_t kSingleMaxSamples = 1 << 14;

// voxelize_parametric in one launch + one synchronisation (see single_chain_kernel). Returns
// false when the segment is too long (or non-finite) for it: the caller takes the batch path.
bool single_chain(vxg_context* ctx, const vxg_segment* seg, vxg_voxel* out, int64_t cap,
                  int64_t* count, vxg_status* st) {
    // dispatch bound on N + 1 from the endpoints (the kernel recomputes N exactly and refuses,
    // writing nothing, if the bound was wrong)
    const double dx = seg->ex - seg->sx, dy = seg->ey - seg->sy, dz = seg->ez - seg->sz;
    // N = max(floor(len), ceil(max|d|), 1) and max|d| <= len, so N + 1 <= len + 2 (+ slack for
    // this host-side len differing from the kernel's in the last place)
    const double ext = std::max(std::fabs(dx), std::max(std::fabs(dy), std::fabs(dz)));
    const double bound = std::max(std::sqrt(dx * dx + dy * dy + dz * dz), ext) + 4.0;
    if (!(bound < (double)kSingleMaxSamples)) return false;  // long, or non-finite: batch path
    if (!ctx->h_single) {
        void* p = nullptr;
        if (cudaHostAlloc(&p, 12 * (size_t)kSingleMaxSamples + sizeof(Control), cudaHostAllocMapped) !=
            cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        ctx->h_single = static_cast<int32_t*>(p);
        ctx->h_single_ctl = reinterpret_cast<Control*>(ctx->h_single + 3 * kSingleMaxSamples);
    }
    std::memset(ctx->h_single_ctl, 0, sizeof(Control));
    vxg::SingleArgs a{{seg->sx, seg->sy, seg->sz, seg->ex, seg->ey, seg->ez},
                      kSingleMaxSamples, kSingleMaxSamples, ctx->h_single, ctx->h_single_ctl};
    cudaError_t e = vxg::launch_single_chain(a, ctx->stream);
    ctx->launches++;
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
        *st = ctx->cuda_fail(e, "voxelize_parametric");
        return true;
    }
    const Control c = *ctx->h_single_ctl;
    if (c.n_entries != 0) return false;  // longer than the bound: batch path
    *st = ctl_status(ctx, c, "voxelize_parametric");
    if (*st) return true;
    *count = c.total;
    const int64_t ncopy = std::min<int64_t>(c.total, cap);
    if (ncopy > 0) std::memcpy(out, ctx->h_single, 12 * (size_t)ncopy);
    if (c.total > cap)
        *st = ctx->fail(VXG_LOGIC_ERROR, 0, "voxelize_parametric: chain of %lld voxels exceeds cap %lld",
                        (long long)c.total, (long long)cap);
    return true;
}

// Longer chains (up to kLongMaxSamples): one launch of long_chain_kernel over as many CTAs as the
// host-side bound on N + 1 asks for, writing at most `cap` voxels to device memory, then one
// readback of the control block. Returns false when the segment is too long or non-finite (or the
// look-back words cannot be allocated): the caller takes the batch path.
constexpr double kLongMaxSamples = (double)(1ll << 30);

bool long_chain(vxg_context* ctx, const vxg_segment* seg, int32_t* d_out, int64_t cap,
                int64_t* count, vxg_status* st) {
    const double dx = seg->ex - seg->sx, dy = seg->ey - seg->sy, dz = seg->ez - seg->sz;
    const double ext = std::max(std::fabs(dx), std::max(std::fabs(dy), std::fabs(dz)));
    const double bound = std::max(std::sqrt(dx * dx + dy * dy + dz * dz), ext) + 4.0;  // (as above)
    if (!(bound < kLongMaxSamples)) return false;
    const long long per = vxg::long_chain_samples_per_cta();
    const long long ctas = (long long)bound / per + 1;
    DBuf buf;
    const size_t bytes = sizeof(Control) + sizeof(unsigned long long) * (size_t)ctas;
    if (!buf.ensure(ctx, bytes)) return false;
    Control* d_ctl = buf.as<Control>();
    cudaMemsetAsync(buf.p, 0, bytes, ctx->stream);
    vxg::LongArgs a{{seg->sx, seg->sy, seg->sz, seg->ex, seg->ey, seg->ez}, cap, ctas * per, d_out,
                    reinterpret_cast<unsigned long long*>(d_ctl + 1), d_ctl};
    if (!ctx->lev[0] && (cudaEventCreate(&ctx->lev[0]) != cudaSuccess ||
                         cudaEventCreate(&ctx->lev[1]) != cudaSuccess))
        return false;
    cudaEventRecord(ctx->lev[0], ctx->stream);
    cudaError_t e = vxg::launch_long_chain(a, ctas, ctx->stream);
    cudaEventRecord(ctx->lev[1], ctx->stream);
    ctx->lev_set = true;
    ctx->launches++;
    if (e == cudaSuccess) e = cudaMemcpyAsync(ctx->h_ctl, d_ctl, sizeof(Control), cudaMemcpyDeviceToHost,
                                              ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
        *st = ctx->cuda_fail(e, "voxelize_parametric");
        return true;
    }
    const Control c = *ctx->h_ctl;
    if (c.n_entries != 0) return false;  // longer than the bound: batch path
    *st = ctl_status(ctx, c, "voxelize_parametric");
    if (*st) return true;
    *count = c.total;
    if (c.total > cap)
        *st = ctx->fail(VXG_LOGIC_ERROR, 0, "voxelize_parametric: chain of %lld voxels exceeds cap %lld",
                        (long long)c.total, (long long)cap);
    return true;
}

VXG_API vxg_status vxg_voxelize_parametric(vxg_context* ctx, const vxg_segment* seg,
                                           vxg_voxel* out, int64_t cap, int64_t* count) {
    if (!ctx || !seg || !count || cap < 0 || (cap > 0 && !out)) return VXG_INVALID_ARGUMENT;
    ctx->ok();
    cudaSetDevice(ctx->device);
    if (!std::getenv("VXG_NO_SINGLE")) {
        vxg_status st = VXG_OK;
        if (single_chain(ctx, seg, out, cap, count, &st)) return st;
        // a long chain: one launch into device memory, then its voxels come back
        const double dx = seg->ex - seg->sx, dy = seg->ey - seg->sy, dz = seg->ez - seg->sz;
        const double bound = std::max(std::sqrt(dx * dx + dy * dy + dz * dz),
                                      std::max(std::fabs(dx), std::max(std::fabs(dy), std::fabs(dz)))) + 4.0;
        DBuf dout;
        const int64_t dcap = bound < kLongMaxSamples ? std::min<int64_t>(cap, (int64_t)bound + 1) : 0;
        int64_t total = 0;
        if (dcap >= 0 && bound < kLongMaxSamples && dout.ensure(ctx, 12 * (size_t)std::max<int64_t>(dcap, 1)) &&
            long_chain(ctx, seg, dout.as<int32_t>(), dcap, &total, &st)) {
            if (st && st != VXG_LOGIC_ERROR) return st;  // (a plan / range error: nothing to copy)
            if (st) st = VXG_OK, ctx->ok();             // (total > dcap: decided against cap below)
            *count = total;
            const int64_t ncopy = std::min(total, cap);
            if (ncopy > 0) {
                cudaError_t e = cudaMemcpyAsync(out, dout.p, 12 * (size_t)ncopy, cudaMemcpyDeviceToHost,
                                                ctx->stream);
                if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
                if (e != cudaSuccess) return ctx->cuda_fail(e, "voxelize_parametric readback");
            }
            if (total > cap)
                return ctx->fail(VXG_LOGIC_ERROR, 0, "voxelize_parametric: chain of %lld voxels exceeds cap %lld",
                                 (long long)total, (long long)cap);
            return VXG_OK;
        }
    }
    vxg_batch* b = nullptr;
    vxg_status s = vxg_batch_create(ctx, seg, 1, VXG_MEM_HOST, &b);
    if (!s) s = plan_ready(b);
    if (s) {
        vxg_batch_destroy(b);
        return s;
    }
    if (!b->out.ensure(ctx, 12 * (size_t)b->capacity) || !b->chain.ensure(ctx, 16)) {
        vxg_batch_destroy(b);
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "voxelize_parametric: out of device memory");
    }
    int64_t total = 0;
    s = emit_list_device(b, b->out.as<int32_t>(), b->capacity, b->chain.as<long long>(), &total);
    if (!s) {
        *count = total;
        const int64_t ncopy = std::min(total, cap);
        if (ncopy > 0) {
            const cudaError_t e = cudaMemcpyAsync(out, b->out.p, 12 * (size_t)ncopy,
                                                  cudaMemcpyDeviceToHost, ctx->stream);
            if (e == cudaSuccess) cudaStreamSynchronize(ctx->stream);
            else s = ctx->cuda_fail(e, "voxelize_parametric readback");
        }
        if (!s && total > cap)
            s = ctx->fail(VXG_LOGIC_ERROR, 0, "voxelize_parametric: chain of %lld voxels exceeds cap %lld",
                          (long long)total, (long long)cap);
    }
    vxg_batch_destroy(b);
    return s;
}

VXG_API vxg_status vxg_voxelize_parametric_device(vxg_context* ctx, const vxg_segment* seg,
                                                  vxg_voxel* d_out, int64_t cap, int64_t* count) {
    if (!ctx || !seg || !count || cap < 0 || (cap > 0 && !d_out)) return VXG_INVALID_ARGUMENT;
    if ((reinterpret_cast<uintptr_t>(d_out) & 3u) != 0)
        return ctx->fail(VXG_INVALID_ARGUMENT, -1, "voxelize_parametric: output must be 4-byte aligned");
    ctx->ok();
    cudaSetDevice(ctx->device);
    vxg_status st = VXG_OK;
    if (long_chain(ctx, seg, reinterpret_cast<int32_t*>(d_out), cap, count, &st)) return st;
    // (too long for one launch: the batch passes, straight into the caller's buffer)
    vxg_batch* b = nullptr;
    vxg_status s = vxg_batch_create(ctx, seg, 1, VXG_MEM_HOST, &b);
    if (!s) s = plan_ready(b);
    DBuf chain;
    if (!s && !chain.ensure(ctx, 16)) s = ctx->fail(VXG_OUT_OF_MEMORY, -1, "voxelize_parametric: out of device memory");
    int64_t total = 0;
    if (!s) s = emit_list_device(b, reinterpret_cast<int32_t*>(d_out), cap, chain.as<long long>(), &total);
    if (!s) *count = total;
    vxg_batch_destroy(b);
    return s;
}

VXG_API vxg_status vxg_voxelize_parametric_timing(vxg_context* ctx, vxg_timing* t) {
    if (!ctx || !t) return VXG_INVALID_ARGUMENT;
    *t = vxg_timing{0, 0, 0};
    if (!ctx->lev_set) return VXG_OK;
    float ms = 0.f;
    const cudaError_t e = cudaEventElapsedTime(&ms, ctx->lev[0], ctx->lev[1]);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "voxelize_parametric_timing");
    t->kernel_ns = (int64_t)((double)ms * 1e6);
    return VXG_OK;
}

VXG_API vxg_status vxg_chain_length_bounds(vxg_context* ctx, const vxg_segment* seg, int64_t* lo,
                                           int64_t* hi) {
    if (!ctx || !seg || !lo || !hi) return VXG_INVALID_ARGUMENT;
    // rounded endpoints and the plan both come from the GPU (src/parametric.cpp:42-50)
    const double pts[6] = {seg->sx, seg->sy, seg->sz, seg->ex, seg->ey, seg->ez};
    int32_t v[6];
    vxg_status s = vxg_round_points(ctx, pts, 2, v);
    if (s) return s;
    int64_t n = 0;
    s = vxg_make_plans(ctx, seg, 1, &n, nullptr);
    if (s) return s;
    int64_t span = 0;
    for (int a = 0; a < 3; ++a) span = std::max<int64_t>(span, std::llabs((int64_t)v[3 + a] - v[a]));
    *lo = span + 1;
    *hi = n + 1;
    return VXG_OK;
}

// ------------------------------------------------------------------------------- batch
VXG_API vxg_status vxg_batch_create(vxg_context* ctx, const vxg_segment* segs, int64_t n,
                                    vxg_mem where, vxg_batch** out) {
    if (!ctx || !out) return VXG_INVALID_ARGUMENT;
    ctx->ok();
    *out = nullptr;
    if (n <= 0) return ctx->fail(VXG_INVALID_ARGUMENT, -1, "batch_preprocess: empty segment list");
    if (!segs) return ctx->fail(VXG_INVALID_ARGUMENT, -1, "batch_preprocess: null segments");
    cudaSetDevice(ctx->device);
    vxg_batch* b = nullptr;
    vxg_status s = new_batch(ctx, &b);
    if (s) return s;
    b->n = n;
    const auto t0 = Clock::now();
    s = upload_segments(b, segs, n, where);
    if (!s) s = run_plan(b);
    // host segments: resolve now (the call is synchronous for host pointers, and plan errors
    // surface here as batch_preprocess's do); device segments: lazily (see vxg_batch)
    if (!s && where == VXG_MEM_HOST) s = plan_ready(b);
    b->timing.preprocess_ns = ns_since(t0);
    if (s) {
        delete b;
        return s;
    }
    *out = b;
    return VXG_OK;
}

VXG_API vxg_status vxg_batch_set_slab(vxg_batch* b, int64_t z_lo, int64_t z_hi) {
    if (!b) return VXG_INVALID_ARGUMENT;
    b->ctx->ok();
    if (z_hi <= z_lo) return b->ctx->fail(VXG_INVALID_ARGUMENT, -1, "batch_set_slab: empty slab");
    b->slab_lo = z_lo;
    b->slab_hi = z_hi;
    return VXG_OK;
}

VXG_API vxg_status vxg_batch_from_plan(vxg_context* ctx, const vxg_segment* segs,
                                       const vxg_segment_plan* plans, int64_t n,
                                       int64_t max_steps, int64_t capacity, vxg_batch** out) {
    if (!ctx || !out) return VXG_INVALID_ARGUMENT;
    ctx->ok();
    *out = nullptr;
    // src/batch.cpp:98-105
    if (n <= 0 || !segs || !plans) return ctx->fail(VXG_LOGIC_ERROR, -1, "batch_voxelize: malformed plan");
    const vxg_segment_plan& last = plans[n - 1];
    if (last.output_offset + last.step_count + 1 != capacity)
        return ctx->fail(VXG_LOGIC_ERROR, -1, "batch_voxelize: plan capacity mismatch");
    // The reference checks only the last offset and the capacity. A max_steps above every N_i
    // only widens kernel_work_item's grid (its redundant items stay redundant), so it is kept as
    // given; one below some N_i would make the reference's kernel phase (k = 0..N_max) truncate
    // those chains, which this path does not reproduce: rejected as a malformed plan.
    int64_t mx = 0;
    for (int64_t i = 0; i < n; ++i) mx = std::max(mx, plans[i].step_count);
    if (mx > max_steps)
        return ctx->fail(VXG_LOGIC_ERROR, -1, "batch_voxelize: plan max_steps below a step count");
    cudaSetDevice(ctx->device);
    vxg_batch* b = nullptr;
    vxg_status s = new_batch(ctx, &b);
    if (s) return s;
    b->n = n;
    DBuf dplans;
    s = upload_segments(b, segs, n, VXG_MEM_HOST);
    if (!s && (!b->rec.ensure(ctx, sizeof(SegRec) * (size_t)n) ||
               !b->off.ensure(ctx, 8 * (size_t)(n + 1)) ||
               !dplans.ensure(ctx, sizeof(vxg_segment_plan) * (size_t)n)))
        s = ctx->fail(VXG_OUT_OF_MEMORY, -1, "batch_voxelize: out of device memory");
    if (!s) {
        cudaMemcpyAsync(dplans.p, plans, sizeof(vxg_segment_plan) * (size_t)n, cudaMemcpyHostToDevice,
                        ctx->stream);
        cudaMemcpyAsync(b->off.as<long long>() + n, &capacity, 8, cudaMemcpyHostToDevice, ctx->stream);
        cudaMemsetAsync(ctl_slot(b, 0), 0, sizeof(Control), ctx->stream);
        vxg::launch_pack_plan(b->d_segs, dplans.as<vxg_segment_plan>(), n, b->rec.as<SegRec>(),
                              b->off.as<long long>(), ctl_slot(b, 0),
                              ctx->stream);
        ctx->launches++;
        Control c;
        s = read_ctl(ctx, ctl_slot(b, 0), c, "batch_voxelize");
        if (s == VXG_LOGIC_ERROR) ctx->err = "batch_voxelize: malformed plan (offsets are not the prefix sum of N_i + 1)";
    }
    if (s) {
        delete b;
        return s;
    }
    b->max_steps = max_steps;
    b->capacity = capacity;
    *out = b;
    return VXG_OK;
}

// No synchronisation: the batch's buffers go back to the context cache, whose next user works
// on the same stream (stream order keeps the reuse safe; vxg_set_stream synchronises).
VXG_API void vxg_batch_destroy(vxg_batch* b) {
    if (!b) return;
    delete b;
}

VXG_API vxg_status vxg_batch_info(const vxg_batch* b, int64_t* n, int64_t* max_steps,
                                  int64_t* capacity) {
    if (!b) return VXG_INVALID_ARGUMENT;
    b->ctx->ok();
    const vxg_status s = plan_ready(const_cast<vxg_batch*>(b));
    if (s) return s;
    if (n) *n = b->n;
    if (max_steps) *max_steps = b->max_steps;
    if (capacity) *capacity = b->capacity;
    return VXG_OK;
}

VXG_API vxg_status vxg_batch_plans(vxg_batch* b, vxg_segment_plan* out) {
    if (!b || !out) return VXG_INVALID_ARGUMENT;
    vxg_context* ctx = b->ctx;
    ctx->ok();
    cudaSetDevice(ctx->device);
    if (const vxg_status s = plan_ready(b)) return s;
    DBuf d;
    if (!d.ensure(ctx, sizeof(vxg_segment_plan) * (size_t)b->n))
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "plans: out of device memory");
    vxg::launch_export_plans(b->rec.as<SegRec>(), b->off.as<long long>(), b->n,
                             d.as<vxg_segment_plan>(), ctx->stream);
    ctx->launches++;
    cudaError_t e = cudaMemcpyAsync(out, d.p, sizeof(vxg_segment_plan) * (size_t)b->n,
                                    cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    return e == cudaSuccess ? VXG_OK : ctx->cuda_fail(e, "plans readback");
}

VXG_API vxg_status vxg_batch_item_count(const vxg_batch* b, int64_t* live, int64_t* redundant) {
    if (!b) return VXG_INVALID_ARGUMENT;
    b->ctx->ok();
    if (const vxg_status s = plan_ready(const_cast<vxg_batch*>(b))) return s;
    if (live) *live = b->capacity;
    if (redundant) *redundant = b->n * (b->max_steps + 1) - b->capacity;
    return VXG_OK;
}

VXG_API vxg_status vxg_batch_work_item(vxg_batch* b, int64_t i, int64_t k, int32_t out[3],
                                       int* live) {
    if (!b || !out || !live) return VXG_INVALID_ARGUMENT;
    vxg_context* ctx = b->ctx;
    ctx->ok();
    if (const vxg_status s = plan_ready(b)) return s;
    if (i < 0 || i >= b->n || k < 0 || k > b->max_steps)
        return ctx->fail(VXG_OUT_OF_RANGE, -1,
                         "kernel_work_item: item index outside the %lld x %lld grid",
                         (long long)b->n, (long long)(b->max_steps + 1));
    cudaSetDevice(ctx->device);
    long long off2[2];
    cudaError_t e = cudaMemcpyAsync(off2, b->off.as<long long>() + i, 16, cudaMemcpyDeviceToHost,
                                    ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "kernel_work_item");
    if (k > off2[1] - off2[0] - 1) {
        *live = 0;
        return VXG_OK;
    }
    DBuf d;
    if (!d.ensure(ctx, 16)) return ctx->fail(VXG_OUT_OF_MEMORY, -1, "kernel_work_item: oom");
    cudaMemsetAsync(ctl_slot(b, 3), 0, sizeof(Control), ctx->stream);
    vxg::launch_work_item(b->rec.as<SegRec>(), b->off.as<long long>(), i, k, d.as<int32_t>(),
                          ctl_slot(b, 3), ctx->stream);
    ctx->launches++;
    cudaMemcpyAsync(out, d.p, 12, cudaMemcpyDeviceToHost, ctx->stream);
    Control c;
    const vxg_status s = read_ctl(ctx, ctl_slot(b, 3), c, "kernel_work_item");
    if (s) return s;
    *live = 1;
    return VXG_OK;
}

VXG_API vxg_status vxg_batch_emit_list(vxg_batch* b, vxg_voxel* out, int64_t out_cap,
                                       int64_t* chain_off, int64_t* total, vxg_mem where) {
    if (!b || !total || (!out && out_cap > 0) || !chain_off) return VXG_INVALID_ARGUMENT;
    vxg_context* ctx = b->ctx;
    ctx->ok();
    cudaSetDevice(ctx->device);
    const auto t0 = Clock::now();
    vxg_status s;
    if (where == VXG_MEM_DEVICE) {  // (a small batch's pending plan resolves in the emit's readback)
        s = emit_list_device(b, reinterpret_cast<int32_t*>(out), out_cap,
                             reinterpret_cast<long long*>(chain_off), total);
        b->timing.kernel_ns = ns_since(t0);
        b->timing.assemble_ns = 0;
        return s;
    }
    if ((s = plan_ready(b))) return s;
    if (!b->out.ensure(ctx, 12 * (size_t)std::max<int64_t>(b->capacity, 1)) ||
        !b->chain.ensure(ctx, 8 * (size_t)(b->n + 1)))
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "batch_voxelize: out of device memory");
    s = emit_list_device(b, b->out.as<int32_t>(), b->capacity, b->chain.as<long long>(), total);
    b->timing.kernel_ns = ns_since(t0);
    if (s) return s;
    if (*total > out_cap)
        return ctx->fail(VXG_LOGIC_ERROR, -1, "batch_voxelize: %lld voxels exceed the output capacity %lld",
                         (long long)*total, (long long)out_cap);
    const auto t1 = Clock::now();
    cudaError_t e = cudaMemcpyAsync(out, b->out.p, 12 * (size_t)*total, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(chain_off, b->chain.p, 8 * (size_t)(b->n + 1), cudaMemcpyDeviceToHost,
                            ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    b->timing.assemble_ns = ns_since(t1);
    return e == cudaSuccess ? VXG_OK : ctx->cuda_fail(e, "batch_voxelize readback");
}

VXG_API vxg_status vxg_batch_count_voxels(vxg_batch* b, int64_t* total) {
    if (!b || !total) return VXG_INVALID_ARGUMENT;
    b->ctx->ok();
    cudaSetDevice(b->ctx->device);
    return count_voxels_device(b, total);
}

VXG_API vxg_status vxg_batch_emit_bitmap(vxg_batch* b, uint64_t* words, int64_t V, int64_t z_lo,
                                         int64_t z_hi, int flags, int64_t* outside, vxg_mem where) {
    if (!b || !words || (flags & ~(VXG_BITMAP_CLIP | VXG_BITMAP_OVERWRITE))) return VXG_INVALID_ARGUMENT;
    const int clip = flags & VXG_BITMAP_CLIP;
    const bool overwrite = (flags & VXG_BITMAP_OVERWRITE) != 0;
    vxg_context* ctx = b->ctx;
    ctx->ok();
    if (const vxg_status s = plan_ready(b)) return s;
    if (V <= 0 || V > (1ll << 21) || z_lo < 0 || z_hi > V || z_lo > z_hi)
        return ctx->fail(VXG_INVALID_ARGUMENT, -1, "bitmap: invalid volume / slab");
    if ((V * V * (z_hi - z_lo) + 63) / 64 >= 0xffffffffll)  // word indices are 32-bit keys in-kernel
        return ctx->fail(VXG_INVALID_ARGUMENT, -1, "bitmap: slab larger than 2^32 words; split it");
    cudaSetDevice(ctx->device);
    const size_t nwords = (size_t)((V * V * (z_hi - z_lo) + 63) / 64);
    const auto t0 = Clock::now();
    if (where == VXG_MEM_DEVICE) {
        const vxg_status s = emit_bitmap_device(b, reinterpret_cast<unsigned long long*>(words), V,
                                                z_lo, z_hi, clip, outside, overwrite);
        b->timing.kernel_ns = ns_since(t0);
        return s;
    }
    DBuf d;
    if (!d.ensure(ctx, 8 * std::max<size_t>(nwords, 1)))
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "bitmap: out of device memory");
    // (overwrite on the tile path: the fill stores every word itself)
    if (!overwrite)
        cudaMemcpyAsync(d.p, words, 8 * nwords, cudaMemcpyHostToDevice, ctx->stream);
    // large slabs through the tile path: streamed readback (each finished z-layer of tiles goes
    // over PCIe while the fill continues)
    const char* smin = std::getenv("VXG_BITMAP_STREAM_MIN");  // bytes (tests lower it)
    if (use_tiles(b, V, z_lo, z_hi) && 8 * nwords >= (smin ? std::strtoull(smin, nullptr, 10) : (64ull << 20)) &&
        !std::getenv("VXG_BITMAP_NO_STREAM")) {
        const vxg_status s = emit_bitmap_tiles(b, d.as<unsigned long long>(), V, z_lo, z_hi,
                                               outside, words, overwrite);
        b->timing.kernel_ns = ns_since(t0);
        b->timing.assemble_ns = 0;
        return s;
    }
    vxg_status s = emit_bitmap_device(b, d.as<unsigned long long>(), V, z_lo, z_hi, clip, outside,
                                      overwrite);
    b->timing.kernel_ns = ns_since(t0);
    if (s) return s;
    const auto t1 = Clock::now();
    cudaError_t e = cudaMemcpyAsync(words, d.p, 8 * nwords, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    b->timing.assemble_ns = ns_since(t1);
    return e == cudaSuccess ? VXG_OK : ctx->cuda_fail(e, "bitmap readback");
}

VXG_API vxg_status vxg_select_slab_segments(vxg_context* ctx, const vxg_segment* segs, int64_t n,
                                            int64_t z_lo, int64_t z_hi, vxg_segment* out,
                                            int64_t* n_out) {
    if (!ctx || !segs || !out || !n_out || n < 0) return VXG_INVALID_ARGUMENT;
    ctx->ok();
    cudaSetDevice(ctx->device);
    *n_out = 0;
    if (n == 0) return VXG_OK;
    DBuf cnt;
    if (!cnt.ensure(ctx, sizeof(unsigned long long)))
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "select_slab_segments: out of device memory");
    cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), ctx->stream);
    vxg::launch_select_slab(reinterpret_cast<const double*>(segs), n, z_lo, z_hi,
                            reinterpret_cast<double*>(out), cnt.as<unsigned long long>(), ctx->stream);
    ctx->launches++;
    unsigned long long c = 0;
    cudaError_t e = cudaMemcpyAsync(ctx->h_ctl, cnt.p, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "select_slab_segments");
    std::memcpy(&c, ctx->h_ctl, sizeof(c));
    *n_out = (int64_t)c;
    return VXG_OK;
}

VXG_API vxg_status vxg_batch_slab_samples(vxg_batch* b, int64_t z_lo, int64_t z_hi,
                                          int64_t* samples) {
    if (!b || !samples) return VXG_INVALID_ARGUMENT;
    b->ctx->ok();
    cudaSetDevice(b->ctx->device);
    if (const vxg_status s = plan_ready(b)) return s;
    int64_t ne = 0;
    return run_clip(b, z_lo, z_hi, &ne, samples);
}

VXG_API vxg_status vxg_batch_timing(const vxg_batch* b, vxg_timing* t) {
    if (!b || !t) return VXG_INVALID_ARGUMENT;
    b->ctx->ok();
    if (const vxg_status s = plan_ready(const_cast<vxg_batch*>(b))) return s;
    t->preprocess_ns = (int64_t)((double)b->plan_ms * 1e6);
    t->kernel_ns = (int64_t)((double)b->emit_ms * 1e6);
    t->assemble_ns = (int64_t)((double)b->aux_ms * 1e6);
    return VXG_OK;
}

VXG_API vxg_status vxg_run_batch(vxg_context* ctx, const vxg_segment* segs, int64_t n,
                                 vxg_voxel* out, int64_t out_cap, int64_t* chain_off,
                                 int64_t* total, vxg_timing* timing) {
    if (!ctx) return VXG_INVALID_ARGUMENT;
    vxg_batch* b = nullptr;
    vxg_status s = vxg_batch_create(ctx, segs, n, VXG_MEM_HOST, &b);
    if (s) return s;
    s = vxg_batch_emit_list(b, out, out_cap, chain_off, total, VXG_MEM_HOST);
    if (timing) *timing = b->timing;
    vxg_batch_destroy(b);
    return s;
}

// ------------------------------------------------------------------------------- small batches
namespace {

// The multi-pass path for a batch the one-launch kernel handed back (a segment with N > 2^14).
vxg_status small_reroute(vxg_context* ctx, const vxg_segment* segs, int64_t n, vxg_voxel* out,
                         int64_t out_cap, int64_t* chain, int64_t* total, int64_t* max_steps,
                         int64_t* capacity) {
    vxg_batch* b = nullptr;
    vxg_status s = vxg_batch_create(ctx, segs, n, VXG_MEM_DEVICE, &b);
    if (s) return s;
    s = emit_list_device(b, reinterpret_cast<int32_t*>(out), out_cap,
                         reinterpret_cast<long long*>(chain), total);
    if (!s) {  // (the one-launch kernel's partials clamp N at 2^14 + 1: the plan's own values)
        if (max_steps) *max_steps = b->max_steps;
        if (capacity) *capacity = b->capacity;
    }
    vxg_batch_destroy(b);
    return s;
}

vxg_status small_result(vxg_context* ctx, int64_t* total, int64_t* max_steps, int64_t* capacity) {
    vxg_context::SmallState* st = ctx->small;
    st->pending = false;
    const int64_t calls = st->calls;
    st->calls = 0;
    cudaError_t e = cudaMemcpyAsync(st->h_ctl, st->ctl.p, sizeof(Control), cudaMemcpyDeviceToHost,
                                    ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "run_batch_device");
    const Control c = *st->h_ctl;
    if (c.n_entries && calls > 1)
        return ctx->fail(VXG_INVALID_ARGUMENT, -1,
                         "run_batch_device: a batch enqueued asynchronously holds a segment of more "
                         "than 2^14 steps (only the synchronous form re-routes it)");
    if (c.n_entries) {  // long segment: the multi-pass path
        int64_t t = 0;
        vxg_status s = small_reroute(ctx, st->segs, st->n, st->out, st->out_cap, st->chain, &t,
                                     max_steps, capacity);
        if (s) return s;
        if (total) *total = t;
        return VXG_OK;
    }
    // (plan errors first: they are batch_preprocess's; ctl_status reports the lowest segment)
    const vxg_status s = ctl_status(ctx, c, "run_batch");
    if (s) return s;
    if (total) *total = c.total;
    if (max_steps) *max_steps = (int64_t)c.max_steps;
    if (capacity) *capacity = (int64_t)c.pad0;
    return VXG_OK;
}

}  // namespace

extern "C" {

VXG_API vxg_status vxg_run_batch_device(vxg_context* ctx, const vxg_segment* segs, int64_t n,
                                        vxg_voxel* out, int64_t out_cap, int64_t* chain_off,
                                        int64_t* total) {
    if (!ctx) return VXG_INVALID_ARGUMENT;
    ctx->ok();
    if (n <= 0) return ctx->fail(VXG_INVALID_ARGUMENT, -1, "batch_preprocess: empty segment list");
    if (!segs || !chain_off || (!out && out_cap > 0))
        return ctx->fail(VXG_INVALID_ARGUMENT, -1, "run_batch_device: null buffer");
    if (!is_aligned16(segs) || (reinterpret_cast<uintptr_t>(out) & 3u))
        return ctx->fail(VXG_INVALID_ARGUMENT, -1, "run_batch_device: misaligned buffer");
    cudaSetDevice(ctx->device);
    if (!ctx->small) {
        ctx->small = new (std::nothrow) vxg_context::SmallState();
        if (!ctx->small) return ctx->fail(VXG_OUT_OF_MEMORY, -1, "run_batch_device: oom");
    }
    vxg_context::SmallState* st = ctx->small;
    // Asynchronous calls chain without synchronising: each resets only its own counters, while
    // the error words (and the long-segment flag) stay set until the result reads them. A
    // synchronous call first settles any pending ones.
    const bool chain = st->pending && !total;
    if (st->pending && total) {
        const vxg_status s = small_result(ctx, nullptr, nullptr, nullptr);
        if (s) return s;
    }
    if (!st->h_ctl &&
        cudaHostAlloc(reinterpret_cast<void**>(&st->h_ctl), sizeof(Control), cudaHostAllocDefault) !=
            cudaSuccess) {
        cudaGetLastError();
        st->h_ctl = nullptr;
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "run_batch_device: pinned memory");
    }
    int spw = vxg::small_spw(n, ctx->num_sms);
    if (const char* e = std::getenv("VXG_SMALL_SPW")) spw = std::atoi(e);  // (experiments)
    const long long ntiles = vxg::small_tile_count(n, spw);
    if (!st->status.ensure(ctx, sizeof(unsigned long long) * (size_t)ntiles) ||
        !st->ctl.ensure(ctx, sizeof(Control)))
        return ctx->fail(VXG_OUT_OF_MEMORY, -1, "run_batch_device: out of device memory");
    cudaMemsetAsync(st->status.p, 0, sizeof(unsigned long long) * (size_t)ntiles, ctx->stream);
    if (chain) {  // max_steps; pad0 (capacity), total, tile_counter -- not err_seg / n_entries / abort
        static_assert(offsetof(Control, err_seg) == 8 && offsetof(Control, pad0) == 16 &&
                      offsetof(Control, tile_counter) == 32, "Control layout");
        cudaMemsetAsync(st->ctl.p, 0, 8, ctx->stream);
        cudaMemsetAsync(static_cast<char*>(st->ctl.p) + 16, 0, 24, ctx->stream);
    } else {
        cudaMemsetAsync(st->ctl.p, 0, sizeof(Control), ctx->stream);
    }
    vxg::SmallArgs a{reinterpret_cast<const double*>(segs), n, ntiles,
                     reinterpret_cast<int32_t*>(out), out_cap,
                     reinterpret_cast<long long*>(chain_off),
                     st->status.as<unsigned long long>(), st->ctl.as<Control>(), spw};
    const cudaError_t e = vxg::launch_list_small(a, ctx->num_sms, ctx->stream);
    ctx->launches++;
    if (e != cudaSuccess) return ctx->cuda_fail(e, "list_small_kernel");
    st->pending = true;
    st->calls++;
    st->segs = segs;
    st->n = n;
    st->out = out;
    st->out_cap = out_cap;
    st->chain = chain_off;
    if (!total) return VXG_OK;
    return small_result(ctx, total, nullptr, nullptr);
}

VXG_API vxg_status vxg_run_batch_device_result(vxg_context* ctx, int64_t* total,
                                               int64_t* max_steps, int64_t* capacity) {
    if (!ctx) return VXG_INVALID_ARGUMENT;
    ctx->ok();
    if (!ctx->small || !ctx->small->pending)
        return ctx->fail(VXG_LOGIC_ERROR, -1, "run_batch_device_result: no call pending");
    cudaSetDevice(ctx->device);
    return small_result(ctx, total, max_steps, capacity);
}

}  // extern "C"

// ------------------------------------------------------------------------------- generators
VXG_API vxg_status vxg_gen_segments(vxg_context* ctx, int64_t n, const int64_t* lens,
                                    const uint64_t* seeds, int64_t len_fixed, int64_t len_max,
                                    int64_t V, uint64_t seed, vxg_segment* out, vxg_mem where) {
    if (!ctx || !out) return VXG_INVALID_ARGUMENT;
    ctx->ok();
    if (n < 1) return ctx->fail(VXG_INVALID_ARGUMENT, -1, "gen: need >= 1 segment");
    if (!lens && len_max <= 0 && len_fixed < 1)
        return ctx->fail(VXG_INVALID_ARGUMENT, -1, "gen_segment_of_length: target must be >= 1");
    cudaSetDevice(ctx->device);
    DBuf dout, dl, ds, dctl;
    double* d_out = reinterpret_cast<double*>(out);
    if (where == VXG_MEM_HOST) {
        if (!dout.ensure(ctx, 48 * (size_t)n)) return ctx->fail(VXG_OUT_OF_MEMORY, -1, "gen: oom");
        d_out = dout.as<double>();
    }
    const long long* d_lens = reinterpret_cast<const long long*>(lens);
    const unsigned long long* d_seeds = reinterpret_cast<const unsigned long long*>(seeds);
    if (lens && where == VXG_MEM_HOST) {
        if (!dl.ensure(ctx, 8 * (size_t)n) || !ds.ensure(ctx, 8 * (size_t)n))
            return ctx->fail(VXG_OUT_OF_MEMORY, -1, "gen: oom");
        cudaMemcpyAsync(dl.p, lens, 8 * (size_t)n, cudaMemcpyHostToDevice, ctx->stream);
        cudaMemcpyAsync(ds.p, seeds, 8 * (size_t)n, cudaMemcpyHostToDevice, ctx->stream);
        d_lens = dl.as<long long>();
        d_seeds = ds.as<unsigned long long>();
    }
    if (!dctl.ensure(ctx, sizeof(Control))) return ctx->fail(VXG_OUT_OF_MEMORY, -1, "gen: oom");
    cudaMemsetAsync(dctl.p, 0, sizeof(Control), ctx->stream);
    vxg::GenArgs a{n, d_lens, d_seeds, len_fixed, len_max, V, seed, d_out, dctl.as<Control>()};
    vxg::launch_gen(a, ctx->stream);
    ctx->launches++;
    if (where == VXG_MEM_HOST)
        cudaMemcpyAsync(out, d_out, 48 * (size_t)n, cudaMemcpyDeviceToHost, ctx->stream);
    Control c;
    vxg_status s = read_ctl(ctx, dctl.as<Control>(), c, "gen_segments");
    if (s == VXG_LOGIC_ERROR) ctx->err = "gen_segment_of_length: direction sampling failed";
    if (s == VXG_INVALID_ARGUMENT) ctx->err = "gen_segment_of_length: target must be >= 1 (and fit the volume)";
    return s;
}

VXG_API vxg_status vxg_gen_arbitrary_batch(vxg_context* ctx, int64_t total, int64_t count,
                                           uint64_t seed, vxg_segment* out) {
    if (!ctx || !out) return VXG_INVALID_ARGUMENT;
    ctx->ok();
    // src/bench.cpp:85-136: length planning on the host (glibc exp/log, as the reference), the
    // segments themselves on the GPU.
    if (count < 1) return ctx->fail(VXG_INVALID_ARGUMENT, -1, "gen_arbitrary_batch: need >= 1 segment");
    if (total < count)
        return ctx->fail(VXG_INVALID_ARGUMENT, -1,
                         "gen_arbitrary_batch: target %lld is infeasible for %lld segments of length >= 1",
                         (long long)total, (long long)count);
    uint64_t st = seed;
    auto next = [&]() {
        st += vxg::kGamma;
        return vxg::mix64(st);
    };
    auto uniform = [&](double lo, double hi) {
        volatile double u = (double)(next() >> 11) * 0x1.0p-53;
        volatile double span = hi - lo;
        volatile double prod = span * u;
        return lo + prod;
    };
    const double mean = (double)total / (double)count;
    const double log_hi = std::log(std::max(2.0 * mean, 2.0));
    std::vector<double> raw((size_t)count);
    double raw_sum = 0.0;
    for (double& r : raw) {
        r = std::exp(uniform(0.0, log_hi));
        raw_sum += r;
    }
    const double scale = (double)total / raw_sum;
    std::vector<int64_t> lens((size_t)count);
    std::vector<uint64_t> seeds((size_t)count);
    int64_t sum = 0;
    for (size_t i = 0; i < raw.size(); ++i) {
        volatile double x = raw[i] * scale;
        lens[i] = std::max<int64_t>(1, std::llround(x));
        sum += lens[i];
    }
    for (size_t i = 0; sum < total; i = (i + 1) % lens.size()) {
        ++lens[i];
        ++sum;
    }
    for (size_t i = 0; sum > total; i = (i + 1) % lens.size()) {
        if (lens[i] > 1) {
            --lens[i];
            --sum;
        }
    }
    for (auto& s : seeds) s = next();
    return vxg_gen_segments(ctx, count, lens.data(), seeds.data(), 0, 0, 0, 0, out, VXG_MEM_HOST);
}

}  // extern "C"
