// voxline_gpu_core.cpp -- the reference's C++ hot-path API, re-pointed at the B200 path.
//
// Implements, with the reference's own headers (compiled with -I /root/reference/proj/include,
// never copied), exactly the functions of the parametric hot path:
//
//   include/voxline/parametric.hpp:35-56   make_plan, voxelize_parametric, chain_length_bounds
//                                          (replaces src/parametric.cpp:8-50)
//   include/voxline/batch.hpp:59-87        batch_preprocess, kernel_work_item, batch_voxelize,
//                                          run_batch, effective_item_count
//                                          (replaces src/batch.cpp:23-170)
//
// Every voxel is computed on the GPU through the C ABI of libvoxgpu.so (include/voxgpu.h); this
// file only marshals std:: containers and turns vxg_status codes back into the exception classes
// the reference throws. The rest of the reference (geometry.cpp, walk.cpp,
// bench.cpp, formats.cpp, bindings/pybind_module.cpp, tests/acceptance_main.cpp) links against
// this translation unit UNCHANGED (integration/Makefile), which is the drop-in claim.
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "voxline/batch.hpp"
#include "voxline/parametric.hpp"

#include "voxgpu.h"

static_assert(sizeof(voxline::Segment) == sizeof(vxg_segment), "Segment layout");
static_assert(sizeof(voxline::Voxel) == sizeof(vxg_voxel), "Voxel layout");
static_assert(sizeof(voxline::SegmentPlan) == sizeof(vxg_segment_plan), "SegmentPlan layout");

namespace {

using Clock = std::chrono::steady_clock;

std::int64_t ns_between(Clock::time_point a, Clock::time_point b) {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(b - a).count();
}

// One context per host thread (the reference functions are re-entrant): each
// thread gets its own stream, staging and device cache, so concurrent callers never serialise on
// a shared context. VXG_DEVICE selects the GPU (default 0).
struct CtxHolder {
    vxg_context* ctx = nullptr;
    ~CtxHolder() {
        if (ctx) vxg_destroy(ctx);
    }
};

vxg_context* ctx() {
    thread_local CtxHolder h;
    if (!h.ctx) {
        const char* dev = std::getenv("VXG_DEVICE");
        const vxg_status s = vxg_create(dev ? std::atoi(dev) : 0, &h.ctx);
        if (s != VXG_OK)
            throw std::runtime_error("voxline (B200): no usable CUDA device for libvoxgpu (status " +
                                     std::to_string((int)s) + "); there is no CPU fallback");
    }
    return h.ctx;
}

// vxg_status -> the reference's exception class (src/geometry.cpp:16-26, src/batch.cpp:58-105).
void check(vxg_status s) {
    if (s == VXG_OK) return;
    const std::string msg = vxg_last_error(ctx());
    switch (s) {
        case VXG_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case VXG_RANGE_ERROR: throw std::range_error(msg);
        case VXG_OUT_OF_RANGE: throw std::out_of_range(msg);
        case VXG_LOGIC_ERROR: throw std::logic_error(msg);
        case VXG_OUT_OF_MEMORY: throw std::bad_alloc();
        default: throw std::runtime_error(msg);
    }
}

const vxg_segment* as_vxg(const voxline::Segment* s) {
    return reinterpret_cast<const vxg_segment*>(s);
}

struct BatchHandle {
    vxg_batch* b = nullptr;
    ~BatchHandle() {
        if (b) vxg_batch_destroy(b);
    }
};

// Device batch of a caller-supplied plan (batch_voxelize / kernel_work_item take a BatchPlan by
// const reference; the reference validates it at src/batch.cpp:93-105).
void upload_plan(const voxline::BatchPlan& plan, BatchHandle& h) {
    check(vxg_batch_from_plan(ctx(), as_vxg(plan.segments.data()),
                              reinterpret_cast<const vxg_segment_plan*>(plan.per_segment.data()),
                              (int64_t)plan.segments.size(), plan.max_steps,
                              plan.total_voxel_capacity, &h.b));
}

}  // namespace

namespace voxline {

// ------------------------------------------------------------------ parametric.hpp
ParametricPlan make_plan(const Segment& seg) {
    int64_t n = 0;
    double w[3] = {0.0, 0.0, 0.0};
    check(vxg_make_plans(ctx(), as_vxg(&seg), 1, &n, w));
    return {n, {w[0], w[1], w[2]}};
}

VoxelChain voxelize_parametric(const Segment& seg) {
    VoxelChain chain;
    chain.source = seg;
    std::vector<Voxel> buf(4096);
    for (;;) {
        int64_t count = 0;
        const vxg_status s = vxg_voxelize_parametric(
            ctx(), as_vxg(&seg), reinterpret_cast<vxg_voxel*>(buf.data()), (int64_t)buf.size(), &count);
        if (s == VXG_LOGIC_ERROR && count > (int64_t)buf.size()) {  // chain longer than the buffer
            buf.resize((size_t)count);
            continue;
        }
        check(s);
        buf.resize((size_t)count);
        chain.voxels = std::move(buf);
        return chain;
    }
}

std::pair<std::int64_t, std::int64_t> chain_length_bounds(const Segment& seg) {
    int64_t lo = 0, hi = 0;
    check(vxg_chain_length_bounds(ctx(), as_vxg(&seg), &lo, &hi));
    return {lo, hi};
}

// ------------------------------------------------------------------ batch.hpp
BatchPlan batch_preprocess(const std::vector<Segment>& segments) {
    if (segments.empty()) throw std::invalid_argument("batch_preprocess: empty segment list");
    BatchHandle h;
    check(vxg_batch_create(ctx(), as_vxg(segments.data()), (int64_t)segments.size(), VXG_MEM_HOST,
                           &h.b));
    BatchPlan plan;
    plan.segments = segments;
    plan.per_segment.resize(segments.size());
    check(vxg_batch_plans(h.b, reinterpret_cast<vxg_segment_plan*>(plan.per_segment.data())));
    int64_t n = 0;
    check(vxg_batch_info(h.b, &n, &plan.max_steps, &plan.total_voxel_capacity));
    return plan;
}

std::optional<Voxel> kernel_work_item(const BatchPlan& plan, std::int64_t segment_index,
                                      std::int64_t k) {
    const auto count = static_cast<std::int64_t>(plan.segments.size());
    if (segment_index < 0 || segment_index >= count || k < 0 || k > plan.max_steps)
        throw std::out_of_range("kernel_work_item: item index outside the " +
                                std::to_string(count) + " x " +
                                std::to_string(plan.max_steps + 1) + " grid");
    const SegmentPlan& sp = plan.per_segment[(size_t)segment_index];
    if (k > sp.step_count) return std::nullopt;  // redundant item
    // One item: the reference's own inline parametric_sample (include/voxline/parametric.hpp:
    // 41-48) and round_point (src/geometry.cpp, linked unchanged) over the plan the GPU made --
    // src/batch.cpp:86-89 verbatim in effect; a device round trip per item would cost ~100 us.
    return round_point(
        parametric_sample(plan.segments[(size_t)segment_index],
                          ParametricPlan{sp.step_count, sp.step_vector}, k));
}

namespace {
// Per-thread pinned staging for batch_voxelize's list (grown, never shrunk): pinning is a
// per-call cost of milliseconds per GB, so it is paid once per thread, not once per call.
struct PinnedCache {
    void* p = nullptr;
    size_t bytes = 0;
    ~PinnedCache() { vxg_host_free(p); }
    void* ensure(size_t b) {
        if (b <= bytes) return p;
        vxg_host_free(p);
        const size_t grow = b + b / 4;
        p = vxg_host_alloc(grow);
        bytes = p ? grow : 0;
        if (!p) throw std::bad_alloc();
        return p;
    }
};
thread_local PinnedCache t_vox, t_off;
}  // namespace

BatchResult batch_voxelize(const BatchPlan& plan, const PartitionConfig& cfg) {
    if (cfg.group_size < 1 || cfg.worker_count < 1)
        throw std::invalid_argument("batch_voxelize: group_size and worker_count must be >= 1");
    if (plan.segments.empty() || plan.per_segment.size() != plan.segments.size())
        throw std::logic_error("batch_voxelize: malformed plan");
    const SegmentPlan& last = plan.per_segment.back();
    if (last.output_offset + last.step_count + 1 != plan.total_voxel_capacity)
        throw std::logic_error("batch_voxelize: plan capacity mismatch");
    // The partitioning (cfg) cannot change the output: the GPU grid replaces the worker pool.
    BatchResult result;
    BatchHandle h;
    upload_plan(plan, h);
    const size_t n = plan.segments.size();
    const auto k0 = Clock::now();
    // flat list + chain offsets straight into this thread's cached pinned staging (one D2H
    // each). The list needs room for total_voxels, not the capacity: when the cache is smaller
    // than the capacity, the voxel count comes first (the count pass alone).
    int64_t need = plan.total_voxel_capacity;
    if (t_vox.bytes < sizeof(Voxel) * (size_t)std::max<int64_t>(need, 1))
        check(vxg_batch_count_voxels(h.b, &need));
    void* vp = t_vox.ensure(sizeof(Voxel) * (size_t)std::max<int64_t>(need, 1));
    void* op = t_off.ensure(sizeof(int64_t) * (n + 1));
    int64_t total = 0;
    check(vxg_batch_emit_list(h.b, static_cast<vxg_voxel*>(vp), need, static_cast<int64_t*>(op),
                              &total, VXG_MEM_HOST));
    const auto k1 = Clock::now();
    result.timing.kernel_ns = ns_between(k0, k1);
    // assemble: the chains the API returns by value (std::vector per segment)
    const Voxel* v = static_cast<const Voxel*>(vp);
    const int64_t* o = static_cast<const int64_t*>(op);
    result.chains.resize(n);
    for (size_t i = 0; i < n; ++i) {
        VoxelChain& c = result.chains[i];
        c.source = plan.segments[i];
        c.voxels.assign(v + o[i], v + o[i + 1]);
    }
    result.total_voxels = total;
    result.timing.assemble_ns = ns_between(k1, Clock::now());
    return result;
}

BatchResult run_batch(const std::vector<Segment>& segments, const PartitionConfig& cfg) {
    const auto t0 = Clock::now();
    const BatchPlan plan = batch_preprocess(segments);
    const auto t1 = Clock::now();
    BatchResult result = batch_voxelize(plan, cfg);
    result.timing.preprocess_ns = ns_between(t0, t1);
    return result;
}

ItemCount effective_item_count(const BatchPlan& plan) {
    ItemCount c;
    c.live = plan.total_voxel_capacity;
    c.redundant = static_cast<std::int64_t>(plan.segments.size()) * (plan.max_steps + 1) - c.live;
    return c;
}

}  // namespace voxline
