// ref_wrapper.cpp -- flat extern "C" view of the UNMODIFIED reference implementation.
//
// TEST INFRASTRUCTURE. oracle/Makefile compiles this file together with the reference's own
// sources (/root/reference/proj/src/{geometry,parametric,batch,bench,formats}.cpp, read in place, never
// copied) into oracle/_ref/libref_voxline.so. It is used to (1) pin the C restatement in
// oracle/voxline_oracle.c, (2) generate tests/golden fixtures, and (3) serve as the CPU
// baseline ("kind": "reference") in bench.py. Exceptions are mapped to the codes in
// oracle/voxline_oracle.h.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include <fstream>
#include <sstream>

#include "voxline/batch.hpp"
#include "voxline/bench.hpp"
#include "voxline/formats.hpp"
#include "voxline/geometry.hpp"
#include "voxline/parametric.hpp"

namespace {

voxline::Segment seg_at(const double* p) {
    return {{p[0], p[1], p[2]}, {p[3], p[4], p[5]}};
}

std::vector<voxline::Segment> to_segments(const double* segs, int64_t n) {
    std::vector<voxline::Segment> v;
    v.reserve(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) v.push_back(seg_at(segs + 6 * i));
    return v;
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::range_error&) {
        return 2;
    } catch (const std::out_of_range&) {
        return 3;
    } catch (const std::logic_error&) {
        return 4;
    } catch (...) {
        return 5;
    }
}

}  // namespace

extern "C" {

int ref_round_point(const double p[3], int32_t out[3]) {
    return guarded([&] {
        const voxline::Voxel v = voxline::round_point({p[0], p[1], p[2]});
        out[0] = v.x;
        out[1] = v.y;
        out[2] = v.z;
    });
}

double ref_segment_length(const double seg[6]) { return voxline::segment_length(seg_at(seg)); }

int ref_make_plan(const double seg[6], int64_t* n, double w[3]) {
    return guarded([&] {
        const voxline::ParametricPlan p = voxline::make_plan(seg_at(seg));
        *n = p.step_count;
        w[0] = p.step_vector.x;
        w[1] = p.step_vector.y;
        w[2] = p.step_vector.z;
    });
}

int ref_voxelize_parametric(const double seg[6], int32_t* out, int64_t cap, int64_t* count) {
    return guarded([&] {
        const voxline::VoxelChain c = voxline::voxelize_parametric(seg_at(seg));
        *count = static_cast<int64_t>(c.voxels.size());
        if (out) {
            if (*count > cap) throw std::logic_error("cap");
            std::memcpy(out, c.voxels.data(), c.voxels.size() * sizeof(voxline::Voxel));
        }
    });
}

int ref_chain_length_bounds(const double seg[6], int64_t* lo, int64_t* hi) {
    return guarded([&] {
        const auto b = voxline::chain_length_bounds(seg_at(seg));
        *lo = b.first;
        *hi = b.second;
    });
}

int ref_batch_preprocess(const double* segs, int64_t n, int64_t* steps, double* w3,
                         int64_t* offsets, int64_t* max_steps, int64_t* capacity,
                         int64_t* live, int64_t* redundant) {
    return guarded([&] {
        const voxline::BatchPlan plan = voxline::batch_preprocess(to_segments(segs, n));
        for (int64_t i = 0; i < n; ++i) {
            const voxline::SegmentPlan& sp = plan.per_segment[static_cast<std::size_t>(i)];
            if (steps) steps[i] = sp.step_count;
            if (w3) {
                w3[3 * i + 0] = sp.step_vector.x;
                w3[3 * i + 1] = sp.step_vector.y;
                w3[3 * i + 2] = sp.step_vector.z;
            }
            if (offsets) offsets[i] = sp.output_offset;
        }
        *max_steps = plan.max_steps;
        *capacity = plan.total_voxel_capacity;
        const voxline::ItemCount c = voxline::effective_item_count(plan);
        if (live) *live = c.live;
        if (redundant) *redundant = c.redundant;
    });
}

int ref_kernel_work_item(const double* segs, int64_t n, int64_t i, int64_t k, int32_t out[3],
                         int* live) {
    return guarded([&] {
        const voxline::BatchPlan plan = voxline::batch_preprocess(to_segments(segs, n));
        const std::optional<voxline::Voxel> v = voxline::kernel_work_item(plan, i, k);
        *live = v.has_value() ? 1 : 0;
        if (v) {
            out[0] = v->x;
            out[1] = v->y;
            out[2] = v->z;
        }
    });
}

// run_batch flattened: chain i = out[chain_off[i] .. chain_off[i+1]). out may be NULL.
// timing_ns[3] = {preprocess, kernel, assemble}.
int ref_run_batch(const double* segs, int64_t n, int workers, int group_size, int32_t* out,
                  int64_t out_cap, int64_t* chain_off, int64_t* total, int64_t* timing_ns) {
    return guarded([&] {
        const voxline::BatchResult r =
            voxline::run_batch(to_segments(segs, n), {group_size, workers});
        int64_t acc = 0;
        for (std::size_t i = 0; i < r.chains.size(); ++i) {
            if (chain_off) chain_off[i] = acc;
            const auto& vox = r.chains[i].voxels;
            if (out) {
                if (acc + static_cast<int64_t>(vox.size()) > out_cap) throw std::logic_error("cap");
                std::memcpy(out + 3 * acc, vox.data(), vox.size() * sizeof(voxline::Voxel));
            }
            acc += static_cast<int64_t>(vox.size());
        }
        if (chain_off) chain_off[r.chains.size()] = acc;
        *total = r.total_voxels;
        if (timing_ns) {
            timing_ns[0] = r.timing.preprocess_ns;
            timing_ns[1] = r.timing.kernel_ns;
            timing_ns[2] = r.timing.assemble_ns;
        }
    });
}

// The bitmap configs' CPU arm: the reference's own run_batch (src/batch.cpp:154-162) over the
// segments, then the harness's bit-setting pass over its chains -- bit x + V*(y + V*(z - z_lo))
// of 64-bit words for voxels in [0,V)^2 x [z_lo, z_hi); voxels outside [0,V)^3 are counted in
// *outside. The pass runs on `workers` threads over contiguous chain ranges; a chain's run of
// voxels in one word is OR-ed in with one atomic. times_ns = {run_batch, bit-setting}.
int ref_run_batch_bitmap(const double* segs, int64_t n, int workers, int group_size,
                         uint64_t* words, int64_t V, int64_t z_lo, int64_t z_hi, int64_t* total,
                         int64_t* outside, int64_t* times_ns) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        const auto t0 = clk::now();
        const voxline::BatchResult r =
            voxline::run_batch(to_segments(segs, n), {group_size, workers});
        const auto t1 = clk::now();
        const std::size_t nc = r.chains.size();
        const int nt = std::max(1, workers);
        std::atomic<int64_t> out_total{0};
        auto body = [&](int t) {
            const std::size_t c0 = nc * (std::size_t)t / (std::size_t)nt;
            const std::size_t c1 = nc * (std::size_t)(t + 1) / (std::size_t)nt;
            int64_t out = 0;
            for (std::size_t c = c0; c < c1; ++c) {
                uint64_t cur_w = ~0ull, cur_b = 0;
                for (const voxline::Voxel& v : r.chains[c].voxels) {
                    if (v.x < 0 || v.x >= V || v.y < 0 || v.y >= V || v.z < 0 || v.z >= V) {
                        ++out;
                        continue;
                    }
                    if (v.z < z_lo || v.z >= z_hi) continue;
                    const uint64_t b = (uint64_t)v.x +
                                       (uint64_t)V * ((uint64_t)v.y + (uint64_t)V * (uint64_t)(v.z - z_lo));
                    if ((b >> 6) != cur_w) {
                        if (cur_b) __atomic_fetch_or(&words[cur_w], cur_b, __ATOMIC_RELAXED);
                        cur_w = b >> 6;
                        cur_b = 0;
                    }
                    cur_b |= 1ull << (b & 63);
                }
                if (cur_b) __atomic_fetch_or(&words[cur_w], cur_b, __ATOMIC_RELAXED);
            }
            out_total += out;
        };
        std::vector<std::thread> th;
        for (int t = 1; t < nt; ++t) th.emplace_back(body, t);
        body(0);
        for (auto& x : th) x.join();
        const auto t2 = clk::now();
        *total = r.total_voxels;
        if (outside) *outside = out_total.load();
        if (times_ns) {
            times_ns[0] = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
            times_ns[1] = std::chrono::duration_cast<std::chrono::nanoseconds>(t2 - t1).count();
        }
    });
}

// The reference harness's sequential method (src/bench.cpp:188-205): one voxelize_parametric
// call per segment on the calling thread; *total = the sum of chain lengths.
int ref_sequential_map(const double* segs, int64_t n, int64_t* total) {
    return guarded([&] {
        const std::vector<voxline::Segment> v = to_segments(segs, n);
        int64_t t = 0;
        for (const voxline::Segment& seg : v)
            t += static_cast<int64_t>(voxline::voxelize_parametric(seg).voxels.size());
        *total = t;
    });
}

int ref_gen_segment_of_length(int64_t target, uint64_t seed, double out[6]) {
    return guarded([&] {
        const voxline::Segment s = voxline::gen_segment_of_length(target, seed);
        const double v[6] = {s.start.x, s.start.y, s.start.z, s.end.x, s.end.y, s.end.z};
        std::memcpy(out, v, sizeof(v));
    });
}

int ref_gen_arbitrary_batch(int64_t total, int64_t count, uint64_t seed, double* out) {
    return guarded([&] {
        const std::vector<voxline::Segment> segs =
            voxline::gen_arbitrary_batch(total, count, seed);
        for (std::size_t i = 0; i < segs.size(); ++i) {
            const voxline::Segment& s = segs[i];
            const double v[6] = {s.start.x, s.start.y, s.start.z, s.end.x, s.end.y, s.end.z};
            std::memcpy(out + 6 * i, v, sizeof(v));
        }
    });
}

uint64_t ref_splitmix_next(uint64_t* state) {
    voxline::SplitMix64 r(*state);
    const uint64_t v = r.next();
    *state = r.state;
    return v;
}

double ref_compute_mvps(int64_t total, double ms, int* err) {
    double v = 0.0;
    *err = guarded([&] { v = voxline::compute_mvps(total, ms); });
    return v;
}

// read_segments_csv (src/formats.cpp:92-132) of a file: up to cap segments into out, the count
// in *n; on a malformed line returns 1 with the reference's message in msg (size msg_cap).
int ref_read_segments_csv(const char* path, double* out, int64_t cap, int64_t* n, char* msg,
                          int64_t msg_cap) {
    if (msg && msg_cap > 0) msg[0] = 0;
    try {
        std::ifstream in(path);
        const std::vector<voxline::Segment> v = voxline::read_segments_csv(in);
        *n = static_cast<int64_t>(v.size());
        for (int64_t i = 0; i < *n && i < cap; ++i) {
            const voxline::Segment& s = v[static_cast<std::size_t>(i)];
            const double q[6] = {s.start.x, s.start.y, s.start.z, s.end.x, s.end.y, s.end.z};
            std::memcpy(out + 6 * i, q, sizeof q);
        }
        return 0;
    } catch (const std::invalid_argument& e) {
        if (msg && msg_cap > 0) {
            std::strncpy(msg, e.what(), static_cast<std::size_t>(msg_cap - 1));
            msg[msg_cap - 1] = 0;
        }
        return 1;
    } catch (...) {
        return 5;
    }
}

// The CLI's batch output (tools/voxline_cli.cpp:101-129 + 46-70): run_batch, then
// write_vox3_multi (format 0) or write_xyz_multi (format 1) to path.
int ref_batch_write(const double* segs, int64_t n, const char* path, int format) {
    return guarded([&] {
        const voxline::BatchResult r = voxline::run_batch(to_segments(segs, n), {64, 1});
        std::vector<std::vector<voxline::Voxel>> chains;
        chains.reserve(r.chains.size());
        for (const auto& c : r.chains) chains.push_back(c.voxels);
        std::ofstream out(path, std::ios::binary);
        if (format == 1) voxline::write_xyz_multi(out, chains);
        else voxline::write_vox3_multi(out, chains);
    });
}

}  // extern "C"
