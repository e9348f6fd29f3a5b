// vxg_kernels.cu -- the B200 hot path: plan + look-back offset scan, thread-per-sample emit
// (voxel list with in-kernel dedup + single-pass compaction, or occupancy bitmap), z-slab
// k-range clipping, and the synthetic-input generator.
//
// Reference semantics (paths relative to /root/reference/proj):
//   make_plan            src/parametric.cpp:8-26        -> plan_kernel / plan_clip_kernel
//   batch_preprocess     src/batch.cpp:57-73            -> plan_kernel (offsets via look-back)
//   kernel phase         src/batch.cpp:107-126          -> emit_list_kernel (no N_max grid:
//                                                          the flat sample space is tiled)
//   assemble phase       src/batch.cpp:128-150          -> fused into emit_list_kernel
//   parametric_sample    include/voxline/parametric.hpp:41-48
//   round_point          src/geometry.cpp:15-34
//   gen_segment_of_length src/bench.cpp:62-83           -> gen_kernel
#include <cstdint>
#include <cstdio>

#include "vxg_device.cuh"
#include "vxg_internal.h"

namespace vxg {

// =============================================================================== plan kernel
// One tile = BLOCK*IPT segments. Segments are read striped (coalesced), the (N_i + 1) counts are
// transposed through shared memory into a blocked arrangement for the in-order scan, and the
// tile prefix comes from the decoupled look-back. Outputs: rec[i], steps[i], offsets[0..n].
template <int BLOCK, int IPT>
__global__ void __launch_bounds__(BLOCK) plan_kernel(PlanArgs a) {
    constexpr int TN = BLOCK * IPT;
    __shared__ long long s_cnt[TN];
    __shared__ long long s_warp[BLOCK / 32 + 1];
    __shared__ long long s_tile, s_prefix;
    const int tid = threadIdx.x;
    if (tid == 0) s_tile = (long long)atomicAdd(&a.ctl->tile_counter, 1ull);
    __syncthreads();
    const long long tile = s_tile;
    const long long base = tile * TN;

    unsigned long long mx = 0;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
        const long long i = base + (long long)q * BLOCK + tid;
        long long cnt = 0;
        if (i < a.n) {
            const double2* p = reinterpret_cast<const double2*>(a.segs + 6 * i);
            const double2 a0 = p[0], a1 = p[1], a2 = p[2];
            const double sx = a0.x, sy = a0.y, sz = a1.x, ex = a1.y, ey = a2.x, ez = a2.y;
            Plan pl;
            if (!make_plan(sx, sy, sz, ex, ey, ez, pl)) record_error(a.ctl, i, 2);
            SegRec r;
            r.sx = sx;
            r.sy = sy;
            r.sz = sz;
            r.wx = pl.wx;
            r.wy = pl.wy;
            r.wz = pl.wz;
            r.ex = pl.ex;
            r.ey = pl.ey;
            r.ez = pl.ez;
            r.flags = rec_flags(sx, sy, sz, ex, ey, ez);
            a.rec[i] = r;
            cnt = pl.n + 1;
            mx = (unsigned long long)pl.n > mx ? (unsigned long long)pl.n : mx;
        }
        s_cnt[q * BLOCK + tid] = cnt;
    }
    // N_max: warp max, block max in shared memory, one global atomic per tile (a per-warp
    // atomic on the single counter serialises in L2: 2M of them for 64M segments)
    __shared__ unsigned long long s_max;
    if (tid == 0) s_max = 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = t > mx ? t : mx;
    }
    __syncthreads();
    if ((tid & 31) == 0 && mx) atomicMax(&s_max, mx);
    __syncthreads();
    if (tid == 0 && s_max) atomicMax(&a.ctl->max_steps, s_max);

    long long local[IPT];
    long long sum = 0;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
        local[q] = s_cnt[tid * IPT + q];
        sum += local[q];
    }
    long long agg;
    const long long excl = block_excl_scan<BLOCK>(sum, s_warp, agg);
    if (tid < 32) {
        const long long pre = lookback_warp(a.status, tile, agg, a.ctl);
        if (tid == 0) s_prefix = pre;
    }
    __syncthreads();
    long long run = s_prefix + excl;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
        s_cnt[tid * IPT + q] = run;
        run += local[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
        const long long i = base + (long long)q * BLOCK + tid;
        if (i < a.n) a.offsets[i] = s_cnt[q * BLOCK + tid];
    }
    if (base + TN >= a.n && tid == 0) {  // last tile: capacity
        const long long cap = s_prefix + agg;
        a.offsets[a.n] = cap;
        a.ctl->total = cap;
    }
}

// =============================================================================== tile index
// tile_seg[t] = the entry containing flat sample t*TS (entries with zero samples write nothing).
__global__ void tile_index_kernel(const long long* __restrict__ off, long long n_entries,
                                  int ts_log2, long long* __restrict__ tile_seg) {
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_entries) return;
    const long long o = off[c], e = off[c + 1];
    if (e <= o) return;
    const long long ts = 1ll << ts_log2;
    const long long t_first = (o + ts - 1) >> ts_log2;
    const long long t_last = (e - 1) >> ts_log2;
    for (long long t = t_first; t <= t_last; ++t) tile_seg[t] = c;
}

// =============================================================================== clip
// z-slab partitioner: for every segment, the k-range whose rounded z lies in [z_lo, z_hi).
// For k < N, z_k = fl(S.z + fl(W.z*k)) is monotone in k (both roundings are monotone), so
// round(z_k) is monotone and the in-slab set is one interval [ka, kb) found by an analytic
// guess plus exact fix-up (binary search fallback). The k = N sample is E and is handled on
// its own (it need not continue the interval under rounding). Segments with no in-slab sample
// are compacted away: entry indices and sample offsets come from two look-back scans.
__device__ __forceinline__ long long zround(const SegRec& r, long long k) {
    return (long long)round_fast(sample_axis(r.sz, r.wz, __ll2double_rn(k)));
}

// first k in [0, N) with pred(k) (monotone false -> true), N if none.
// dir > 0: pred(k) = round(z_k) >= B; dir < 0: pred(k) = round(z_k) < B.
__device__ __forceinline__ long long first_cross(const SegRec& r, long long N, long long B,
                                                 int dir) {
    auto pred = [&](long long k) {
        const long long zr = zround(r, k);
        return dir > 0 ? zr >= B : zr < B;
    };
    if (N <= 0) return N;
    long long g;
    if (r.wz == 0.0) {
        g = pred(0) ? 0 : N;
        return g;
    }
    double gd = __ddiv_rn(__dsub_rn(__dsub_rn((double)B, 0.5), r.sz), r.wz);
    gd = fmin(fmax(ceil(gd), 0.0), (double)N);
    g = (long long)gd;
    int steps = 0;
    while (g > 0 && pred(g - 1) && steps < 4) {
        --g;
        ++steps;
    }
    while (g < N && !pred(g) && steps < 8) {
        ++g;
        ++steps;
    }
    const bool ok = (g == N || pred(g)) && (g == 0 || !pred(g - 1));
    if (ok) return g;
    long long lo = 0, hi = N;  // exact fallback
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (pred(mid)) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

template <int BLOCK, int IPT>
__global__ void __launch_bounds__(BLOCK) clip_kernel(ClipArgs a) {
    constexpr int TN = BLOCK * IPT;
    __shared__ long long s_cnt[TN];
    __shared__ long long s_nz[TN];
    __shared__ long long s_warp[BLOCK / 32 + 1];
    __shared__ long long s_tile, s_pre_s, s_pre_e, s_agg_s, s_agg_e;
    const int tid = threadIdx.x;
    if (tid == 0) s_tile = (long long)atomicAdd(&a.ctl->tile_counter, 1ull);
    __syncthreads();
    const long long tile = s_tile;
    const long long base = tile * TN;
    long long kas[IPT], kbs[IPT], ns[IPT], cnts[IPT];
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
        const long long i = base + (long long)q * BLOCK + tid;
        long long cnt = 0;
        kas[q] = kbs[q] = ns[q] = 0;
        if (i < a.n) {
            const SegRec r = load_rec(a.rec + i);
            const long long N = a.off[i + 1] - a.off[i] - 1;
            long long ka, kb;
            if (r.wz >= 0.0) {
                ka = first_cross(r, N, a.z_lo, +1);
                kb = first_cross(r, N, a.z_hi, +1);
            } else {
                ka = first_cross(r, N, a.z_hi, -1);
                kb = first_cross(r, N, a.z_lo, -1);
            }
            if (kb < ka) kb = ka;
            const bool e_in = r.ez >= a.z_lo && r.ez < a.z_hi;
            cnt = (kb - ka) + (e_in ? 1 : 0);
            kas[q] = ka;
            kbs[q] = kb;
            ns[q] = N;
        }
        cnts[q] = cnt;
        s_cnt[q * BLOCK + tid] = cnt;
        s_nz[q * BLOCK + tid] = cnt > 0 ? 1 : 0;
    }
    __syncthreads();
    long long lc[IPT], ln[IPT];
    long long sc = 0, sn = 0;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
        lc[q] = s_cnt[tid * IPT + q];
        ln[q] = s_nz[tid * IPT + q];
        sc += lc[q];
        sn += ln[q];
    }
    long long agg_s, agg_e;
    const long long ex_s = block_excl_scan<BLOCK>(sc, s_warp, agg_s);
    __syncthreads();
    const long long ex_e = block_excl_scan<BLOCK>(sn, s_warp, agg_e);
    if (tid < 32) {
        const long long ps = lookback_warp(a.status, tile, agg_s, a.ctl);
        const long long pe = lookback_warp(a.status2, tile, agg_e, a.ctl);
        if (tid == 0) {
            s_pre_s = ps;
            s_pre_e = pe;
            s_agg_s = agg_s;
            s_agg_e = agg_e;
        }
    }
    __syncthreads();
    long long rs = s_pre_s + ex_s, re = s_pre_e + ex_e;
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
        s_cnt[tid * IPT + q] = rs;
        s_nz[tid * IPT + q] = re;
        rs += lc[q];
        re += ln[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
        const long long i = base + (long long)q * BLOCK + tid;
        if (i < a.n && cnts[q] > 0) {
            const long long e = s_nz[q * BLOCK + tid];
            ClipEntry ce;
            ce.seg = i;
            ce.ka = kas[q];
            ce.kb = kbs[q];
            ce.n = ns[q];
            a.entries[e] = ce;
            a.ent_off[e] = s_cnt[q * BLOCK + tid];
        }
    }
    if (base + TN >= a.n && tid == 0) {
        const long long ne = s_pre_e + s_agg_e;
        const long long ts = s_pre_s + s_agg_s;
        a.ent_off[ne] = ts;
        a.ctl->total = ts;
        a.ctl->n_entries = ne;
    }
}

// =============================================================================== small kernels
__global__ void round_points_kernel(const double* __restrict__ p, long long n,
                                    int32_t* __restrict__ out, Control* ctl) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t v[3];
    bool ok = true;
    for (int d = 0; d < 3; ++d) ok &= round_checked(p[3 * i + d], v[d]);
    if (!ok) record_error(ctl, i, 2);
    for (int d = 0; d < 3; ++d) out[3 * i + d] = v[d];
}

__global__ void segment_lengths_kernel(const double* __restrict__ s, long long n,
                                       double* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* q = s + 6 * i;
    const double dx = __dsub_rn(q[3], q[0]), dy = __dsub_rn(q[4], q[1]), dz = __dsub_rn(q[5], q[2]);
    out[i] = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

// BatchPlan::per_segment export (vxg_segment_plan AoS, 40 B).
__global__ void export_plans_kernel(const SegRec* __restrict__ rec, const long long* __restrict__ off,
                                    long long n, vxg_segment_plan* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const SegRec r = rec[i];
    vxg_segment_plan p;
    p.output_offset = off[i];
    p.step_count = off[i + 1] - off[i] - 1;
    p.wx = r.wx;
    p.wy = r.wy;
    p.wz = r.wz;
    out[i] = p;
}

// The z-slab filter (vxg_select_slab_segments): segments whose endpoints' z range, widened by 2
// planes (every sample lies between S and E up to rounding), meets [z_lo, z_hi); one list
// append per block.
__global__ void __launch_bounds__(256) select_slab_kernel(const double* __restrict__ segs,
                                                          long long n, long long z_lo,
                                                          long long z_hi, double* __restrict__ out,
                                                          unsigned long long* count) {
    __shared__ unsigned s_cnt[8];
    __shared__ unsigned long long s_base;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool keep = false;
    double2 a0 = make_double2(0, 0), a1 = a0, a2 = a0;
    if (i < n) {
        const double2* p = reinterpret_cast<const double2*>(segs + 6 * i);
        a0 = p[0];
        a1 = p[1];
        a2 = p[2];
        const double sz = a1.x, ez = a2.y;
        const double lo = fmin(sz, ez), hi = fmax(sz, ez);
        // any non-finite coordinate: keep it (the plan reports it, as on every rank)
        const bool finite = isfinite(a0.x) && isfinite(a0.y) && isfinite(a1.x) &&
                            isfinite(a1.y) && isfinite(a2.x) && isfinite(a2.y);
        keep = !finite || (hi + 2.0 >= (double)z_lo && lo - 2.0 < (double)z_hi);
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_cnt[warp] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned tot = 0;
        for (int w = 0; w < 8; ++w) {
            const unsigned c = s_cnt[w];
            s_cnt[w] = tot;
            tot += c;
        }
        s_base = tot ? atomicAdd(count, (unsigned long long)tot) : 0ull;
    }
    __syncthreads();
    if (keep) {
        double2* q = reinterpret_cast<double2*>(out + 6 * (s_base + s_cnt[warp] +
                                                             __popc(m & ((1u << lane) - 1u))));
        q[0] = a0;
        q[1] = a1;
        q[2] = a2;
    }
}

void launch_select_slab(const double* segs, long long n, long long z_lo, long long z_hi,
                        double* out, unsigned long long* count, cudaStream_t s) {
    select_slab_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(segs, n, z_lo, z_hi, out, count);
}

// A plan given by the caller (batch_voxelize(const BatchPlan&)): build records, check offsets
// are the exclusive prefix of N_i + 1 (src/batch.cpp:98-105 checks only the last one).
__global__ void pack_plan_kernel(const double* __restrict__ segs,
                                 const vxg_segment_plan* __restrict__ plans, long long n,
                                 SegRec* __restrict__ rec, long long* __restrict__ off,
                                 Control* ctl) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* s = segs + 6 * i;
    const vxg_segment_plan p = plans[i];
    SegRec r;
    r.sx = s[0];
    r.sy = s[1];
    r.sz = s[2];
    r.wx = p.wx;
    r.wy = p.wy;
    r.wz = p.wz;
    bool ok = round_checked(s[3], r.ex) & round_checked(s[4], r.ey) & round_checked(s[5], r.ez);
    if (!ok) record_error(ctl, i, 2);
    // W supplied by the caller: bound |S + W*k| through |S| + |W|*N instead of |E|
    const double nd = (double)p.step_count;
    const double mx = fmax(fmax(fabs(s[0]) + fabs(p.wx) * nd, fabs(s[1]) + fabs(p.wy) * nd),
                           fabs(s[2]) + fabs(p.wz) * nd);
    // caller-supplied W: checked rounding unless provably in range, always the exact duplicate
    // test (the packed-key comparison relies on neighbouring samples -- E included -- lying
    // within 2 voxels of each other, which only the plan kernel's own W guarantees), and never
    // the positive-rounding shortcut (samples need not lie between S and E)
    r.flags = ((mx > kCheckThreshold || !(mx == mx)) ? REC_CHECK : 0u) |
              (rec_flags(s[0], s[1], s[2], s[3], s[4], s[5]) & REC_CHECK) | REC_WIDE;
    rec[i] = r;
    off[i] = p.output_offset;
    if (p.step_count < 0) record_error(ctl, i, 4);
    if (i > 0 && plans[i - 1].output_offset + plans[i - 1].step_count + 1 != p.output_offset)
        record_error(ctl, i, 4);
    if (i == 0 && p.output_offset != 0) record_error(ctl, 0, 4);
}

// kernel_work_item (src/batch.cpp:75-90) for one (i, k) on device.
__global__ void work_item_kernel(const SegRec* __restrict__ rec, const long long* __restrict__ off,
                                 long long i, long long k, int32_t* __restrict__ out, Control* ctl) {
    const SegRec r = rec[i];
    const long long N = off[i + 1] - off[i] - 1;
    int32_t x, y, z;
    bool b = false;
    SegRec rc = r;
    rc.flags |= REC_CHECK;
    eval_sample(rc, k, N, x, y, z, b);
    if (b) record_error(ctl, i, 2);
    out[0] = x;
    out[1] = y;
    out[2] = z;
}

// =============================================================================== generator
// gen_segment_of_length (src/bench.cpp:62-83) and the volume-fitted variant; bit-identical to
// oracle/voxline_oracle.c (same SplitMix64 draws, same FMA-free arithmetic).
__device__ __forceinline__ void sphere_dir(SplitMix& rng, double d[3]) {
    for (;;) {
        const double u = rng.uniform(-1.0, 1.0);
        const double v = rng.uniform(-1.0, 1.0);
        const double s = __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v));
        if (s >= 1.0 || s == 0.0) continue;
        const double f = __dmul_rn(2.0, __dsqrt_rn(__dsub_rn(1.0, s)));
        d[0] = __dmul_rn(u, f);
        d[1] = __dmul_rn(v, f);
        d[2] = __dsub_rn(1.0, __dmul_rn(2.0, s));
        return;
    }
}

__global__ void gen_kernel(GenArgs a) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    long long L;
    uint64_t seed;
    if (a.lens) {
        L = a.lens[i];
        seed = a.seeds[i];
    } else if (a.len_max > 0) {
        L = 1 + (long long)(splitmix_draw(a.seed, 2ull * (uint64_t)i) % (uint64_t)a.len_max);
        seed = splitmix_draw(a.seed, 2ull * (uint64_t)i + 1ull);
    } else {
        L = a.len_fixed;
        seed = splitmix_draw(a.seed, (uint64_t)i);
    }
    double* out = a.out + 6 * i;
    if (L < 1) {
        record_error(a.ctl, i, 1);
        return;
    }
    SplitMix rng{seed};
    const double dist = __dadd_rn(__ll2double_rn(L), 0.5);
    double s[3] = {0, 0, 0};
    if (a.V <= 0) {
        s[0] = rng.uniform(-50.0, 50.0);
        s[1] = rng.uniform(-50.0, 50.0);
        s[2] = rng.uniform(-50.0, 50.0);
    } else if (!(dist < __dsub_rn(__ll2double_rn(a.V), 3.0))) {
        record_error(a.ctl, i, 1);
        return;
    }
    const double vmax = __ll2double_rn(a.V - 2);
    for (int attempt = 0; attempt < 10000; ++attempt) {
        double d[3], e[3];
        sphere_dir(rng, d);
        for (int ax = 0; ax < 3; ++ax) {
            const double dd = __dmul_rn(d[ax], dist);
            if (a.V > 0) {
                const double lo = __dadd_rn(1.0, dd < 0.0 ? -dd : 0.0);
                const double hi = __dsub_rn(vmax, dd > 0.0 ? dd : 0.0);
                s[ax] = rng.uniform(lo, hi);
            }
            e[ax] = __dadd_rn(s[ax], dd);
        }
        Plan p;
        if (make_plan(s[0], s[1], s[2], e[0], e[1], e[2], p) && p.n == L) {
            out[0] = s[0];
            out[1] = s[1];
            out[2] = s[2];
            out[3] = e[0];
            out[4] = e[1];
            out[5] = e[2];
            return;
        }
    }
    record_error(a.ctl, i, 4);
}

}  // namespace vxg

// =============================================================================== launchers
namespace vxg {

// 1024-segment tiles of 128 threads x 8: the tiles wait on their look-back prefix at a barrier
// (47% of the stall samples at 256 x 4); smaller CTAs with more segments each keep more of the SM
// busy meanwhile (cfg5: 2.35 -> 2.07 ms; 256 x 8 2.12, 512 x 4 2.23, 256 x 16 2.09).
static constexpr int kPlanBlock = 128, kPlanIPT = 8;
static constexpr int kClipBlock = 256, kClipIPT = 2;

int plan_tile_count(long long n) { return (int)((n + kPlanBlock * kPlanIPT - 1) / (kPlanBlock * kPlanIPT)); }
int clip_tile_count(long long n) { return (int)((n + kClipBlock * kClipIPT - 1) / (kClipBlock * kClipIPT)); }

void launch_plan(const PlanArgs& a, cudaStream_t s) {
    plan_kernel<kPlanBlock, kPlanIPT><<<plan_tile_count(a.n), kPlanBlock, 0, s>>>(a);
}

void launch_tile_index(const long long* off, long long n_entries, int ts_log2, long long* tile_seg,
                       cudaStream_t s) {
    const int b = 256;
    tile_index_kernel<<<(unsigned)((n_entries + b - 1) / b), b, 0, s>>>(off, n_entries, ts_log2,
                                                                         tile_seg);
}

void launch_clip(const ClipArgs& a, cudaStream_t s) {
    clip_kernel<kClipBlock, kClipIPT><<<clip_tile_count(a.n), kClipBlock, 0, s>>>(a);
}

void launch_round_points(const double* p, long long n, int32_t* out, Control* ctl, cudaStream_t s) {
    round_points_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, n, out, ctl);
}
void launch_segment_lengths(const double* segs, long long n, double* out, cudaStream_t s) {
    segment_lengths_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(segs, n, out);
}
void launch_export_plans(const SegRec* rec, const long long* off, long long n,
                         vxg_segment_plan* out, cudaStream_t s) {
    export_plans_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(rec, off, n, out);
}
void launch_pack_plan(const double* segs, const vxg_segment_plan* plans, long long n, SegRec* rec,
                      long long* off, Control* ctl, cudaStream_t s) {
    pack_plan_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(segs, plans, n, rec, off, ctl);
}
void launch_work_item(const SegRec* rec, const long long* off, long long i, long long k,
                      int32_t* out, Control* ctl, cudaStream_t s) {
    work_item_kernel<<<1, 1, 0, s>>>(rec, off, i, k, out, ctl);
}
void launch_gen(const GenArgs& a, cudaStream_t s) {
    gen_kernel<<<(unsigned)((a.n + 127) / 128), 128, 0, s>>>(a);
}

}  // namespace vxg
