// vxg_small.cu -- run_batch of a small batch in ONE launch (the latency regime, config 1).
//
// For a few hundred thousand short segments the multi-pass list path (plan kernel with its
// offset scan, count pass, range scan, emit pass: four launches and a readback) costs more in
// launch gaps and per-pass start-up than the samples themselves. Here one kernel does all of
// batch_preprocess and batch_voxelize (src/batch.cpp:57-73, 107-150) per tile of segments:
//
//   1. plan   : one thread per segment of the tile runs make_plan (src/parametric.cpp:8-26)
//               into shared memory; N_max and the capacity go to the control block;
//   2. count  : one warp per segment walks its samples k = 0..N in rows of 32 (sample k < N is
//               S + W*k, k = N is E; include/voxline/parametric.hpp:41-48) and counts the kept
//               voxels (consecutive duplicates dropped, src/batch.cpp:139-142);
//   3. prefix : the tile's voxel count is published and its output position found by decoupled
//               look-back over the tiles (tile ids are claimed in order, so the predecessors are
//               already counting or done);
//   4. emit   : the warps walk their segments again, now writing each kept voxel at its position
//               and every chain's start offset.
//
// Every sample is evaluated twice (count, emit) but in the same kernel, from shared memory, with
// no grid-wide barrier. Segments whose N exceeds kSmallMaxSteps make the call ask for the
// multi-pass path instead (Control::n_entries), before anything that path would not overwrite.
#include <cstdint>

#include "vxg_device.cuh"
#include "vxg_internal.h"

namespace vxg {

constexpr int kSmallNW = 8;    // warps per tile
constexpr int kSmallSPW = 8;   // segments per warp
constexpr int kSmallTS = kSmallNW * kSmallSPW;
constexpr long long kSmallMaxSteps = 1 << 14;

// One segment, one warp: rows of 32 samples; returns the kept voxels (warp-uniform). EMIT: kept
// voxel of rank r goes to out + 3 * (pos + r).
template <bool EMIT>
__device__ __forceinline__ int small_walk(const SegRec& R, long long N, int32_t* __restrict__ out,
                                          long long pos, bool& bad) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int running = 0;
    int32_t carry = 0;
    const bool pos_rec = (R.flags & (REC_CHECK | REC_POS)) == REC_POS;
    for (long long r0 = 0; r0 <= N; r0 += 32) {
        const long long k = r0 + lane;
        int32_t x = 0, y = 0, z = 0;
        if (k < N) {
            if (pos_rec) {
                const double t = __ll2double_rn(k);
                x = round_pos(sample_axis(R.sx, R.wx, t));
                y = round_pos(sample_axis(R.sy, R.wy, t));
                z = round_pos(sample_axis(R.sz, R.wz, t));
            } else {
                eval_sample(R, k, N, x, y, z, bad);
            }
        } else if (k == N) {  // the final sample is E itself
            x = R.ex;
            y = R.ey;
            z = R.ez;
        }
        const int32_t key = voxel_key(x, y, z);
        const int32_t up = __shfl_up_sync(0xffffffffu, key, 1);
        const bool keep = k <= N && (k == 0 || key != (lane == 0 ? carry : up));
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (EMIT && keep) {
            int32_t* d = out + 3 * (pos + running + __popc(m & lt));
            d[0] = x;
            d[1] = y;
            d[2] = z;
        }
        running += __popc(m);
        carry = __shfl_sync(0xffffffffu, key, 31);
    }
    return running;
}

__global__ void __launch_bounds__(kSmallNW * 32) list_small_kernel(SmallArgs a) {
    __shared__ SegRec s_rec[kSmallTS];
    __shared__ long long s_n[kSmallTS];
    __shared__ int s_cnt[kSmallTS];
    __shared__ long long s_tile, s_prefix;
    __shared__ unsigned long long s_max, s_cap;
    __shared__ int s_long;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_tile = (long long)atomicAdd(&a.ctl->tile_counter, 1ull);
        s_max = s_cap = 0;
        s_long = 0;
    }
    __syncthreads();
    const long long tile = s_tile;
    const long long seg0 = tile * kSmallTS;

    // ---- 1. plan (one thread per segment of the tile)
    if (tid < kSmallTS) {
        const long long i = seg0 + tid;
        long long N = -1;  // (no segment: no samples)
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
            s_rec[tid] = r;
            N = pl.n;
            atomicMax(&s_max, (unsigned long long)N);
            atomicAdd(&s_cap, (unsigned long long)(N + 1));
            if (N > kSmallMaxSteps) s_long = 1;
        }
        s_n[tid] = N;
    }
    __syncthreads();
    if (tid == 0) {
        atomicMax(&a.ctl->max_steps, s_max);
        atomicAdd(reinterpret_cast<unsigned long long*>(&a.ctl->pad0), s_cap);  // capacity
        if (s_long) atomicExch(reinterpret_cast<unsigned long long*>(&a.ctl->n_entries), 1ull);
    }

    // ---- 2. count
    bool bad = false;
    long long bad_seg = 0;
    if (!s_long) {
        for (int j = 0; j < kSmallSPW; ++j) {
            const int s = warp * kSmallSPW + j;
            const long long N = s_n[s];
            int c = 0;
            if (N >= 0) {
                bool b = false;
                c = small_walk<false>(s_rec[s], N, nullptr, 0, b);
                if (b) {
                    bad = true;
                    bad_seg = seg0 + s;
                }
            }
            if (lane == 0) s_cnt[s] = c;
        }
    }
    __syncthreads();

    // ---- 3. prefix: tile-local exclusive offsets of the segments, tile total, look-back
    if (warp == 0) {
        static_assert(kSmallTS == 64, "two segments per lane");
        const int v0 = s_long ? 0 : s_cnt[2 * lane], v1 = s_long ? 0 : s_cnt[2 * lane + 1];
        int incl = v0 + v1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int excl = incl - v0 - v1;
        s_cnt[2 * lane] = excl;
        s_cnt[2 * lane + 1] = excl + v0;
        const long long agg = __shfl_sync(0xffffffffu, incl, 31);
        const long long pre = lookback_warp(a.status, tile, agg, a.ctl);
        if (lane == 0) {
            s_prefix = pre;
            if (pre + agg > a.out_cap) {  // caller's buffer too small: nothing written
                record_error(a.ctl, 0, 4);
                s_prefix = -1;
            }
            if (tile == a.ntiles - 1) {
                if (a.chain_off) a.chain_off[a.n] = pre + agg;
                a.ctl->total = pre + agg;
            }
        }
    }
    __syncthreads();
    if (s_long || s_prefix < 0) {
        if (bad) record_error(a.ctl, bad_seg, 2);
        return;
    }

    // ---- 4. emit
    for (int j = 0; j < kSmallSPW; ++j) {
        const int s = warp * kSmallSPW + j;
        const long long N = s_n[s];
        if (N < 0) continue;
        const long long pos = s_prefix + s_cnt[s];
        if (lane == 0 && a.chain_off) a.chain_off[seg0 + s] = pos;
        bool b = false;
        small_walk<true>(s_rec[s], N, a.out, pos, b);
    }
    if (bad) record_error(a.ctl, bad_seg, 2);
}

long long small_tile_count(long long n) { return (n + kSmallTS - 1) / kSmallTS; }

cudaError_t launch_list_small(const SmallArgs& a, cudaStream_t s) {
    list_small_kernel<<<(unsigned)a.ntiles, kSmallNW * 32, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace vxg
