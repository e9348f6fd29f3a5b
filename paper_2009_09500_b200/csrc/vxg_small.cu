// vxg_small.cu -- run_batch of a small batch in ONE launch (the latency regime, config 1).
//
// For a few hundred thousand short segments the multi-pass list path (plan kernel with its
// offset scan, count pass, range scan, emit pass: four launches and a readback) costs more in
// launch gaps and per-pass start-up than the samples themselves. Here one kernel does all of
// batch_preprocess and batch_voxelize (src/batch.cpp:57-73, 107-150); a warp owns tiles of 8
// segments, two at a time:
//
//   1. plan   : lane j runs make_plan (src/parametric.cpp:8-26) for segment j into shared memory;
//               N_max and the capacity are pooled per CTA and added to the control block once;
//   2. count  : the warp evaluates the tile's samples k = 0..N of every segment (sample k < N is
//               S + W*k, k = N is E; include/voxline/parametric.hpp:41-48), each lane a contiguous
//               share of one segment, and counts the kept voxels per segment (consecutive
//               duplicates dropped, src/batch.cpp:139-142); the tile's total is published
//               (decoupled look-back, flag A);
//   3. prefix : after counting its NEXT tile too, the warp finds this tile's output position by
//               look-back over the tiles (ids are claimed in order);
//   4. emit   : the warp walks the tile's segments again in rows of 32 samples, writing each kept
//               voxel at its position and every chain's start offset.
//
// Every sample is evaluated twice (count, emit) inside one launch. Measured on cfg1 (65,536 x
// N = 128): 0.078 ms per call (round 1); round 2: records copied from shared memory into
// registers (the count loop re-read them per sample) 0.076 -> 0.074 ms, tiles sized so every
// resident warp takes one pair (small_spw: 10 segments for cfg1) 0.078 -> 0.076, 32.32 fixed-point
// count pieces (vxg_device.cuh) 0.074 -> 0.0696 ms, the E-only last row by lane 0 -> 0.0675,
// N_max / capacity pooled per warp in shared slots instead of 64-bit shared atomics (CAS loops)
// per segment, one rotate shuffle per emit row and 32-bit store indices -> 0.0633 ms, count
// lanes apportioned to segments (one piece per lane instead of two divergent ones) -> 0.0581 ms.
// Variants that did not pay: one tile in flight
// per warp (a third of the instructions were look-back spins: 0.084 ms), a cooperative kernel
// with two grid barriers around a one-CTA scan (0.131 ms), emit rows over the tile's flat sample
// space (0.081 ms), 64 registers for 4 CTAs per SM (spills: 0.080 ms).
// Segments whose N exceeds kSmallMaxSteps make the call ask for the multi-pass path instead
// (Control::n_entries).
#include <algorithm>
#include <cstdint>

#include "vxg_device.cuh"
#include "vxg_internal.h"

namespace vxg {

constexpr int kSmallNW = 8;    // warps per tile
constexpr long long kSmallMaxSteps = 1 << 14;

// Voxel of sample k (0 <= k <= N) of a planned segment (include/voxline/parametric.hpp:41-48).
__device__ __forceinline__ void small_sample(const SegRec& R, bool pos_rec, int k, int N, double t,
                                             int32_t& x, int32_t& y, int32_t& z, bool& bad) {
    if (k < N && pos_rec) {
        x = round_pos(sample_axis(R.sx, R.wx, t));
        y = round_pos(sample_axis(R.sy, R.wy, t));
        z = round_pos(sample_axis(R.sz, R.wz, t));
    } else {
        eval_sample(R, k, N, x, y, z, bad);  // (k == N: E itself)
    }
}

// Key of sample k < N without range checks: the one-DADD rounding for positive records, the
// RZ-bias rounding otherwise (records needing checked rounding never get here).
template <bool POS>
__device__ __forceinline__ int32_t fast_key(const SegRec& R, double t, int32_t& x, int32_t& y,
                                            int32_t& z) {
    if (POS) {
        x = round_pos(sample_axis(R.sx, R.wx, t));
        y = round_pos(sample_axis(R.sy, R.wy, t));
        z = round_pos(sample_axis(R.sz, R.wz, t));
    } else {
        x = round_fast(sample_axis(R.sx, R.wx, t));
        y = round_fast(sample_axis(R.sy, R.wy, t));
        z = round_fast(sample_axis(R.sz, R.wz, t));
    }
    return voxel_key(x, y, z);
}

// Emit pass of one segment, one warp: rows of 32 samples in order; kept voxel of rank r goes to
// out + 3 * (pos + r). FAST: rows wholly below k = N take the branch-free body; the row holding
// k = N (and every row of a record that needs checked rounding) takes the general one.
template <bool FAST, bool POS>
__device__ __forceinline__ void small_emit(const SegRec& R, int N, int32_t* __restrict__ out,
                                           long long pos, bool& bad) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int32_t* const ob = out + 3 * pos;  // (this chain's output: 32-bit indices below)
    int running = 0;
    int32_t carry = 0;
    double t = __int2double_rn(lane);
    int r0 = 0;
    auto commit = [&](bool keep, int32_t key, int32_t x, int32_t y, int32_t z) {
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            int32_t* d = ob + 3 * (running + __popc(m & lt));
            d[0] = x;
            d[1] = y;
            d[2] = z;
        }
        running += __popc(m);
        carry = __shfl_sync(0xffffffffu, key, 31);
    };
    if (FAST) {
        // One rotate per row: lane l gets lane l-1's key, lane 0 this row's lane-31 key -- the
        // previous row's (the carry lane 0 compares with) is what lane 0 got one row earlier.
        for (; r0 + 32 <= N; r0 += 32) {  // every sample of the row has k < N
            int32_t x, y, z;
            const int32_t key = fast_key<POS>(R, t, x, y, z);
            t = __dadd_rn(t, 32.0);
            const int32_t rot = __shfl_sync(0xffffffffu, key, (lane + 31) & 31);
            const bool keep = (r0 | lane) == 0 || key != (lane == 0 ? carry : rot);
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                int32_t* d = ob + 3 * (running + __popc(m & lt));
                d[0] = x;
                d[1] = y;
                d[2] = z;
            }
            running += __popc(m);
            carry = rot;  // (lane 0: this row's last key)
        }
        carry = __shfl_sync(0xffffffffu, carry, 0);
    }
    if (FAST) {  // the row holding k = N: samples below it as above, then E itself
        if (r0 == N && N > 0) {  // (N a multiple of 32: the row holds E alone -- lane 0 does it)
            if (lane == 0) {
                const int32_t key = voxel_key(R.ex, R.ey, R.ez);
                if (key != carry) {
                    int32_t* d = ob + 3 * running;
                    d[0] = R.ex;
                    d[1] = R.ey;
                    d[2] = R.ez;
                }
            }
            return;
        }
        if (r0 <= N) {
            const int k = r0 + lane;
            int32_t x, y, z;
            fast_key<POS>(R, t, x, y, z);
            if (k == N) {
                x = R.ex;
                y = R.ey;
                z = R.ez;
            }
            const int32_t key = voxel_key(x, y, z);
            const int32_t up = __shfl_up_sync(0xffffffffu, key, 1);
            commit(k <= N && (k == 0 || key != (lane == 0 ? carry : up)), key, x, y, z);
        }
        return;
    }
    for (; r0 <= N; r0 += 32) {
        const int k = r0 + lane;
        int32_t x = 0, y = 0, z = 0;
        if (k <= N) small_sample(R, POS, k, N, t, x, y, z, bad);
        t = __dadd_rn(t, 32.0);
        const int32_t key = voxel_key(x, y, z);
        const int32_t up = __shfl_up_sync(0xffffffffu, key, 1);
        commit(k <= N && (k == 0 || key != (lane == 0 ? carry : up)), key, x, y, z);
    }
}

// Kept voxels of samples [k0, k1) of one segment (0 <= k0 < k1 <= N + 1) walked by one lane;
// first / last: the keys of its first and last sample (the first is not counted here).
template <bool FAST, bool POS>
__device__ __forceinline__ int lane_piece(const SegRec& R, int N, int k0, int k1, int32_t& first,
                                          int32_t& last, bool& bad) {
    double t = __int2double_rn(k0);
    int32_t x, y, z;
    int cnt = 0;
    if (FAST && POS && (R.flags & REC_FX) && k0 < N) {
        // 32.32 fixed-point steps (vxg_device.cuh); a lane that meets a sample near a rounding
        // boundary counts its piece again in FP64 below
        const int kf = min(k1, N);
        uint32_t xl, xh, yl, yh, zl, zh, dxl, dxh, dyl, dyh, dzl, dzh;
        fx_start(R.sx, R.wx, t, xl, xh);
        fx_start(R.sy, R.wy, t, yl, yh);
        fx_start(R.sz, R.wz, t, zl, zh);
        fx_delta(R.wx, 0, dxl, dxh);
        fx_delta(R.wy, 0, dyl, dyh);
        fx_delta(R.wz, 0, dzl, dzh);
        bool ok = kf - k0 <= 1024 && __vimin3_u32(xl, yl, zl) >= kFxNear22;
        first = last = voxel_key((int32_t)xh, (int32_t)yh, (int32_t)zh);
#pragma unroll 4
        for (int k = k0 + 1; k < kf; ++k) {
            fx_add(xl, xh, dxl, dxh);
            fx_add(yl, yh, dyl, dyh);
            fx_add(zl, zh, dzl, dzh);
            ok = __vimin3_u32(xl, yl, zl) >= kFxNear22 && ok;
            const int32_t key = voxel_key((int32_t)xh, (int32_t)yh, (int32_t)zh);
            count_ne(cnt, key, last);
            last = key;
        }
        if (ok) {
            if (k1 == N + 1) {  // the piece ends with k = N: E itself
                const int32_t key = voxel_key(R.ex, R.ey, R.ez);
                cnt += key != last;
                last = key;
            }
            return cnt;
        }
        cnt = 0;  // (rare) FP64 below
    }
    if (FAST) {
        const int kf = min(k1, N);  // samples below k = N
        first = last = k0 < N ? fast_key<POS>(R, t, x, y, z) : voxel_key(R.ex, R.ey, R.ez);
        for (int k = k0 + 1; k < kf; ++k) {
            t = __dadd_rn(t, 1.0);
            const int32_t key = fast_key<POS>(R, t, x, y, z);
            count_ne(cnt, key, last);
            last = key;
        }
        if (k1 == N + 1 && k0 < N) {  // the piece ends with k = N: E itself
            const int32_t key = voxel_key(R.ex, R.ey, R.ez);
            cnt += key != last;
            last = key;
        }
    } else {
        small_sample(R, false, k0, N, t, x, y, z, bad);
        first = last = voxel_key(x, y, z);
        for (int k = k0 + 1; k < k1; ++k) {
            t = __dadd_rn(t, 1.0);
            small_sample(R, false, k, N, t, x, y, z, bad);
            const int32_t key = voxel_key(x, y, z);
            cnt += key != last;
            last = key;
        }
    }
    return cnt;
}

// Count pass of a whole tile, one warp: every non-empty segment j gets L_j = 1 +
// floor((32 - segments) * (N_j + 1) / T) consecutive lanes (T: the tile's samples), and each of
// them an equal contiguous share of the segment's samples -- one piece per lane, so the warp's
// fixed-point loop runs as long as the longest share (lanes split across two segments ran two
// divergent loops: twice the iterations on config 1). A lane's first sample is kept when it is
// the segment's k = 0, else compared with the last sample of the lane before (the same segment's
// previous share). myN: lane j < kSmallSPW holds segment j's N (-1: none); cnt[j] must be zero on
// entry.
template <int kSmallSPW>
__device__ __forceinline__ void small_count_flat(const SegRec* rec, int myN, int* cnt, bool& bad,
                                                 int& bad_j) {
    const int lane = threadIdx.x & 31;
    const int M = myN >= 0 ? myN + 1 : 0;
    const int T = (int)__reduce_add_sync(0xffffffffu, (unsigned)M);
    const int nseg = __popc(__ballot_sync(0xffffffffu, M > 0));
    const int L = M > 0 ? 1 + (int)((long long)(32 - nseg) * M / max(T, 1)) : 0;
    int Lx = L;  // inclusive prefix of the lane counts, then exclusive
#pragma unroll
    for (int o = 1; o < kSmallSPW; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, Lx, o);
        if (lane >= o) Lx += u;
    }
    Lx -= L;
    int j = 0;  // this lane's segment: the last non-empty one whose lanes start at or below it
#pragma unroll
    for (int i = 1; i < kSmallSPW; ++i) {
        const int Li = __shfl_sync(0xffffffffu, L, i);
        const int Lxi = __shfl_sync(0xffffffffu, Lx, i);
        if (Li > 0 && Lxi <= lane) j = i;
    }
    const int Lj = __shfl_sync(0xffffffffu, L, j), Lxj = __shfl_sync(0xffffffffu, Lx, j);
    const int Mj = __shfl_sync(0xffffffffu, M, j);
    const int r = lane - Lxj;
    const int q = Lj > 0 ? (Mj + Lj - 1) / Lj : 0;
    const int k0 = r * q, k1 = min(k0 + q, Mj);
    const bool active = r < Lj && k0 < k1;
    int32_t first = 0, last = 0;
    int c = 0;
    if (active) {
        const SegRec R = rec[j];  // (into registers: a shared-memory reference is re-read per sample)
        const int Nj = Mj - 1;
        bool b = false;
        if (R.flags & REC_CHECK) c = lane_piece<false, false>(R, Nj, k0, k1, first, last, b);
        else if (R.flags & REC_POS) c = lane_piece<true, true>(R, Nj, k0, k1, first, last, b);
        else c = lane_piece<true, false>(R, Nj, k0, k1, first, last, b);
        if (b) {
            bad = true;
            bad_j = j;
        }
    }
    const int32_t up = __shfl_up_sync(0xffffffffu, last, 1);
    if (active) {
        c += (k0 == 0 || first != up) ? 1 : 0;
        atomicAdd(&cnt[j], c);
    }
}

// Dispatch on the record's rounding class (warp-uniform).
__device__ __forceinline__ void small_emit_seg(const SegRec& Rs, int N, int32_t* out, long long pos,
                                               bool& bad) {
    const SegRec R = Rs;  // (into registers: a shared-memory reference is re-read per row)
    if (R.flags & REC_CHECK) small_emit<false, false>(R, N, out, pos, bad);
    else if (R.flags & REC_POS) small_emit<true, true>(R, N, out, pos, bad);
    else small_emit<true, false>(R, N, out, pos, bad);
}

// Plan one tile of segments (lane j < kSmallSPW: segment seg0 + j) into `rec` (shared memory).
// Returns the lane's N (-1: no segment); pools N_max / capacity into the lane's partials.
template <int kSmallSPW>
__device__ __forceinline__ int small_plan_tile(const SmallArgs& a, long long seg0, SegRec* rec,
                                               unsigned& w_max, unsigned long long& w_cap,
                                               bool& is_long) {
    const int lane = threadIdx.x & 31;
    int myN = -1;
    is_long = false;
    unsigned n32 = 0, c32 = 0;
    if (lane < kSmallSPW) {
        const long long i = seg0 + lane;
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
            rec[lane] = r;
            // (32-bit partials: a batch holding N > 2^14 is redone by the multi-pass path,
            // which reports its own N_max and capacity)
            n32 = (unsigned)min(pl.n, (long long)kSmallMaxSteps + 1);
            c32 = n32 + 1u;
            is_long = pl.n > kSmallMaxSteps;
            myN = is_long ? 0 : (int)pl.n;
        }
    }
    // the warp's partials (a shared slot per warp: no atomics, nothing held in registers)
    n32 = __reduce_max_sync(0xffffffffu, n32);
    c32 = __reduce_add_sync(0xffffffffu, c32);
    if (lane == 0) {
        w_max = max(w_max, n32);
        w_cap += c32;
    }
    return myN;
}

// A claimed tile between its count and its emit.
struct SmallTile {
    long long tile;  // ticket (>= ntiles: none)
    int myN, myc;    // lane j < kSmallSPW: segment j's N and kept voxels
    bool is_long;    // the tile holds a segment too long for this path
};

// Claim the next tile, plan it into `rec`, count it and publish its total (look-back flag A).
template <int kSmallSPW>
__device__ __forceinline__ SmallTile small_count_tile(const SmallArgs& a, SegRec* rec, int* cnt,
                                                      unsigned& w_max,
                                                      unsigned long long& w_cap, int* s_long,
                                                      bool& bad, long long& bad_seg) {
    const int lane = threadIdx.x & 31;
    SmallTile T;
    unsigned long long tk = 0;
    if (lane == 0) tk = atomicAdd(&a.ctl->tile_counter, 1ull);
    T.tile = (long long)__shfl_sync(0xffffffffu, tk, 0);
    T.myN = -1;
    T.myc = 0;
    T.is_long = false;
    if (T.tile >= a.ntiles) return T;
    const long long seg0 = T.tile * kSmallSPW;
    bool il;
    T.myN = small_plan_tile<kSmallSPW>(a, seg0, rec, w_max, w_cap, il);
    T.is_long = __any_sync(0xffffffffu, il);
    if (T.is_long && lane == 0) *s_long = 1;
    __syncwarp();
    if (!T.is_long) {
        if (lane < kSmallSPW) cnt[lane] = 0;
        __syncwarp();
        bool b = false;
        int bj = 0;
        small_count_flat<kSmallSPW>(rec, T.myN, cnt, b, bj);
        if (b) {
            bad = true;
            bad_seg = seg0 + bj;
        }
        __syncwarp();
        if (lane < kSmallSPW) T.myc = cnt[lane];
    }
    const unsigned agg = __reduce_add_sync(0xffffffffu, (unsigned)T.myc);
    if (lane == 0) lookback_publish(a.status, T.tile, agg);
    return T;
}

// Resolve a counted tile's output position by look-back, then emit it.
template <int kSmallSPW>
__device__ __forceinline__ void small_emit_tile(const SmallArgs& a, const SmallTile& T,
                                                const SegRec* rec) {
    const int lane = threadIdx.x & 31;
    int incl = T.myc;
#pragma unroll
    for (int o = 1; o < kSmallSPW; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    const int excl = incl - T.myc;
    const long long agg = __shfl_sync(0xffffffffu, incl, kSmallSPW - 1);
    const long long pre = lookback_resolve(a.status, T.tile, agg, a.ctl);
    if (lane == 0 && T.tile == a.ntiles - 1) {
        if (a.chain_off) a.chain_off[a.n] = pre + agg;
        a.ctl->total = pre + agg;
    }
    if (pre + agg > a.out_cap) {  // caller's buffer too small: nothing written
        if (lane == 0) record_error(a.ctl, 0, 4);
        return;
    }
    if (T.is_long) return;
    const long long seg0 = T.tile * kSmallSPW;
#pragma unroll 1
    for (int j = 0; j < kSmallSPW; ++j) {
        const int N = __shfl_sync(0xffffffffu, T.myN, j);
        if (N < 0) break;
        const long long pos = pre + __shfl_sync(0xffffffffu, excl, j);
        if (lane == 0 && a.chain_off) a.chain_off[seg0 + j] = pos;
        bool b = false;
        small_emit_seg(rec[j], N, a.out, pos, b);
    }
}

// Persistent warps, two tiles in flight each: claim + count + publish tile A, claim + count +
// publish tile B, then resolve and emit A, then B. Every tile's count is published one tile of
// work before anyone waits for it, so the look-backs rarely spin; no block-wide barrier on the
// way (the CTA only pools the N_max / capacity partials in shared memory).
template <int kSmallSPW>
__global__ void __launch_bounds__(kSmallNW * 32) list_small_kernel(SmallArgs a) {
    __shared__ SegRec s_rec[kSmallNW][2][kSmallSPW];
    __shared__ int s_cnt[kSmallNW][kSmallSPW];
    __shared__ unsigned long long s_max, s_cap;
    __shared__ int s_long;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (tid == 0) {
        s_max = s_cap = 0;
        s_long = 0;
    }
    __syncthreads();
    bool bad = false;
    long long bad_seg = 0;
    __shared__ unsigned s_wmax[kSmallNW];
    __shared__ unsigned long long s_wcap[kSmallNW];
    if ((tid & 31) == 0) {
        s_wmax[warp] = 0;
        s_wcap[warp] = 0;
    }
    __syncwarp();
    for (;;) {
        const SmallTile A = small_count_tile<kSmallSPW>(a, s_rec[warp][0], s_cnt[warp], s_wmax[warp], s_wcap[warp],
                                             &s_long, bad, bad_seg);
        if (A.tile >= a.ntiles) break;
        const SmallTile B = small_count_tile<kSmallSPW>(a, s_rec[warp][1], s_cnt[warp], s_wmax[warp], s_wcap[warp],
                                             &s_long, bad, bad_seg);
        small_emit_tile<kSmallSPW>(a, A, s_rec[warp][0]);
        if (B.tile >= a.ntiles) break;
        small_emit_tile<kSmallSPW>(a, B, s_rec[warp][1]);
        __syncwarp();
    }
    if (bad) record_error(a.ctl, bad_seg, 2);
    if ((tid & 31) == 0) {
        if (s_wmax[warp]) atomicMax(&s_max, (unsigned long long)s_wmax[warp]);
        if (s_wcap[warp]) atomicAdd(&s_cap, s_wcap[warp]);
    }
    __syncthreads();
    if (tid == 0) {
        if (s_max) atomicMax(&a.ctl->max_steps, s_max);
        if (s_cap) atomicAdd(reinterpret_cast<unsigned long long*>(&a.ctl->pad0), s_cap);  // capacity
        if (s_long) atomicExch(reinterpret_cast<unsigned long long*>(&a.ctl->n_entries), 1ull);
    }
}

long long small_tile_count(long long n, int spw) { return (n + spw - 1) / spw; }

template <int SPW>
static int small_per_sm() {
    static int per_sm[64] = {0};  // per device (attributes are per device / context)
    int dev = 0;
    cudaGetDevice(&dev);
    int& p = per_sm[dev & 63];
    if (!p) {
        int q = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&q, list_small_kernel<SPW>, kSmallNW * 32, 0);
        p = q < 1 ? 1 : q;
    }
    return p;
}

// Segments per warp tile: every resident warp takes two tiles at a time, so a batch whose tiles
// all fit the resident warps in one round finishes in one tile-pair time -- the smallest tile
// that does so (the critical path is one pair of tiles); bigger batches use 8-segment tiles.
// (cfg1, 65,536 segments, 3 CTAs of 8 warps per SM: 8-segment tiles left 544 warps with a second
// pair, 10-segment tiles give every warp one.)
int small_spw(long long n, int num_sms) {
    static const int opts[] = {4, 6, 8, 10, 12, 16};
    for (int spw : opts) {
        int per_sm = spw == 4 ? small_per_sm<4>() : spw == 6 ? small_per_sm<6>()
                   : spw == 8 ? small_per_sm<8>() : spw == 10 ? small_per_sm<10>()
                   : spw == 12 ? small_per_sm<12>() : small_per_sm<16>();
        const long long warps = (long long)per_sm * num_sms * kSmallNW;
        if ((small_tile_count(n, spw) + 1) / 2 <= warps) return spw;
    }
    return 8;
}

// Persistent CTAs: as many as are resident at once (tiles are claimed dynamically).
template <int SPW>
static cudaError_t launch_small_spw(const SmallArgs& a, int num_sms, cudaStream_t s) {
    const long long need = (a.ntiles + 2 * kSmallNW - 1) / (2 * kSmallNW);
    const long long grid =
        std::max<long long>(1, std::min<long long>(need, (long long)small_per_sm<SPW>() * num_sms));
    list_small_kernel<SPW><<<(unsigned)grid, kSmallNW * 32, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_list_small(const SmallArgs& a, int num_sms, cudaStream_t s) {
    switch (a.spw) {
        case 4: return launch_small_spw<4>(a, num_sms, s);
        case 6: return launch_small_spw<6>(a, num_sms, s);
        case 10: return launch_small_spw<10>(a, num_sms, s);
        case 12: return launch_small_spw<12>(a, num_sms, s);
        case 16: return launch_small_spw<16>(a, num_sms, s);
        default: return launch_small_spw<8>(a, num_sms, s);
    }
}

}  // namespace vxg
