// vxg_emit.cu -- the emit kernels: thread-per-sample evaluation of G_k = S + W*k over the flat
// (segment, k) sample space (the paper's N_P x (N_max + 1) grid without redundant items,
// SURVEY.md §2 row 3), writing either the deduplicated voxel list (batch_voxelize's kernel AND
// assemble phases, src/batch.cpp:107-150, fused) or an occupancy bitmap.
#include <cstdint>
#include <mutex>

#include "vxg_device.cuh"
#include "vxg_internal.h"

namespace vxg {

// =============================================================================== row walker
// The flat sample space is cut into warp chunks of 32*IPT consecutive samples, walked in rows of
// 32 (lane L holds sample row_start + L). Instead of searching every sample's segment, the warp
// carries the entry c containing the row's first sample and, only for rows that cross an entry
// boundary, loads the next 32 entry starts, builds a bitmask of boundary positions in the row
// with one OR-reduction and gives every lane its entry with one popc. Entries always hold at
// least one sample, so a 32-sample row crosses at most 31 boundaries.
struct RowWalker {
    long long c;        // entry containing the row's first sample
    long long so_c;     // its first flat sample
    long long so_next;  // first flat sample of entry c + 1
};

constexpr long long kNoEntry = 0x7fffffffffffffffll;

// Largest c in [lo, hi] with off[c] <= f (off[lo] <= f guaranteed); warp-cooperative 32-ary
// search, all lanes return the same value.
__device__ __forceinline__ long long warp_find_entry(const long long* __restrict__ off,
                                                     long long lo, long long hi, long long f) {
    const int lane = threadIdx.x & 31;
    while (hi - lo > 31) {
        const long long step = (hi - lo + 32) / 32;  // ceil((hi - lo + 1) / 32): covers hi
        const long long p = lo + (long long)lane * step;
        const unsigned m = __ballot_sync(0xffffffffu, p <= hi && __ldg(off + p) <= f);
        const int last = 31 - __clz(m);
        lo = lo + (long long)last * step;
        hi = min(hi, lo + step - 1);
    }
    const long long p = lo + lane;
    const unsigned m = __ballot_sync(0xffffffffu, p <= hi && __ldg(off + p) <= f);
    return lo + (31 - __clz(m));
}

__device__ __forceinline__ void walker_init(RowWalker& w, const long long* __restrict__ off,
                                            long long lo, long long hi, long long f) {
    w.c = warp_find_entry(off, lo, hi, f);
    w.so_c = __ldg(off + w.c);
    w.so_next = __ldg(off + w.c + 1);
}

// Entry of this lane's sample in the row starting at row_start; advances the walker to the row
// starting at row_start + 32. Warp-uniform control flow; all lanes must call it.
__device__ __forceinline__ void walker_row(RowWalker& w, const long long* __restrict__ off,
                                           long long n_entries, long long row_start,
                                           long long& my_entry, long long& my_start,
                                           long long& my_next) {
    const int lane = threadIdx.x & 31;
    if (w.so_next > row_start + 32) {  // no boundary in this row nor at the next row's start
        my_entry = w.c;
        my_start = w.so_c;
        my_next = w.so_next;
        return;
    }
    const long long idx = w.c + 1 + lane;
    const long long B = idx <= n_entries ? __ldg(off + idx) : kNoEntry;
    const long long d = B - row_start;  // >= 1
    const unsigned pos = __reduce_or_sync(0xffffffffu, d < 32 ? (1u << (int)d) : 0u);
    const unsigned upto = lane == 31 ? pos : (pos & ((2u << lane) - 1u));
    const int nb = __popc(upto);
    const long long b_prev = __shfl_sync(0xffffffffu, B, nb == 0 ? 0 : nb - 1);
    const long long b_next = __shfl_sync(0xffffffffu, B, nb);
    my_entry = w.c + nb;
    my_start = nb == 0 ? w.so_c : b_prev;
    my_next = b_next;
    const int adv = __popc(__ballot_sync(0xffffffffu, d <= 32));
    if (adv > 0) {
        const long long nc = __shfl_sync(0xffffffffu, B, adv - 1);
        const long long nn = __shfl_sync(0xffffffffu, B, adv & 31);
        w.c += adv;
        w.so_c = nc;
        w.so_next = adv < 32 ? nn : __ldg(off + w.c + 1);
    }
}

// =============================================================================== emit: list
// batch_voxelize's kernel and assemble phases (src/batch.cpp:107-150) as two passes over the flat
// (segment, k) sample space, which is cut into R equal contiguous ranges, one per resident warp
// (multiples of 32*IPT samples):
//   list_count_kernel : every warp walks its range and counts the kept (deduplicated) voxels
//   range_scan_kernel : exclusive prefix of the R range counts (one CTA)
//   list_emit_kernel  : every warp walks the same range again from its known output position,
//                       staging kept voxels in shared memory (12-B records at their rank, at the
//                       output's 16-B phase) and writing each block of 32*IPT samples out with one
//                       TMA bulk store (cp.async.bulk); chain offsets are written as the k = 0
//                       samples go by
// No inter-warp waiting anywhere (a single pass would need a look-back whose waits couple every
// warp to its predecessors). Each warp walks one long contiguous range, so the per-block start-up
// (entry search, record load, dedup carry) happens once per range, not once per block.
// Large batches use list_fused_kernel instead: the same count and emit walks as tasks over 32x
// finer ranges in one persistent kernel, so the FP64-bound counting and the store-bound emitting
// share the SMs (see its comment).
//
// A warp walks rows of 32 consecutive samples (lane L holds sample row_start + L). Rows without an
// entry boundary (most rows: config-4 segments are ~1000 samples long) take the fast path: one
// warp-uniform record, t = (row_start - so_c) + lane, S + W*t, llround, and a keep flag from
// comparing the voxel key with the previous lane's (lane 0: the previous row's lane 31). The
// k == N (E) sample always lies in a boundary row. Boundary rows, partial rows and records that
// need checked rounding or exact comparison take the generic path through the row walker.

// Walker state carried from block to block along a warp's range. Records are not carried:
// each fast run / boundary row loads the record(s) it needs (a uniform 64-B load that hits L1
// after the first row of a segment), which keeps the register count low enough for 24 warps.
struct Walk {
    RowWalker w;
    int32_t carry;  // voxel key of the sample before the next row (lane 0's predecessor)
};

__device__ __forceinline__ void walk_start(const ListArgs& a, long long f0, Walk& W) {
    walker_init(W.w, a.off, 0, a.nseg - 1, f0);
    W.carry = 0;
    if (f0 > W.w.so_c) {
        const SegRec R = load_rec(a.rec + W.w.c);
        int32_t px, py, pz;
        bool b = false;
        eval_sample(R, f0 - 1 - W.w.so_c, W.w.so_next - W.w.so_c - 1, px, py, pz, b);
        W.carry = voxel_key(px, py, pz);
    }
}

// Walk samples [wbase, wend) (wbase a multiple of 32, wend - wbase <= 32*IPT). EMIT: stage kept
// voxels at stage + 3*rank and write chain_off[e] = pos + rank for every k = 0 sample. Returns the
// number of kept voxels (warp-uniform). The walker is left standing at sample wend.
template <int IPT, bool EMIT>
__device__ __forceinline__ int walk_block(const ListArgs& a, Walk& W, long long wbase,
                                          long long wend, uint32_t* stage, long long pos) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    RowWalker& w = W.w;
    int32_t& carry = W.carry;
    bool bad = false;
    long long bad_seg = 0;
    int running = 0;

    auto commit = [&](bool keep, int32_t x, int32_t y, int32_t z) {
        const unsigned mask = __ballot_sync(0xffffffffu, keep);
        if (EMIT && keep) {
            uint32_t* d = stage + 3 * (running + __popc(mask & lt));
            d[0] = (uint32_t)x;
            d[1] = (uint32_t)y;
            d[2] = (uint32_t)z;
        }
        running += __popc(mask);
    };

    int j = 0;
    while (j < IPT) {
        const long long row_start = wbase + (long long)j * 32;
        if (row_start >= wend) break;
        // (the walker may stand one past the last entry only at the end of the sample space)
        const uint32_t flags = __ldg(&a.rec[w.c].flags);
        // ---- fast rows: row r is fast iff row_start_r + 32 <= min(so_next - 1, wend)
        const long long lim = min(w.so_next - 1, wend);
        int nfast = 0;
        if (!(flags & (REC_CHECK | REC_WIDE)) && lim >= row_start + 32)
            nfast = (int)min((lim - row_start) >> 5, (long long)(IPT - j));
        if (!EMIT && nfast > 0) {
            // counting only: the run's 32 * nfast samples are split into 32 contiguous lane
            // sub-ranges of nfast samples, so a sample's predecessor is the lane's own previous
            // sample (a register) -- no shuffle, ballot or popc per sample; one shuffle joins
            // the sub-ranges and one warp reduction sums the counts
            const SegRec R = load_rec(a.rec + w.c);
            // the next segment's record into L2 while this run is walked (its flags and record
            // are the next row's first loads; the count tasks are the first to touch a range's
            // records). Measured with the same prefetch in the emit runs: cfg4 fused 10.84 ->
            // 10.67 ms; 2 or 4 records ahead and L1 prefetches were no better.
            if (lane == 0 && w.c + 1 < a.nseg) prefetch_l2(a.rec + w.c + 1);
            const double t0 = __ll2double_rn(row_start - w.so_c + (long long)lane * nfast);
            int32_t first_key, key;
            int cnt = 0;
            auto exact_pos = [&](const SegRec& R) {  // FP64 samples, one-DADD rounding (REC_POS)
                double t = t0;
                first_key = key = voxel_key(round_pos(sample_axis(R.sx, R.wx, t)),
                                            round_pos(sample_axis(R.sy, R.wy, t)),
                                            round_pos(sample_axis(R.sz, R.wz, t)));
#pragma unroll 4
                for (int f = 1; f < nfast; ++f) {
                    t = __dadd_rn(t, 1.0);
                    const int32_t k2 = voxel_key(round_pos(sample_axis(R.sx, R.wx, t)),
                                                 round_pos(sample_axis(R.sy, R.wy, t)),
                                                 round_pos(sample_axis(R.sz, R.wz, t)));
                    count_ne(cnt, k2, key);
                    key = k2;
                }
            };
            if ((flags & (REC_POS | REC_FX)) == (REC_POS | REC_FX) && nfast <= 1023 &&
                !(a.fx_off)) {
                // 32.32 fixed-point steps (vxg_device.cuh): no FP64 per sample; a lane that meets
                // a sample near a rounding boundary counts its sub-range again in FP64
                uint32_t xl, xh, yl, yh, zl, zh, dxl, dxh, dyl, dyh, dzl, dzh;
                fx_start(R.sx, R.wx, t0, xl, xh);
                fx_start(R.sy, R.wy, t0, yl, yh);
                fx_start(R.sz, R.wz, t0, zl, zh);
                fx_delta(R.wx, 0, dxl, dxh);
                fx_delta(R.wy, 0, dyl, dyh);
                fx_delta(R.wz, 0, dzl, dzh);
                bool ok = __vimin3_u32(xl, yl, zl) >= kFxNear22;
                first_key = key = voxel_key((int32_t)xh, (int32_t)yh, (int32_t)zh);
#pragma unroll 4
                for (int f = 1; f < nfast; ++f) {
                    fx_add(xl, xh, dxl, dxh);
                    fx_add(yl, yh, dyl, dyh);
                    fx_add(zl, zh, dzl, dzh);
                    ok = __vimin3_u32(xl, yl, zl) >= kFxNear22 && ok;
                    const int32_t k2 = voxel_key((int32_t)xh, (int32_t)yh, (int32_t)zh);
                    count_ne(cnt, k2, key);
                    key = k2;
                }
                if (!ok) {  // (rare; the record is reloaded: it is not kept live across the loop)
                    cnt = 0;
                    exact_pos(load_rec(a.rec + w.c));
                }
            } else if (flags & REC_POS) {
                exact_pos(R);
            } else {
                double t = t0;
                first_key = key = voxel_key(round_fast(sample_axis(R.sx, R.wx, t)),
                                            round_fast(sample_axis(R.sy, R.wy, t)),
                                            round_fast(sample_axis(R.sz, R.wz, t)));
#pragma unroll 2
                for (int f = 1; f < nfast; ++f) {
                    t = __dadd_rn(t, 1.0);
                    const int32_t k2 = voxel_key(round_fast(sample_axis(R.sx, R.wx, t)),
                                                 round_fast(sample_axis(R.sy, R.wy, t)),
                                                 round_fast(sample_axis(R.sz, R.wz, t)));
                    count_ne(cnt, k2, key);
                    key = k2;
                }
            }
            // predecessor of a lane's first sample: lane - 1's last one (lane 0: the carry);
            // k == 0 (lane 0 of a run that starts the segment) is always kept
            const int32_t up = __shfl_up_sync(0xffffffffu, key, 1);
            const bool kfirst = lane == 0 && row_start == w.so_c;
            cnt += (kfirst || first_key != (lane == 0 ? carry : up)) ? 1 : 0;
            running += (int)__reduce_add_sync(0xffffffffu, (unsigned)cnt);
            carry = __shfl_sync(0xffffffffu, key, 31);
            j += nfast;
            continue;
        }
        if (nfast > 0) {
            const SegRec R = load_rec(a.rec + w.c);
            if (lane == 0 && w.c + 1 < a.nseg) prefetch_l2(a.rec + w.c + 1);  // (as above)
            double t = __ll2double_rn(row_start - w.so_c + lane);
            // k == 0 (always kept) can only sit at lane 0 of the first fast row
            bool first = lane == 0 && row_start == w.so_c;
            if (EMIT && first) a.chain_off[w.c] = pos + running;
            // lane 0's predecessor key arrives through a rotate: after row r, lane 0 holds lane
            // 31's key of row r, which is its predecessor in row r + 1
            int32_t prev0 = carry;
            if (flags & REC_POS) {
#pragma unroll 4
                for (int f = 0; f < nfast; ++f) {
                    const int32_t x = round_pos(sample_axis(R.sx, R.wx, t));
                    const int32_t y = round_pos(sample_axis(R.sy, R.wy, t));
                    const int32_t z = round_pos(sample_axis(R.sz, R.wz, t));
                    const int32_t key = voxel_key(x, y, z);
                    const int32_t rot = __shfl_sync(0xffffffffu, key, (lane + 31) & 31);
                    const int32_t pk = lane == 0 ? prev0 : rot;
                    prev0 = rot;
                    commit(key != pk || first, x, y, z);
                    first = false;
                    t = __dadd_rn(t, 32.0);
                }
            } else {
#pragma unroll 2
                for (int f = 0; f < nfast; ++f) {
                    const int32_t x = round_fast(sample_axis(R.sx, R.wx, t));
                    const int32_t y = round_fast(sample_axis(R.sy, R.wy, t));
                    const int32_t z = round_fast(sample_axis(R.sz, R.wz, t));
                    const int32_t key = voxel_key(x, y, z);
                    const int32_t rot = __shfl_sync(0xffffffffu, key, (lane + 31) & 31);
                    const int32_t pk = lane == 0 ? prev0 : rot;
                    prev0 = rot;
                    commit(key != pk || first, x, y, z);
                    first = false;
                    t = __dadd_rn(t, 32.0);
                }
            }
            carry = __shfl_sync(0xffffffffu, prev0, 0);
            j += nfast;
            continue;
        }
        // ---- boundary row: the row holds entry c's last sample (E) at lane d-1 and, if d < 32,
        // the first 32-d samples of entry c+1, which continues past the row. Same arithmetic as a
        // fast row; every lane loads the record of its own entry. Rows with more boundaries,
        // partial rows and records that need checked rounding or exact comparison take the
        // generic path below.
        if ((flags & (REC_CHECK | REC_WIDE | REC_POS)) == REC_POS && row_start + 32 <= wend) {
            const int d = (int)(w.so_next - row_start);  // 1..32 (the row is not fast)
            const long long c1 = w.c + 1;
            bool ok = true;
            long long so2 = 0;
            if (d < 32) {
                ok = c1 < a.nseg;
                if (ok) {
                    so2 = __ldg(a.off + c1 + 1);
                    const uint32_t f2 = __ldg(&a.rec[c1].flags);
                    ok = so2 > row_start + 32 && (f2 & (REC_CHECK | REC_WIDE | REC_POS)) == REC_POS;
                }
            }
            if (ok) {
                const bool in_c = lane < d;
                const SegRec M = load_rec(a.rec + (in_c ? w.c : c1));
                const long long kk = in_c ? row_start - w.so_c + lane : (long long)(lane - d);
                const double t = __ll2double_rn(kk);
                int32_t x = round_pos(sample_axis(M.sx, M.wx, t));
                int32_t y = round_pos(sample_axis(M.sy, M.wy, t));
                int32_t z = round_pos(sample_axis(M.sz, M.wz, t));
                if (lane == d - 1) {  // k == N_c: the sample is E itself
                    x = M.ex;
                    y = M.ey;
                    z = M.ez;
                }
                const int32_t key = voxel_key(x, y, z);
                const int32_t rot = __shfl_sync(0xffffffffu, key, (lane + 31) & 31);
                const bool start = (lane == d && d < 32) || (lane == 0 && row_start == w.so_c);
                const bool keep = start || key != (lane == 0 ? carry : rot);
                const unsigned mask = __ballot_sync(0xffffffffu, keep);
                const int rank = running + __popc(mask & lt);
                if (EMIT) {
                    if (keep) {
                        uint32_t* dd = stage + 3 * rank;
                        dd[0] = (uint32_t)x;
                        dd[1] = (uint32_t)y;
                        dd[2] = (uint32_t)z;
                    }
                    if (start) a.chain_off[in_c ? w.c : c1] = pos + rank;  // chain start
                }
                running += __popc(mask);
                carry = __shfl_sync(0xffffffffu, key, 31);
                // the walker moves to entry c+1 (which holds the next row's first sample)
                w.c = c1;
                w.so_c = w.so_next;
                if (d < 32) w.so_next = so2;
                else if (c1 < a.nseg) w.so_next = __ldg(a.off + c1 + 1);
                ++j;
                continue;
            }
        }
        // ---- generic row: entry boundaries, the k == N sample, partial rows, checked records
        long long e, st, nx;
        walker_row(w, a.off, a.nseg, row_start, e, st, nx);
        const long long f = row_start + lane;
        const bool valid = f < wend;
        long long k = 0;
        int32_t x = 0, y = 0, z = 0, px, py, pz;
        const SegRec rr = load_rec(a.rec + min(e, a.nseg - 1));
        if (valid) {
            k = f - st;
            bool b = false;
            eval_sample(rr, k, nx - st - 1, x, y, z, b);
            if (b) {
                bad = true;
                bad_seg = e;
            }
        }
        px = __shfl_up_sync(0xffffffffu, x, 1);
        py = __shfl_up_sync(0xffffffffu, y, 1);
        pz = __shfl_up_sync(0xffffffffu, z, 1);
        bool same;
        if (lane == 0) {
            // lane 0's previous sample (same entry iff k > 0): the carried key, or recomputed
            // exactly for records whose |W| > 1 (key equality is exact only for small steps)
            if (rr.flags & REC_WIDE) {
                bool b = false;
                if (valid && k > 0) eval_sample(rr, k - 1, nx - st - 1, px, py, pz, b);
                same = x == px && y == py && z == pz;
            } else {
                same = voxel_key(x, y, z) == carry;
            }
        } else {
            same = x == px && y == py && z == pz;
        }
        carry = __shfl_sync(0xffffffffu, voxel_key(x, y, z), 31);
        const bool keep = valid && (k == 0 || !same);
        {
            const unsigned mask = __ballot_sync(0xffffffffu, keep);
            const int rank = running + __popc(mask & lt);
            if (EMIT) {
                if (keep) {
                    uint32_t* d = stage + 3 * rank;
                    d[0] = (uint32_t)x;
                    d[1] = (uint32_t)y;
                    d[2] = (uint32_t)z;
                }
                if (valid && k == 0) a.chain_off[e] = pos + rank;  // chain start
            }
            running += __popc(mask);
        }
        ++j;
    }
    if (bad) record_error(a.ctl, bad_seg, 2);
    return running;
}

// Pass 1: kept voxels of every warp range, counted by kCountSplit warps per range (the count
// pass needs no shared memory, so it can run more warps than the emit pass has ranges).
constexpr int kCountSplit = 2;

// Two-pass geometry: host-given, or ("deferred", total_samples < 0) derived from the capacity the
// plan kernel left in off[nseg] -- the same arithmetic the host uses (vxg_api.cu
// emit_list_device). Returns false (nothing to do) if the plan recorded an error.
__device__ __forceinline__ bool list_geometry(const ListArgs& a, long long& total,
                                              long long& range_len) {
    if (a.total_samples >= 0) {
        total = a.total_samples;
        range_len = a.range_len;
        return true;
    }
    if (*reinterpret_cast<const volatile long long*>(&a.plan_ctl->err_seg) != 0 ||
        *reinterpret_cast<const volatile int*>(&a.plan_ctl->abort) != 0)
        return false;
    total = __ldg(a.off + a.nseg);
    const long long blocks = (total + a.range_len - 1) / a.range_len;
    range_len = (blocks + a.nranges - 1) / a.nranges * a.range_len;
    return range_len > 0;
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 4) list_count_kernel(ListArgs a) {
    const int lane = threadIdx.x & 31;
    const long long q = (long long)blockIdx.x * NW + (threadIdx.x >> 5);
    const long long r = q / kCountSplit;
    if (r >= a.nranges) return;
    long long total, range_len;
    if (!list_geometry(a, total, range_len)) {
        if (lane == 0) a.range_cnt[q] = 0;
        return;
    }
    const long long r0 = r * range_len, r1 = min(r0 + range_len, total);
    const long long part = ((range_len / kCountSplit) + 31) & ~31ll;  // whole rows
    const long long f0 = min(r0 + (q % kCountSplit) * part, r1);
    const long long f1 = (q % kCountSplit) == kCountSplit - 1 ? r1 : min(f0 + part, r1);
    long long cnt = 0;
    if (f0 < f1) {  // one walk over the whole part: fast runs span whole segments
        Walk W;
        walk_start(a, f0, W);
        cnt = walk_block<(1 << 30), false>(a, W, f0, f1, nullptr, 0);
    }
    if (lane == 0) a.range_cnt[q] = cnt;
}

// Exclusive prefix of the range counts (one CTA of 1024 threads, any number of ranges).
__global__ void __launch_bounds__(1024) range_scan_kernel(ListArgs a) {
    __shared__ long long s_warp[33];
    __shared__ long long s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (long long base = 0; base < a.nranges; base += 1024) {
        const long long i = base + tid;
        long long v = 0;
        if (i < a.nranges)
            for (int h = 0; h < kCountSplit; ++h) v += a.range_cnt[kCountSplit * i + h];
        long long incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const long long x = s_warp[lane];
            long long xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long t = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += t;
            }
            s_warp[lane] = xi - x;
            if (lane == 31) s_warp[32] = xi;
        }
        __syncthreads();
        if (i < a.nranges) a.range_pre[i] = s_carry + s_warp[warp] + incl - v;
        __syncthreads();
        if (tid == 0) s_carry += s_warp[32];
        __syncthreads();
    }
    if (tid == 0) {
        a.range_pre[a.nranges] = s_carry;
        if (a.chain_off) a.chain_off[a.nseg] = s_carry;  // (count only: no list)
        a.ctl->total = s_carry;
    }
}

// Pass 2: the same ranges again, now from their known output positions. The block's output
// position is known before it is walked, so the records are staged at the global address's
// offset mod 16: the 16-B-aligned middle of the block's output then leaves shared memory in ONE
// bulk copy (cp.async.bulk, the TMA engine), only the head and tail words go through registers.
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(ssrc);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int NW, int IPT>
__global__ void __launch_bounds__(NW * 32, 3) list_emit_kernel(ListArgs a) {
    constexpr int CH = 32 * IPT;
    constexpr int REGION = 3 * CH + 4;  // words per warp: records + up to 3 words of skew
    extern __shared__ __align__(16) uint32_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long r = (long long)blockIdx.x * NW + warp;
    if (r >= a.nranges) return;
    long long total, range_len;
    if (!list_geometry(a, total, range_len)) return;
    const long long f0 = r * range_len, f1 = min(f0 + range_len, total);
    if (f0 >= f1) return;
    uint32_t* region = smem + warp * REGION;
    long long pos = __ldg(a.range_pre + r);
    if (__ldg(a.range_pre + r + 1) > a.out_cap) {  // caller's buffer too small: write nothing
        if (lane == 0) record_error(a.ctl, 0, 4);
        return;
    }
    Walk W;
    walk_start(a, f0, W);
    for (long long b = f0; b < f1; b += CH) {
        const uintptr_t g0 = reinterpret_cast<uintptr_t>(a.out) + 12ull * (unsigned long long)pos;
        const int skew = (int)((g0 & 15u) >> 2);  // stage word i <-> global word g0/4 + i
        uint32_t* stage = region + skew;
        // the previous block's bulk copy must have read the staging before it is rewritten
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        const int cnt = walk_block<IPT, true>(a, W, b, min(b + CH, f1), stage, pos);
        const uintptr_t g1 = g0 + 12ull * (unsigned)cnt;
        const uintptr_t a0 = (g0 + 15) & ~(uintptr_t)15;
        const uintptr_t a1 = g1 & ~(uintptr_t)15;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // STS -> async proxy
        __syncwarp();
        if (a1 > a0) {
            const int hw = (int)((a0 - g0) >> 2), tw = (int)((g1 - a1) >> 2);
            if (lane == 0) bulk_store(reinterpret_cast<void*>(a0), stage + hw, (unsigned)(a1 - a0));
            if (lane < hw) reinterpret_cast<uint32_t*>(g0)[lane] = stage[lane];
            else if (lane >= 4 && lane - 4 < tw)
                reinterpret_cast<uint32_t*>(a1)[lane - 4] =
                    stage[hw + (int)((a1 - a0) >> 2) + (lane - 4)];
        } else {
            const int nw = (int)((g1 - g0) >> 2);  // fewer than 8 words
            if (lane < nw) reinterpret_cast<uint32_t*>(g0)[lane] = stage[lane];
        }
        pos += cnt;
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ONE kernel for both passes, overlapping them: every warp takes tasks from two in-order queues
// over finer ranges -- "count range r" and "emit range r" -- keeping the counts up to LA ranges
// ahead of the emits. A count task publishes its range's kept count (decoupled look-back status
// word, flag A); an emit task waits for its own count, resolves its prefix by look-back (the
// counts are already there) and publishes its inclusive prefix (flag P) before streaming its
// records out exactly as list_emit_kernel does. The count pass (FP64/issue-bound) and the emit
// pass (HBM-write-bound) share every SM instead of running back to back.
// Progress: an emit task whose count has not been claimed claims counts itself until it has, so
// a warp never waits on work nobody owns; count tasks never wait.
template <int NW, int IPT>
__global__ void __launch_bounds__(NW * 32, 3) list_fused_kernel(ListArgs a) {
    constexpr int CH = 32 * IPT;
    constexpr int REGION = 3 * CH + 4;
    extern __shared__ __align__(16) uint32_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* region = smem + warp * REGION;
    unsigned long long* cticket = &a.ctl->tile_counter;
    unsigned long long* eticket = reinterpret_cast<unsigned long long*>(&a.ctl->pad0);
    const long long R = a.nranges;
    auto count_range = [&](long long r) {
        const long long f0 = r * a.range_len, f1 = min(f0 + a.range_len, a.total_samples);
        long long cnt = 0;
        if (f0 < f1) {
            Walk W;
            walk_start(a, f0, W);
            cnt = walk_block<(1 << 30), false>(a, W, f0, f1, nullptr, 0);
        }
        if (lane == 0) lookback_publish(a.status, r, cnt);
    };
    for (;;) {
        // ---- choose: a count task while the counts are less than LA ranges ahead
        long long task = 0;
        int kind = 1;
        if (lane == 0) {
            const unsigned long long c = ld_relaxed_u64(cticket), e = ld_relaxed_u64(eticket);
            if ((long long)c < R && c < e + a.lookahead) {
                const unsigned long long t = atomicAdd(cticket, 1ull);
                if ((long long)t < R) {
                    kind = 0;
                    task = (long long)t;
                }
            }
            if (kind) task = (long long)atomicAdd(eticket, 1ull);
        }
        kind = __shfl_sync(0xffffffffu, kind, 0);
        task = __shfl_sync(0xffffffffu, task, 0);
        if (kind == 0) {
            count_range(task);
            continue;
        }
        const long long r = task;
        if (r >= R) break;
        // ---- make sure range r's count is owned by someone (claim counts up to r ourselves)
        while (true) {
            unsigned long long c = 0;
            if (lane == 0) c = ld_relaxed_u64(cticket);
            c = __shfl_sync(0xffffffffu, c, 0);
            if ((long long)c > r) break;
            unsigned long long t = 0;
            if (lane == 0) t = atomicAdd(cticket, 1ull);
            t = __shfl_sync(0xffffffffu, t, 0);
            if ((long long)t < R) count_range((long long)t);
        }
        // ---- own count (flag A or P set by its count task), then the prefix by look-back
        unsigned long long sw = 0;
        if (lane == 0) {
            unsigned spins = 0;
            while (((sw = ld_relaxed_u64(&a.status[r])) >> 62) == 0) {
                __nanosleep(64);
                if (++spins > (1u << 24)) {  // watchdog: report instead of hanging the GPU
                    atomicExch(&a.ctl->abort, 1);
                    break;
                }
            }
        }
        sw = __shfl_sync(0xffffffffu, sw, 0);
        const long long cnt = (long long)(sw & kValMask);
        const long long pre = lookback_resolve(a.status, r, cnt, a.ctl);
        if (r == R - 1 && lane == 0) {  // the last range knows the total
            a.chain_off[a.nseg] = pre + cnt;
            a.ctl->total = pre + cnt;
        }
        if (pre + cnt > a.out_cap) {  // caller's buffer too small: write nothing
            if (lane == 0) record_error(a.ctl, 0, 4);
            continue;
        }
        // ---- emit range r from its known output position (as list_emit_kernel)
        const long long f0 = r * a.range_len, f1 = min(f0 + a.range_len, a.total_samples);
        long long pos = pre;
        Walk W;
        if (f0 < f1) walk_start(a, f0, W);
        for (long long b = f0; b < f1; b += CH) {
            const uintptr_t g0 = reinterpret_cast<uintptr_t>(a.out) + 12ull * (unsigned long long)pos;
            const int skew = (int)((g0 & 15u) >> 2);
            uint32_t* stage = region + skew;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
            const int cn = walk_block<IPT, true>(a, W, b, min(b + CH, f1), stage, pos);
            const uintptr_t g1 = g0 + 12ull * (unsigned)cn;
            const uintptr_t a0 = (g0 + 15) & ~(uintptr_t)15;
            const uintptr_t a1 = g1 & ~(uintptr_t)15;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (a1 > a0) {
                const int hw = (int)((a0 - g0) >> 2), tw = (int)((g1 - a1) >> 2);
                if (lane == 0) bulk_store(reinterpret_cast<void*>(a0), stage + hw, (unsigned)(a1 - a0));
                if (lane < hw) reinterpret_cast<uint32_t*>(g0)[lane] = stage[lane];
                else if (lane >= 4 && lane - 4 < tw)
                    reinterpret_cast<uint32_t*>(a1)[lane - 4] =
                        stage[hw + (int)((a1 - a0) >> 2) + (lane - 4)];
            } else {
                const int nw = (int)((g1 - g0) >> 2);
                if (lane < nw) reinterpret_cast<uint32_t*>(g0)[lane] = stage[lane];
            }
            pos += cn;
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// =============================================================================== emit: bitmap
// Same row walker over a flat sample space of entries (segments, or clipped in-slab k-ranges);
// every sample voxel inside [0,V)^2 x [z_lo,z_hi) sets its bit.
template <int NW, int IPT, bool CLIP>
__global__ void __launch_bounds__(NW * 32) emit_bitmap_kernel(BitmapArgs a) {
    constexpr int CH = 32 * IPT;
    constexpr int TS = CH * NW;
    __shared__ long long s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = (long long)atomicAdd(&a.ctl->tile_counter, 1ull);
    __syncthreads();
    const long long tile = s_tile;
    const long long t0 = tile * TS;
    const long long tend = min(t0 + (long long)TS, a.total_samples);
    const long long e_lo = __ldg(a.tile_seg + tile);
    const long long e_hi = (tile + 1 < a.ntiles) ? __ldg(a.tile_seg + tile + 1) : a.n_entries - 1;
    const long long wbase = t0 + (long long)warp * CH;
    if (wbase >= tend) return;

    const unsigned long long V = (unsigned long long)a.V;
    RowWalker w;
    walker_init(w, a.off, e_lo, e_hi, wbase);
    long long cur = -1, seg = 0, ka = 0, kspan = 0, N = 0;
    // Must be initialised: with an indeterminate loop-carried record the compiler is free to
    // (and did) reuse the registers of r.ex/ey/ez as sample temporaries, so a later k == N
    // sample of a cached entry read the previous voxel instead of round(E).
    SegRec r{};
    bool bad = false;
    long long bad_seg = 0;
    unsigned long long outside = 0;
    for (int j = 0; j < IPT; ++j) {
        const long long row_start = wbase + (long long)j * 32;
        if (row_start >= tend) break;
        long long e, st, nx;
        walker_row(w, a.off, a.n_entries, row_start, e, st, nx);
        const long long f = row_start + lane;
        long long word = -1;
        unsigned long long bit = 0;
        if (f < tend) {
            if (e != cur) {
                cur = e;
                if (CLIP) {
                    const ClipEntry ce = a.entries[e];
                    seg = ce.seg;
                    ka = ce.ka;
                    kspan = ce.kb - ce.ka;
                    N = ce.n;
                } else {
                    seg = e;
                    ka = 0;
                    N = nx - st - 1;
                    kspan = N;
                }
                r = load_rec(a.rec + seg);
            }
            const long long loc = f - st;
            const long long k = loc < kspan ? ka + loc : N;
            int32_t x, y, z;
            bool b = false;
            eval_sample(r, k, N, x, y, z, b);
            if (b) {
                bad = true;
                bad_seg = seg;
            }
            if ((unsigned long long)(long long)x < V && (unsigned long long)(long long)y < V &&
                (unsigned long long)(long long)z < V) {
                if (z >= a.z_lo && z < a.z_hi) {
                    const unsigned long long bi =
                        (unsigned long long)x +
                        V * ((unsigned long long)y + V * (unsigned long long)(z - a.z_lo));
                    word = (long long)(bi >> 6);
                    bit = 1ull << (bi & 63);
                }
            } else {
                ++outside;
            }
        }
        // Consecutive samples of a segment share a word in contiguous lane runs: OR the run's
        // bits into its head lane with a segmented shuffle-down reduction (lanes of other runs
        // with the same word may be folded in too, which is harmless for an OR), then one RED
        // per run head. (__match_any + __reduce_or_sync with per-group masks is avoided: its
        // divergent lowering dropped bits when a lone lane shared a row with an idle group.)
        const unsigned wk = word >= 0 ? (unsigned)word : 0xffffffffu;  // slab words < 2^32 - 1
        unsigned long long v = bit;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long vn = __shfl_down_sync(0xffffffffu, v, o);
            const unsigned kn = __shfl_down_sync(0xffffffffu, wk, o);
            if (lane + o < 32 && kn == wk) v |= vn;
        }
        const unsigned kp = __shfl_up_sync(0xffffffffu, wk, 1);
        if (word >= 0 && (lane == 0 || kp != wk))
            atomicOr(reinterpret_cast<unsigned long long*>(a.words) + word, v);
    }
    if (bad) record_error(a.ctl, bad_seg, 2);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) outside += __shfl_xor_sync(0xffffffffu, outside, o);
    if (lane == 0 && outside) atomicAdd(&a.ctl->outside, outside);
}

// =============================================================================== launchers
// list launch shape: NW warps per CTA, IPT rows of 32 samples per staged block (staging
// NW * (32 * IPT * 12 + 16) B of shared memory per emit CTA: 8 x 24 -> 74 KB, 3 CTAs per SM).
constexpr int kListNW = 8, kListIPT = 24;

template <typename K>
static int resident_ctas(K kernel, int threads, size_t smem, int num_sms) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    return (per_sm < 1 ? 1 : per_sm) * num_sms;
}

int list_block_samples() { return 32 * kListIPT; }

// Function attributes and occupancy are per device: cached per device id (a process may drive
// several contexts on different GPUs), under a lock.
constexpr int kMaxDevices = 64;
static std::mutex g_attr_mu;

static int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d < 0 || d >= kMaxDevices ? 0 : d;
}

// One range per resident emit warp (the count pass uses the same ranges).
long long list_ranges(int num_sms) {
    static long long n[kMaxDevices] = {};
    const int dev = current_device();
    std::lock_guard<std::mutex> g(g_attr_mu);
    if (!n[dev]) {
        const size_t smem = (size_t)kListNW * (3 * 32 * kListIPT + 4) * 4;
        cudaFuncSetAttribute(list_emit_kernel<kListNW, kListIPT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        n[dev] = (long long)resident_ctas(list_emit_kernel<kListNW, kListIPT>, kListNW * 32, smem,
                                          num_sms) * kListNW;
    }
    return n[dev];
}

int list_resident_warps(int num_sms) { return (int)list_ranges(num_sms); }

cudaError_t launch_list_count(const ListArgs& a, cudaStream_t s) {
    const unsigned grid = (unsigned)((a.nranges * kCountSplit + kListNW - 1) / kListNW);
    list_count_kernel<kListNW><<<grid, kListNW * 32, 0, s>>>(a);
    range_scan_kernel<<<1, 1024, 0, s>>>(a);
    return cudaGetLastError();
}

// Fused launch: persistent CTAs (as many as fit), ranges = a.nranges (finer than one per warp).
constexpr int kFusedIPT = 24;  // 768-sample blocks (16 lost to spills and block overhead: measured)
int list_fused_block_samples() { return 32 * kFusedIPT; }

cudaError_t launch_list_fused(const ListArgs& a, int num_sms, cudaStream_t s) {
    const size_t smem = (size_t)kListNW * (3 * 32 * kFusedIPT + 4) * 4;
    static int per_sm_dev[kMaxDevices] = {};
    const int dev = current_device();
    int per_sm;
    {
        std::lock_guard<std::mutex> g(g_attr_mu);
        if (!per_sm_dev[dev]) {
            cudaFuncSetAttribute(list_fused_kernel<kListNW, kFusedIPT>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            int p = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p, list_fused_kernel<kListNW, kFusedIPT>,
                                                          kListNW * 32, smem);
            per_sm_dev[dev] = p < 1 ? 1 : p;
        }
        per_sm = per_sm_dev[dev];
    }
    list_fused_kernel<kListNW, kFusedIPT><<<(unsigned)(per_sm * num_sms), kListNW * 32, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_list_emit(const ListArgs& a, cudaStream_t s) {
    const unsigned grid = (unsigned)((a.nranges + kListNW - 1) / kListNW);
    const size_t smem = (size_t)kListNW * (3 * 32 * kListIPT + 4) * 4;
    list_emit_kernel<kListNW, kListIPT><<<grid, kListNW * 32, smem, s>>>(a);
    return cudaGetLastError();
}

// ======================================================================== single chain
// voxelize_parametric (src/parametric.cpp:28-40) of ONE segment in ONE launch: plan, samples,
// dedup and compaction in a single CTA, the chain written straight into mapped pinned host
// memory -- the latency regime of config 2 and of the reference harness's per-segment
// "sequential" method, where the batch path's plan readback + count/scan/emit launches would
// dominate. Each thread evaluates its sample and its predecessor (no cross-thread dependency);
// chunks of 1024 samples are compacted with a block-wide ballot scan.
__global__ void __launch_bounds__(1024) single_chain_kernel(SingleArgs a) {
    __shared__ int s_warp[33];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Plan pl;
    if (!make_plan(a.seg[0], a.seg[1], a.seg[2], a.seg[3], a.seg[4], a.seg[5], pl)) {
        if (tid == 0) record_error(a.ctl, 0, 2);
        return;
    }
    SegRec r;
    r.sx = a.seg[0];
    r.sy = a.seg[1];
    r.sz = a.seg[2];
    r.wx = pl.wx;
    r.wy = pl.wy;
    r.wz = pl.wz;
    r.ex = pl.ex;
    r.ey = pl.ey;
    r.ez = pl.ez;
    r.flags = rec_flags(a.seg[0], a.seg[1], a.seg[2], a.seg[3], a.seg[4], a.seg[5]);
    const long long N = pl.n, samples = N + 1;
    if (samples > a.max_samples) {  // the host's bound was wrong: nothing written, host reroutes
        if (tid == 0) a.ctl->n_entries = samples;
        return;
    }
    bool bad = false;
    long long running = 0;
    for (long long base = 0; base < samples; base += 1024) {
        const long long k = base + tid;
        bool keep = false;
        int32_t x = 0, y = 0, z = 0;
        if (k < samples) {
            eval_sample(r, k, N, x, y, z, bad);
            keep = true;
            if (k > 0) {
                int32_t px, py, pz;
                eval_sample(r, k - 1, N, px, py, pz, bad);
                keep = x != px || y != py || z != pz;
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_warp[warp] = __popc(m);
        __syncthreads();
        if (warp == 0) {
            const int v = s_warp[lane];
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            s_warp[lane] = incl - v;
            if (lane == 31) s_warp[32] = incl;
        }
        __syncthreads();
        const long long rank = running + s_warp[warp] + __popc(m & ((1u << lane) - 1u));
        if (keep && rank < a.cap) {
            int32_t* d = a.out + 3 * rank;
            d[0] = x;
            d[1] = y;
            d[2] = z;
        }
        running += s_warp[32];
        __syncthreads();
    }
    if (bad) record_error(a.ctl, 0, 2);
    if (tid == 0) {
        a.ctl->total = running;
        a.ctl->max_steps = (unsigned long long)N;
    }
}

cudaError_t launch_single_chain(const SingleArgs& a, cudaStream_t s) {
    single_chain_kernel<<<1, 1024, 0, s>>>(a);
    return cudaGetLastError();
}

// voxelize_parametric of one long chain in one launch (the batch path's plan readback + count /
// scan / emit launches dominate a single segment's ~10 us of work). CTA t (claimed in order)
// takes samples [t * 8192, (t + 1) * 8192): thread 0 plans the segment (make_plan,
// src/parametric.cpp:8-26) into shared memory, each thread evaluates its kLongP samples (1024
// apart) once and holds the voxels in registers; a sample is kept when it is k = 0 or its voxel
// differs from its predecessor's (src/batch.cpp:139-142) -- the lane before (shuffle), the last
// lane of the warp before / the row before (shared memory), or, for the CTA's first sample, the
// voxel thread 0 evaluates for it. The CTA's count goes through the decoupled look-back (one
// window: 123 CTAs for 10^6 samples), then the kept voxels are written in order.
constexpr int kLongThreads = 1024, kLongP = 8, kLongWarps = kLongThreads / 32;
constexpr int kLongGroups = kLongP * kLongWarps;  // (row, warp) groups, scanned 8 per lane
static_assert(kLongGroups == 256, "the offsets scan below takes 8 groups per lane");

__global__ void __launch_bounds__(kLongThreads) long_chain_kernel(LongArgs a) {
    __shared__ int s_off[kLongGroups];    // kept voxels per (row p, warp), then offsets
    __shared__ int s_last[kLongGroups][3];  // voxel of each group's last lane
    __shared__ int s_prev[3];               // voxel of the sample before the CTA's first
    __shared__ SegRec s_rec;
    __shared__ long long s_tile, s_pre, s_n;
    __shared__ int s_ok, s_agg;
    extern __shared__ __align__(16) uint32_t s_stage[];  // the CTA's output: 3 * 8192 + 4 words
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_tile = (long long)atomicAdd(&a.ctl->tile_counter, 1ull);
        Plan pl;
        s_ok = make_plan(a.seg[0], a.seg[1], a.seg[2], a.seg[3], a.seg[4], a.seg[5], pl);
        SegRec r;
        r.sx = a.seg[0];
        r.sy = a.seg[1];
        r.sz = a.seg[2];
        r.wx = pl.wx;
        r.wy = pl.wy;
        r.wz = pl.wz;
        r.ex = pl.ex;
        r.ey = pl.ey;
        r.ez = pl.ez;
        r.flags = rec_flags(a.seg[0], a.seg[1], a.seg[2], a.seg[3], a.seg[4], a.seg[5]);
        s_rec = r;
        s_n = pl.n;
    }
    __syncthreads();
    const long long tile = s_tile;
    if (!s_ok) {
        if (tid == 0 && tile == 0) record_error(a.ctl, 0, 2);
        return;
    }
    const long long N = s_n, samples = N + 1;
    if (samples > a.max_samples) {  // the host's bound was wrong: nothing written, host reroutes
        if (tid == 0 && tile == 0) a.ctl->n_entries = samples;
        return;
    }
    const SegRec r = s_rec;
    const long long base = tile * (kLongThreads * kLongP);
    bool bad = false;
    if (tid == 0 && base > 0 && base < samples)
        eval_sample(r, base - 1, N, s_prev[0], s_prev[1], s_prev[2], bad);
    int32_t vx[kLongP], vy[kLongP], vz[kLongP];
#pragma unroll
    for (int p = 0; p < kLongP; ++p) {
        const long long k = base + p * kLongThreads + tid;
        vx[p] = vy[p] = vz[p] = 0;
        if (k < samples) eval_sample(r, k, N, vx[p], vy[p], vz[p], bad);
        if (lane == 31) {
            s_last[p * kLongWarps + warp][0] = vx[p];
            s_last[p * kLongWarps + warp][1] = vy[p];
            s_last[p * kLongWarps + warp][2] = vz[p];
        }
    }
    if (bad) record_error(a.ctl, 0, 2);
    __syncthreads();
    unsigned keep = 0;
#pragma unroll
    for (int p = 0; p < kLongP; ++p) {
        const long long k = base + p * kLongThreads + tid;
        int32_t px = __shfl_up_sync(0xffffffffu, vx[p], 1);
        int32_t py = __shfl_up_sync(0xffffffffu, vy[p], 1);
        int32_t pz = __shfl_up_sync(0xffffffffu, vz[p], 1);
        if (lane == 0) {  // the group before in sample order, or the CTA's predecessor sample
            const int g = p * kLongWarps + warp - 1;
            const int* q = g >= 0 ? s_last[g] : s_prev;
            px = q[0];
            py = q[1];
            pz = q[2];
        }
        const bool kp = k < samples && (k == 0 || vx[p] != px || vy[p] != py || vz[p] != pz);
        keep |= (unsigned)kp << p;
        const unsigned m = __ballot_sync(0xffffffffu, kp);
        if (lane == 0) s_off[p * kLongWarps + warp] = __popc(m);
    }
    __syncthreads();
    if (warp == 0) {  // offsets of the groups in sample order; the CTA's look-back
        int v[8];
        int sum = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            v[i] = s_off[8 * lane + i];
            sum += v[i];
        }
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        int run = incl - sum;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            s_off[8 * lane + i] = run;
            run += v[i];
        }
        const long long agg = __shfl_sync(0xffffffffu, incl, 31);
        if (lane == 0) lookback_publish(a.status, tile, agg);
        const long long pre = lookback_resolve(a.status, tile, agg, a.ctl);
        if (lane == 0) {
            s_pre = pre;
            s_agg = (int)agg;
            if (tile == (long long)gridDim.x - 1) {  // the last CTA: the chain's length
                a.ctl->total = pre + agg;
                a.ctl->max_steps = (unsigned long long)N;
            }
        }
    }
    __syncthreads();
    // The CTA's voxels are one contiguous run of the output: staged in shared memory at the
    // global address's offset mod 16, the aligned middle leaves in ONE bulk copy (TMA), the head
    // and tail words through registers (as list_emit_kernel does per warp).
    const long long pre = s_pre;
    const long long cnt = max(0ll, min((long long)s_agg, a.cap - pre));  // (ranks past cap: dropped)
    const uintptr_t g0 = reinterpret_cast<uintptr_t>(a.out) + 12ull * (unsigned long long)pre;
    uint32_t* stage = s_stage + (int)((g0 & 15u) >> 2);  // stage word i <-> global word g0/4 + i
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int p = 0; p < kLongP; ++p) {
        const bool kp = (keep >> p) & 1u;
        const unsigned m = __ballot_sync(0xffffffffu, kp);
        const int rank = s_off[p * kLongWarps + warp] + __popc(m & lt);
        if (kp && rank < cnt) {
            uint32_t* d = stage + 3 * rank;
            d[0] = (uint32_t)vx[p];
            d[1] = (uint32_t)vy[p];
            d[2] = (uint32_t)vz[p];
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // STS -> async proxy
    __syncthreads();
    const uintptr_t g1 = g0 + 12ull * (unsigned long long)cnt;
    const uintptr_t a0 = (g0 + 15) & ~(uintptr_t)15, a1 = g1 & ~(uintptr_t)15;
    if (a1 > a0) {
        const int hw = (int)((a0 - g0) >> 2), tw = (int)((g1 - a1) >> 2);
        if (tid == 0) {
            bulk_store(reinterpret_cast<void*>(a0), stage + hw, (unsigned)(a1 - a0));
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        } else if (tid >= 32 && tid - 32 < hw) {
            reinterpret_cast<uint32_t*>(g0)[tid - 32] = stage[tid - 32];
        } else if (tid >= 64 && tid - 64 < tw) {
            reinterpret_cast<uint32_t*>(a1)[tid - 64] = stage[hw + (int)((a1 - a0) >> 2) + (tid - 64)];
        }
    } else if (tid < (int)((g1 - g0) >> 2)) {  // (fewer than 8 words)
        reinterpret_cast<uint32_t*>(g0)[tid] = stage[tid];
    }
}

long long long_chain_samples_per_cta() { return kLongThreads * kLongP; }

cudaError_t launch_long_chain(const LongArgs& a, long long ctas, cudaStream_t s) {
    constexpr size_t smem = (3 * (size_t)kLongThreads * kLongP + 4) * 4;
    static bool set_dev[kMaxDevices] = {};
    const int dev = current_device();
    {
        std::lock_guard<std::mutex> g(g_attr_mu);
        if (!set_dev[dev]) {
            cudaFuncSetAttribute(long_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
            set_dev[dev] = true;
        }
    }
    long_chain_kernel<<<(unsigned)ctas, kLongThreads, smem, s>>>(a);
    return cudaGetLastError();
}

int bitmap_tile_log2() { return 12; }

cudaError_t launch_emit_bitmap(const BitmapArgs& a, bool clip, cudaStream_t s) {
    if (clip) emit_bitmap_kernel<8, 16, true><<<(unsigned)a.ntiles, 256, 0, s>>>(a);
    else emit_bitmap_kernel<8, 16, false><<<(unsigned)a.ntiles, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace vxg
