// vxg_emit.cu -- the emit kernels: thread-per-sample evaluation of G_k = S + W*k over the flat
// (segment, k) sample space (the paper's N_P x (N_max + 1) grid without redundant items,
// SURVEY.md §2 row 3), writing either the deduplicated voxel list (batch_voxelize's kernel AND
// assemble phases, src/batch.cpp:107-150, fused) or an occupancy bitmap.
#include <cstdint>

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
// ONE pass fusing batch_voxelize's kernel and assemble phases (src/batch.cpp:107-150): every
// sample is evaluated once, duplicates are dropped in registers, and the kept voxels are
// compacted into the flat list with a single-pass decoupled look-back over CTA chunks.
//
// Persistent CTAs of NW warps take chunk tickets in order (atomic counter, so every smaller
// ticket is already owned by a running CTA: look-back forward progress). A chunk is NW warp
// sub-chunks of CH = 32*IPT consecutive flat samples. Each warp walks its sub-chunk in rows of 32
// samples, staging kept voxels (12-B records) in its shared-memory region at their chunk-local
// rank. The CTA then publishes the chunk's count, resolves its global position by look-back, and
// every warp streams its records out with 16-B vector stores (the global start of a sub-chunk has
// any 4-B alignment, so the aligned middle is assembled from 4 LDS.32 per vector).
//
// Rows without an entry boundary (most rows: config-4 segments are ~1000 samples long) take the
// fast path: one warp-uniform record, t = (row_start - so_c) + lane, S + W*t, llround, and a keep
// flag from comparing the voxel key with the previous lane's (lane 0: the previous row's lane 31).
// The k == N (E) sample always lies in a boundary row. Boundary rows, partial rows and records
// that need checked rounding or exact comparison take the generic path through the row walker.

// Start state of a warp sub-chunk: the entry containing its first sample, that entry's sample
// range and record, and the voxel key of the sample before it (the dedup carry). Prepared by the
// scan warp one round ahead so the walking warps start computing without a dependent load chain.
struct SubInit {
    long long c, so_c, so_next;
    int32_t carry;
    int32_t pad;
    SegRec R;
};

__device__ __forceinline__ void prepare_subchunk(const ListArgs& a, long long sub, int log2ch,
                                                 SubInit& si) {
    const long long wbase = sub << log2ch;
    si.c = __ldg(a.tile_seg + sub);
    si.so_c = __ldg(a.off + si.c);
    si.so_next = __ldg(a.off + si.c + 1);
    si.R = load_rec(a.rec + si.c);
    si.carry = 0;
    si.pad = 0;
    if (wbase > si.so_c) {
        int32_t px, py, pz;
        bool b = false;
        eval_sample(si.R, wbase - 1 - si.so_c, si.so_next - si.so_c - 1, px, py, pz, b);
        si.carry = voxel_key(px, py, pz);
    }
}

template <int IPT>
__device__ __forceinline__ int walk_subchunk(const ListArgs& a, long long sub, const SubInit& si,
                                             uint32_t* stage, long long& c_first,
                                             long long& c_last) {
    constexpr int CH = 32 * IPT;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const long long wbase = sub * CH;
    const long long wend = min(wbase + (long long)CH, a.total_samples);
    RowWalker w;
    w.c = si.c;
    w.so_c = si.so_c;
    w.so_next = si.so_next;
    c_first = w.c;
    SegRec R = si.R;
    int32_t carry = si.carry;  // voxel key of the sample before the next row (lane 0's predecessor)
    bool bad = false;
    long long bad_seg = 0;
    const double lane_d = (double)lane;
    int running = 0;

    auto commit = [&](bool keep, int32_t x, int32_t y, int32_t z) {
        const unsigned mask = __ballot_sync(0xffffffffu, keep);
        if (keep) {
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
        // ---- fast rows: row r is fast iff row_start_r + 32 <= min(so_next - 1, wend)
        const long long lim = min(w.so_next - 1, wend);
        int nfast = 0;
        if (!(R.flags & (REC_CHECK | REC_WIDE)) && lim >= row_start + 32)
            nfast = (int)min((lim - row_start) >> 5, (long long)(IPT - j));
        if (nfast > 0) {
            double t = __dadd_rn(__ll2double_rn(row_start - w.so_c), lane_d);
            // k == 0 (always kept) can only sit at lane 0 of the first fast row
            bool first = lane == 0 && row_start == w.so_c;
            if (first) a.chain_off[w.c] = running;  // chain start: chunk-local rank
            // lane 0's predecessor key arrives through a rotate: after row r, lane 0 holds lane
            // 31's key of row r, which is its predecessor in row r + 1
            int32_t prev0 = carry;
            if (R.flags & REC_POS) {
#pragma unroll 2
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
        // ---- generic row: entry boundaries, the k == N sample, partial rows, checked records
        const long long c_before = w.c;
        long long e, st, nx;
        walker_row(w, a.off, a.nseg, row_start, e, st, nx);
        const long long f = row_start + lane;
        const bool valid = f < wend;
        long long k = 0;
        int32_t x = 0, y = 0, z = 0, px, py, pz;
        SegRec rr = R;
        if (valid) {
            if (e != c_before) rr = load_rec(a.rec + e);
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
        {  // chain start (k == 0): the chunk-local rank now, rebased once the prefix is known
            const unsigned mask = __ballot_sync(0xffffffffu, keep);
            const int rank = running + __popc(mask & lt);
            if (keep) {
                uint32_t* d = stage + 3 * rank;
                d[0] = (uint32_t)x;
                d[1] = (uint32_t)y;
                d[2] = (uint32_t)z;
            }
            if (valid && k == 0) a.chain_off[e] = rank;
            running += __popc(mask);
        }
        // (the walker may step one past the last entry at the end of the sample space)
        if (w.c != c_before && w.c < a.nseg) R = load_rec(a.rec + w.c);
        ++j;
    }
    if (bad) record_error(a.ctl, bad_seg, 2);
    // the walker stands at sample wend: the last entry with a sample in [wbase, wend) is w.c,
    // or w.c - 1 if w.c starts exactly at wend (then it belongs to the next sub-chunk)
    c_last = w.so_c >= wend ? w.c - 1 : w.c;
    return running;
}

// Copy a warp's staged records (words [0, 3*cnt) of `stage`) to global bytes [g0, g0 + 12*cnt):
// 16-B vector stores for the aligned middle, single words for head and tail.
__device__ __forceinline__ void store_records(const uint32_t* stage, int cnt, char* g0p) {
    const int lane = threadIdx.x & 31;
    const uintptr_t g0 = reinterpret_cast<uintptr_t>(g0p);
    const uintptr_t g1 = g0 + 12ull * (unsigned)cnt;
    const uintptr_t a0 = (g0 + 15) & ~(uintptr_t)15;
    const uintptr_t a1 = g1 & ~(uintptr_t)15;
    if (a1 > a0) {
        const int hw = (int)((a0 - g0) >> 2);  // head words (0..3); stage word of a0 == hw
        const int nv = (int)((a1 - a0) >> 4);
        uint4* dst = reinterpret_cast<uint4*>(a0);
        for (int v = lane; v < nv; v += 32) {
            const uint32_t* src = stage + hw + 4 * v;
            uint4 q;
            q.x = src[0];
            q.y = src[1];
            q.z = src[2];
            q.w = src[3];
            st_stream_v4(dst + v, q);
        }
        const int tw = (int)((g1 - a1) >> 2);
        if (lane < hw)
            reinterpret_cast<uint32_t*>(g0)[lane] = stage[lane];
        else if (lane >= 4 && lane - 4 < tw)
            reinterpret_cast<uint32_t*>(a1)[lane - 4] = stage[hw + 4 * nv + (lane - 4)];
    } else {
        const int nw = (int)((g1 - g0) >> 2);  // fewer than 8 words
        if (lane < nw) reinterpret_cast<uint32_t*>(g0)[lane] = stage[lane];
    }
}

// Named barriers (ids 1..6, parity-double-buffered so a fast producer can never complete a
// phase meant for the previous round): the scan warp arrives, the walking warps sync, or back.
// (Immediate barrier ids keep ptxas from reserving all 16 hardware barriers.)
template <int ID, int N>
__device__ __forceinline__ void bar_sync_i() {
    asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(N) : "memory");
}
template <int ID, int N>
__device__ __forceinline__ void bar_arrive_i() {
    asm volatile("bar.arrive %0, %1;" ::"n"(ID), "n"(N) : "memory");
}
template <int ID, int N>
__device__ __forceinline__ void bar_sync(int parity) {
    if (parity) bar_sync_i<ID + 1, N>();
    else bar_sync_i<ID, N>();
}
template <int ID, int N>
__device__ __forceinline__ void bar_arrive(int parity) {
    if (parity) bar_arrive_i<ID + 1, N>();
    else bar_arrive_i<ID, N>();
}
constexpr int kBarTicket = 1, kBarCounts = 3, kBarPrefix = 5;  // + (round & 1)

// Persistent, warp-specialised CTAs: NW walking warps + 1 scan warp, pipelined over CTA chunks
// (look-back tiles) of NW warp sub-chunks.
//   walking warp, round i: wait for ticket T_i; walk its sub-chunk of T_i into staging buffer
//       i%2 and post the count (the last warp to finish publishes T_i's aggregate at once);
//       wait for T_{i-1}'s prefix; stream T_{i-1}'s records out of buffer (i-1)%2.
//   scan warp, round i: claim and hand out T_{i+1}; wait for T_i's counts; resolve T_i by
//       decoupled look-back (overlapping the walk of T_{i+1}); post T_i's per-warp prefixes.
// Tickets come from an atomic counter in claim order, and a chunk's aggregate is published as
// soon as it is walked; the walk of T_{i+1} waits only on the resolution of T_{i-1}, so every
// wait points at strictly smaller tickets: the look-back is deadlock-free.
template <int NW, int IPT>
__global__ void __launch_bounds__((NW + 1) * 32, 2) list_kernel(ListArgs a) {
    constexpr int CH = 32 * IPT;
    constexpr int NT = (NW + 1) * 32;
    constexpr int kLog2CH = IPT == 8 ? 8 : (IPT == 16 ? 9 : 10);
    static_assert(CH == (1 << kLog2CH), "sub-chunk size");
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ long long s_ticket[2];
    __shared__ int s_cnt[2][NW];
    __shared__ int s_done[2];
    __shared__ long long s_pre[2][NW];
    __shared__ SubInit s_init[2][NW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < 2) s_done[threadIdx.x] = 0;
    __syncthreads();

    if (warp == NW) {  // ------------------------------------------------ scan warp
        unsigned long long tk = 0;
        if (lane == 0) tk = atomicAdd(&a.ctl->tile_counter, 1ull);
        long long T = (long long)__shfl_sync(0xffffffffu, tk, 0);
        if (lane < NW && T < a.nchunks && T * NW + lane < a.nsub)
            prepare_subchunk(a, T * NW + lane, kLog2CH, s_init[0][lane]);
        if (lane == 0) s_ticket[0] = T;
        bar_arrive<kBarTicket, NT>(0);
        for (int i = 0; T < a.nchunks; ++i) {
            const int cur = i & 1;
            if (lane == 0) tk = atomicAdd(&a.ctl->tile_counter, 1ull);
            const long long Tn = (long long)__shfl_sync(0xffffffffu, tk, 0);
            if (lane < NW && Tn < a.nchunks && Tn * NW + lane < a.nsub)
                prepare_subchunk(a, Tn * NW + lane, kLog2CH, s_init[cur ^ 1][lane]);
            if (lane == 0) s_ticket[cur ^ 1] = Tn;
            bar_arrive<kBarTicket, NT>(cur ^ 1);
            bar_sync<kBarCounts, NT>(cur);
            const int v = lane < NW ? s_cnt[cur][lane] : 0;
            int incl = v;
#pragma unroll
            for (int o = 1; o < NW; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const long long agg = __shfl_sync(0xffffffffu, incl, NW - 1);
            const long long pre = lookback_resolve(a.status, T, agg, a.ctl);
            if (lane < NW) s_pre[cur][lane] = pre + (incl - v);
            if (lane == 0 && T == a.nchunks - 1) {  // the last chunk knows the total
                a.chain_off[a.nseg] = pre + agg;
                a.ctl->total = pre + agg;
            }
            bar_arrive<kBarPrefix, NT>(cur);
            T = Tn;
        }
        return;
    }
    // --------------------------------------------------------------------- walking warps
    uint32_t* const stage0 = smem + warp * (3 * CH);
    uint32_t* const stage1 = smem + (NW + warp) * (3 * CH);
    long long pc_first = 0, pc_last = -1;  // entry range of this warp's T_{i-1} sub-chunk
    long long t_prev = -1;
    for (int i = 0;; ++i) {
        const int cur = i & 1, prv = cur ^ 1;
        bar_sync<kBarTicket, NT>(cur);
        const long long T = s_ticket[cur];
        const bool live = T < a.nchunks;
        long long cc_first = 0, cc_last = -1;
        if (live) {
            const long long sub = T * NW + warp;
            int cnt = 0;
            if (sub < a.nsub)
                cnt = walk_subchunk<IPT>(a, sub, s_init[cur][warp], cur ? stage1 : stage0, cc_first,
                                         cc_last);
            if (lane == 0) {
                s_cnt[cur][warp] = cnt;
                __threadfence_block();
                if (atomicAdd(&s_done[cur], 1) == NW - 1) {  // last walker: publish the aggregate
                    __threadfence_block();
                    long long agg = 0;
#pragma unroll
                    for (int w = 0; w < NW; ++w) agg += *reinterpret_cast<volatile int*>(&s_cnt[cur][w]);
                    lookback_publish(a.status, T, agg);
                    s_done[cur] = 0;
                }
            }
            bar_arrive<kBarCounts, NT>(cur);
        }
        if (t_prev >= 0) {
            bar_sync<kBarPrefix, NT>(prv);
            const long long psub = t_prev * NW + warp;
            if (psub < a.nsub) {
                const long long P = s_pre[prv][warp];
                const int pcnt = s_cnt[prv][warp];
                if (P + pcnt > a.out_cap) {  // caller's buffer too small: report, write nothing
                    if (lane == 0) record_error(a.ctl, pc_first, 4);
                } else {
                    store_records(prv ? stage1 : stage0, pcnt,
                                  reinterpret_cast<char*>(a.out) + 12ll * P);
                    // rebase the chain offsets of entries whose k = 0 sample is in the sub-chunk
                    const long long wbase = psub * CH;
                    for (long long q = pc_first + lane; q <= pc_last; q += 32)
                        if (q > pc_first || __ldg(a.off + q) == wbase) a.chain_off[q] += P;
                }
            }
            __syncwarp();  // buffer (i-1)%2 is rewritten in round i+1
        }
        if (!live) break;
        t_prev = T;
        pc_first = cc_first;
        pc_last = cc_last;
    }
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
// list launch shape: NW warps per CTA, IPT rows of 32 samples per warp sub-chunk; staging is
// 2 * NW * 32 * IPT * 12 B of shared memory per CTA (double-buffered; 8 x 16: 96 KB).
constexpr int kListNW = 8, kListIPT = 16;

int list_sub_log2() { return 9; }  // 32 * kListIPT samples per warp sub-chunk
int list_nw() { return kListNW; }

cudaError_t launch_list(const ListArgs& a, int num_sms, cudaStream_t s) {
    const size_t smem = (size_t)2 * kListNW * 32 * kListIPT * 12;
    static int blocks_per_sm = 0;
    if (!blocks_per_sm) {
        cudaFuncSetAttribute(list_kernel<kListNW, kListIPT>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm,
                                                      list_kernel<kListNW, kListIPT>,
                                                      (kListNW + 1) * 32, smem);
        if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    long long grid = (long long)blocks_per_sm * num_sms;
    if (grid > a.nchunks) grid = a.nchunks;
    list_kernel<kListNW, kListIPT><<<(unsigned)grid, (kListNW + 1) * 32, smem, s>>>(a);
    return cudaGetLastError();
}

int bitmap_tile_log2() { return 12; }

cudaError_t launch_emit_bitmap(const BitmapArgs& a, bool clip, cudaStream_t s) {
    if (clip) emit_bitmap_kernel<8, 16, true><<<(unsigned)a.ntiles, 256, 0, s>>>(a);
    else emit_bitmap_kernel<8, 16, false><<<(unsigned)a.ntiles, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace vxg
