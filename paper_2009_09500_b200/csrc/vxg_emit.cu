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
// Two passes over fixed chunks of CH = 32*IPT consecutive flat samples (the paper's
// N_P x (N_max + 1) grid without redundant items), batch_voxelize's kernel and assemble phases
// (src/batch.cpp:107-150) fused:
//   list_count_kernel : kept (deduplicated) voxels per chunk -- pure compute, no shared memory
//   scan_counts       : exclusive prefix of the counts (decoupled look-back, vxg_kernels.cu)
//   list_emit_kernel  : recompute the chunk knowing its output position, stage the kept voxels in
//                       shared memory at their final 16-B alignment and stream them out with one
//                       TMA bulk store (cp.async.bulk) plus 4-B head/tail words
// Recomputing the samples costs ~13 FP64 ops per sample and buys a pass without any inter-warp
// waiting (a single-pass look-back stalls on predecessors and needs double-buffered staging).
//
// A warp walks its chunk in rows of 32 consecutive samples. Rows without an entry boundary (most
// rows: config-4 segments are ~1000 samples long) take the fast path: one warp-uniform record,
// t = (row_start - so_c) + lane, S + W*t, llround, and a keep flag from comparing the voxel key
// with the neighbour lane's (lane 0: the previous row's lane 31). The k == N (E) sample always
// lies in a boundary row. Boundary rows, partial rows and records that need checked rounding or
// exact comparison take the generic path through the row walker.

// Walker state carried from one chunk to the next consecutive one (same warp): the entry of the
// next sample, its record and the key of the last sample.
struct WalkCtx {
    RowWalker w;
    SegRec R;       // record of entry w.c (warp-uniform)
    int32_t carry;  // voxel key of the sample before the next row (if in entry w.c)
    bool valid;
};

template <int IPT>
__device__ __forceinline__ void walk_init(const ListArgs& a, long long chunk, WalkCtx& wc) {
    constexpr int CH = 32 * IPT;
    const long long wbase = chunk * CH;
    RowWalker& w = wc.w;
    w.c = __ldg(a.tile_seg + chunk);  // entry containing the chunk's first sample
    w.so_c = __ldg(a.off + w.c);
    w.so_next = __ldg(a.off + w.c + 1);
    wc.R = load_rec(a.rec + w.c);
    wc.carry = 0;
    if (wbase > w.so_c) {
        int32_t px, py, pz;
        bool b = false;
        eval_sample(wc.R, wbase - 1 - w.so_c, w.so_next - w.so_c - 1, px, py, pz, b);
        wc.carry = voxel_key(px, py, pz);
    }
    wc.valid = true;
}

// Walk one chunk. EMIT: stage kept voxels at stage + 12*rank and keep per-row masks / bases
// (lane j holds row j's) for the chain offsets. Returns the chunk's kept count (warp-uniform).
template <int IPT, bool EMIT>
__device__ __forceinline__ int walk_chunk(const ListArgs& a, long long chunk, WalkCtx& wc,
                                          unsigned char* stage, unsigned& my_mask,
                                          int& my_rowbase) {
    constexpr int CH = 32 * IPT;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const long long wbase = chunk * CH;
    const long long wend = min(wbase + (long long)CH, a.total_samples);
    if (!wc.valid) walk_init<IPT>(a, chunk, wc);
    RowWalker& w = wc.w;
    SegRec& R = wc.R;
    int32_t& carry = wc.carry;
    bool bad = false;
    long long bad_seg = 0;
    const double lane_d = (double)lane;
    int running = 0;

    auto commit = [&](int j, bool keep, int32_t x, int32_t y, int32_t z) {
        const unsigned mask = __ballot_sync(0xffffffffu, keep);
        if (EMIT) {
            if (keep) {
                uint32_t* d = reinterpret_cast<uint32_t*>(stage + 12 * (running + __popc(mask & lt)));
                d[0] = (uint32_t)x;
                d[1] = (uint32_t)y;
                d[2] = (uint32_t)z;
            }
            if (lane == j) {
                my_mask = mask;
                my_rowbase = running;
            }
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
            const bool first0 = lane == 0 && row_start == w.so_c;  // k == 0 at lane 0, row 0
            if (R.flags & REC_POS) {
#pragma unroll 2
                for (int f = 0; f < nfast; ++f) {
                    const int32_t x = round_pos(sample_axis(R.sx, R.wx, t));
                    const int32_t y = round_pos(sample_axis(R.sy, R.wy, t));
                    const int32_t z = round_pos(sample_axis(R.sz, R.wz, t));
                    const int32_t key = voxel_key(x, y, z);
                    int32_t pk = __shfl_up_sync(0xffffffffu, key, 1);
                    if (lane == 0) pk = carry;
                    carry = __shfl_sync(0xffffffffu, key, 31);
                    commit(j + f, key != pk || (f == 0 && first0), x, y, z);
                    t = __dadd_rn(t, 32.0);
                }
            } else {
#pragma unroll 2
                for (int f = 0; f < nfast; ++f) {
                    const int32_t x = round_fast(sample_axis(R.sx, R.wx, t));
                    const int32_t y = round_fast(sample_axis(R.sy, R.wy, t));
                    const int32_t z = round_fast(sample_axis(R.sz, R.wz, t));
                    const int32_t key = voxel_key(x, y, z);
                    int32_t pk = __shfl_up_sync(0xffffffffu, key, 1);
                    if (lane == 0) pk = carry;
                    carry = __shfl_sync(0xffffffffu, key, 31);
                    commit(j + f, key != pk || (f == 0 && first0), x, y, z);
                    t = __dadd_rn(t, 32.0);
                }
            }
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
        int32_t x = 0, y = 0, z = 0, px = 0, py = 0, pz = 0;
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
        commit(j, valid && (k == 0 || !same), x, y, z);
        // (the walker may step one past the last entry at the end of the sample space)
        if (w.c != c_before && w.c < a.nseg) R = load_rec(a.rec + w.c);
        ++j;
    }
    if (bad) record_error(a.ctl, bad_seg, 2);
    // the walker now stands at sample wend: valid for chunk + 1 unless this was the last chunk
    wc.valid = wend == wbase + CH && w.c < a.nseg;
    return running;
}

// Pass 1: one warp per G consecutive chunks (walker carried across them).
template <int NW, int IPT, int G>
__global__ void __launch_bounds__(NW * 32) list_count_kernel(ListArgs a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long first = ((long long)blockIdx.x * NW + warp) * G;
    if (first >= a.nchunks) return;
    WalkCtx wc;
    wc.valid = false;
    unsigned m;
    int rb;
    for (int q = 0; q < G; ++q) {
        const long long chunk = first + q;
        if (chunk >= a.nchunks) break;
        const int cnt = walk_chunk<IPT, false>(a, chunk, wc, nullptr, m, rb);
        if (lane == 0) a.counts[chunk] = cnt;
    }
}

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(ssrc);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Pass 2: one warp per chunk; the chunk's output position is known before it starts.
template <int NW, int IPT>
__global__ void __launch_bounds__(NW * 32) list_emit_kernel(ListArgs a) {
    constexpr int CH = 32 * IPT;
    constexpr int REGION = CH * 12 + 16;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long chunk = (long long)blockIdx.x * NW + warp;
    if (chunk >= a.nchunks) return;
    unsigned char* region = smem + warp * REGION;
    const long long prefix = __ldg(a.chunk_prefix + chunk);
    const uintptr_t g0 = reinterpret_cast<uintptr_t>(a.out) + 12ull * (unsigned long long)prefix;
    const int head = (int)(g0 & 15u);
    unsigned char* stage = region + head;  // stage byte b <-> global byte g0 + b, same mod 16
    WalkCtx wc;
    wc.valid = false;
    unsigned my_mask = 0;
    int my_rowbase = 0;
    const long long wbase = chunk * CH;
    const long long wend = min(wbase + (long long)CH, a.total_samples);
    walk_init<IPT>(a, chunk, wc);
    const long long c_first = wc.w.c;
    const int count = walk_chunk<IPT, true>(a, chunk, wc, stage, my_mask, my_rowbase);
    const long long c_last = wc.w.c;
    const long long last = prefix + count;
    if (last > a.out_cap) {  // caller's buffer too small: report, write nothing
        if (lane == 0) record_error(a.ctl, c_first, 4);
        return;
    }
    // chain offsets of the entries whose k = 0 sample lies in the chunk (always kept)
    for (long long q0 = c_first; q0 <= c_last; q0 += 32) {
        const long long q = q0 + lane;
        const long long st = q <= c_last && q < a.nseg ? __ldg(a.off + q) : -1;
        const bool in = st >= wbase && st < wend;
        const int loc = in ? (int)(st - wbase) : 0;
        const unsigned mk = __shfl_sync(0xffffffffu, my_mask, loc >> 5);
        const int rb = __shfl_sync(0xffffffffu, my_rowbase, loc >> 5);
        if (in) a.chain_off[q] = prefix + rb + __popc(mk & ((1u << (loc & 31)) - 1u));
    }
    if (wend == a.total_samples && lane == 0) {
        a.chain_off[a.nseg] = last;
        a.ctl->total = last;
    }
    // stream out: global bytes [g0, g1); the 16-B aligned middle by one bulk copy
    const uintptr_t g1 = g0 + 12ull * (unsigned)count;
    const uintptr_t a0 = (g0 + 15) & ~(uintptr_t)15;
    const uintptr_t a1 = g1 & ~(uintptr_t)15;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // STS -> async proxy
    __syncwarp();
    if (a1 > a0) {
        if (lane == 0) {
            bulk_store(reinterpret_cast<void*>(a0), stage + (a0 - g0), (unsigned)(a1 - a0));
        }
        // head words [g0, a0) and tail words [a1, g1)
        const int hw = (int)((a0 - g0) >> 2), tw = (int)((g1 - a1) >> 2);
        if (lane < hw)
            reinterpret_cast<uint32_t*>(g0)[lane] = reinterpret_cast<const uint32_t*>(stage)[lane];
        else if (lane >= 4 && lane - 4 < tw)
            reinterpret_cast<uint32_t*>(a1)[lane - 4] =
                reinterpret_cast<const uint32_t*>(stage + (a1 - g0))[lane - 4];
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    } else {
        const int nw = (int)((g1 - g0) >> 2);  // fewer than 8 words
        if (lane < nw)
            reinterpret_cast<uint32_t*>(g0)[lane] = reinterpret_cast<const uint32_t*>(stage)[lane];
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
// list launch shape: NW warps per block, IPT rows per chunk (CH = 32*IPT samples), G chunks per
// counting warp. variant 0 = 8 x 16 x 4 (512-sample chunks, 6 KB staging per warp),
// 1 = 8 x 32 x 2 (1024-sample chunks, 12 KB), 2 = 8 x 8 x 8 (256, 3 KB).
template <int NW, int IPT, int G>
static cudaError_t launch_list_t(const ListArgs& a, int phase, cudaStream_t s) {
    if (phase == 0) {
        const long long warps = (a.nchunks + G - 1) / G;
        list_count_kernel<NW, IPT, G><<<(unsigned)((warps + NW - 1) / NW), NW * 32, 0, s>>>(a);
    } else {
        const size_t smem = (size_t)NW * (32 * IPT * 12 + 16);
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(list_emit_kernel<NW, IPT>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            attr = true;
        }
        list_emit_kernel<NW, IPT><<<(unsigned)((a.nchunks + NW - 1) / NW), NW * 32, smem, s>>>(a);
    }
    return cudaGetLastError();
}

int list_chunk_log2(int variant) {
    switch (variant) {
        case 1: return 10;
        case 2: return 8;
        default: return 9;
    }
}

cudaError_t launch_list_phase(const ListArgs& a, int variant, int phase, cudaStream_t s) {
    switch (variant) {
        case 1: return launch_list_t<8, 32, 2>(a, phase, s);
        case 2: return launch_list_t<8, 8, 8>(a, phase, s);
        default: return launch_list_t<8, 16, 4>(a, phase, s);
    }
}

int bitmap_tile_log2() { return 12; }

cudaError_t launch_emit_bitmap(const BitmapArgs& a, bool clip, cudaStream_t s) {
    if (clip) emit_bitmap_kernel<8, 16, true><<<(unsigned)a.ntiles, 256, 0, s>>>(a);
    else emit_bitmap_kernel<8, 16, false><<<(unsigned)a.ntiles, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace vxg
