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
// Persistent, software-pipelined warps. Each warp claims groups of K consecutive chunks of
// CH = 32*IPT samples. For every chunk it walks the rows, keeps a sample iff its voxel differs
// from the previous sample's (k == 0 always kept), compacts the kept voxels into one of its two
// shared-memory buffers and publishes the chunk's count (decoupled look-back, flag A). Only
// after computing the NEXT chunk does it resolve the previous chunk's output position, write the
// chain offsets of the segments starting in it and stream it out with 16-B stores: by then its
// predecessors have long published, so the look-back rarely spins.
//
// Rows without an entry boundary (most rows: config-4 segments are ~1000 samples long) take a
// fast path: one warp-uniform record, t = (row_start - so_c) + lane, S + W*t, llround, compare
// with the neighbour lane. The k == N (E) sample always lies in a boundary row. Boundary rows,
// partially valid rows and records that need checked rounding take the generic path.
struct ChunkState {
    long long chunk, wbase, wend, c_first, c_last;
    int count;
    unsigned mask;  // lane j: keep mask of row j
    int rowbase;    // lane j: kept voxels before row j
};

template <int IPT>
__device__ __forceinline__ void list_compute(const ListArgs& a, long long chunk,
                                             unsigned char* region, ChunkState& cs) {
    constexpr int CH = 32 * IPT;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int32_t* reg32 = reinterpret_cast<int32_t*>(region);
    const long long wbase = chunk * CH;
    const long long wend = min(wbase + (long long)CH, a.total_samples);
    const long long e_lo = __ldg(a.tile_seg + chunk);
    const long long e_hi = chunk + 1 < a.nchunks ? __ldg(a.tile_seg + chunk + 1) : a.nseg - 1;
    RowWalker w;
    walker_init(w, a.off, e_lo, e_hi, wbase);
    cs.chunk = chunk;
    cs.wbase = wbase;
    cs.wend = wend;
    cs.c_first = w.c;
    SegRec R = load_rec(a.rec + w.c);  // record of entry w.c (warp-uniform)

    // voxel of sample wbase - 1 when it belongs to the same entry (lane 0's previous sample)
    int32_t cx = 0, cy = 0, cz = 0;
    bool bad = false;
    long long bad_seg = 0;
    if (wbase > w.so_c) {
        bool b = false;
        eval_sample(R, wbase - 1 - w.so_c, w.so_next - w.so_c - 1, cx, cy, cz, b);
    }
    const double lane_d = (double)lane;
    int running = 0;
    unsigned my_mask = 0;
    int my_rowbase = 0;
#pragma unroll 1
    for (int j = 0; j < IPT; ++j) {
        const long long row_start = wbase + (long long)j * 32;
        if (row_start >= wend) break;
        int32_t x, y, z;
        bool keep;
        if (w.so_next > row_start + 32 && row_start + 32 <= wend && !(R.flags & REC_CHECK)) {
            // ---- fast path: 32 consecutive samples of one entry, none of them the last
            const double t = __dadd_rn(__ll2double_rn(row_start - w.so_c), lane_d);
            x = round_fast(sample_axis(R.sx, R.wx, t));
            y = round_fast(sample_axis(R.sy, R.wy, t));
            z = round_fast(sample_axis(R.sz, R.wz, t));
            int32_t px = __shfl_up_sync(0xffffffffu, x, 1);
            int32_t py = __shfl_up_sync(0xffffffffu, y, 1);
            int32_t pz = __shfl_up_sync(0xffffffffu, z, 1);
            if (lane == 0) {
                px = cx;
                py = cy;
                pz = cz;
            }
            keep = (lane == 0 && row_start == w.so_c) || x != px || y != py || z != pz;
        } else {
            // ---- generic path
            const long long c_before = w.c;
            long long e, st, nx;
            walker_row(w, a.off, a.nseg, row_start, e, st, nx);
            const long long f = row_start + lane;
            const bool valid = f < wend;
            long long k = 0;
            x = y = z = 0;
            if (valid) {
                const SegRec rr = e == c_before ? R : load_rec(a.rec + e);
                k = f - st;
                bool b = false;
                eval_sample(rr, k, nx - st - 1, x, y, z, b);
                if (b) {
                    bad = true;
                    bad_seg = e;
                }
            }
            int32_t px = __shfl_up_sync(0xffffffffu, x, 1);
            int32_t py = __shfl_up_sync(0xffffffffu, y, 1);
            int32_t pz = __shfl_up_sync(0xffffffffu, z, 1);
            if (lane == 0) {
                px = cx;
                py = cy;
                pz = cz;
            }
            keep = valid && (k == 0 || x != px || y != py || z != pz);
            // (the walker may step one past the last entry at the end of the sample space)
            if (w.c != c_before && w.c < a.nseg) R = load_rec(a.rec + w.c);
        }
        cx = __shfl_sync(0xffffffffu, x, 31);
        cy = __shfl_sync(0xffffffffu, y, 31);
        cz = __shfl_sync(0xffffffffu, z, 31);
        const unsigned mask = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            int32_t* d = reg32 + 3 * (running + __popc(mask & lt));
            d[0] = x;
            d[1] = y;
            d[2] = z;
        }
        if (lane == j) {
            my_mask = mask;
            my_rowbase = running;
        }
        running += __popc(mask);
    }
    if (bad) record_error(a.ctl, bad_seg, 2);
    cs.c_last = w.c;
    cs.count = running;
    cs.mask = my_mask;
    cs.rowbase = my_rowbase;
}

template <int IPT>
__device__ __forceinline__ void list_finish(const ListArgs& a, const ChunkState& cs,
                                            const unsigned char* region) {
    const int lane = threadIdx.x & 31;
    const long long prefix = (a.debug & 1)
                                 ? cs.wbase
                                 : lookback_resolve(a.status, cs.chunk, (long long)cs.count, a.ctl);
    // chain offsets of the entries whose k = 0 sample lies in the chunk (always kept)
    for (long long q0 = cs.c_first; q0 <= cs.c_last; q0 += 32) {
        const long long q = q0 + lane;
        const long long st = q <= cs.c_last ? __ldg(a.off + q) : -1;
        const bool in = st >= cs.wbase && st < cs.wend;
        const int loc = in ? (int)(st - cs.wbase) : 0;
        const unsigned mk = __shfl_sync(0xffffffffu, cs.mask, loc >> 5);
        const int rb = __shfl_sync(0xffffffffu, cs.rowbase, loc >> 5);
        if (in) a.chain_off[q] = prefix + rb + __popc(mk & ((1u << (loc & 31)) - 1u));
    }
    if (cs.wend == a.total_samples && lane == 0) {
        a.chain_off[a.nseg] = prefix + cs.count;
        a.ctl->total = prefix + cs.count;
    }
    if (prefix + cs.count > a.out_cap) {
        if (lane == 0) record_error(a.ctl, cs.c_first, 4);
        __syncwarp();
        return;
    }
    // region bytes [0, 12*count) -> out + 12*prefix, 16-B stores, unaligned head/tail words
    const uintptr_t g0 = reinterpret_cast<uintptr_t>(a.out) + 12ull * (unsigned long long)prefix;
    const int head = (int)(g0 & 15u);
    const int nbytes = 12 * cs.count;
    const int nchunks = (head + nbytes + 15) >> 4;
    unsigned char* gbase = reinterpret_cast<unsigned char*>(g0 - (uintptr_t)head);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(region);
    for (int ch = lane; ch < nchunks; ch += 32) {
        const int lo = (ch << 4) - head;  // region byte of the 16-B chunk's first word
        if (lo >= 0 && lo + 16 <= nbytes) {
            uint4 v;
            v.x = src[(lo >> 2) + 0];
            v.y = src[(lo >> 2) + 1];
            v.z = src[(lo >> 2) + 2];
            v.w = src[(lo >> 2) + 3];
            st_stream_v4(gbase + (ch << 4), v);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int b = lo + 4 * q;
                if (b >= 0 && b < nbytes)
                    *reinterpret_cast<uint32_t*>(gbase + (ch << 4) + 4 * q) = src[b >> 2];
            }
        }
    }
    __syncwarp();  // the region may be overwritten by the warp's next chunk
}

// Persistent warps claim groups of K consecutive chunks. A warp computes and publishes ALL K
// chunks of its group (into K shared-memory buffers) before it resolves any of them, so the
// aggregate of every claimed chunk is published without waiting on anything: a resolution waits
// at most for chunks claimed earlier by other warps, never on a chain of resolutions (an
// interleaved compute/resolve order inside a group serialises the warps). Only the group's first
// resolution can wait; the others find their predecessor (the warp's own chunk) resolved.
template <int NWB, int IPT, int K, int MINB>
__global__ void __launch_bounds__(NWB * 32, MINB) emit_list_kernel(ListArgs a) {
    static_assert(IPT <= 32, "row bookkeeping is kept one row per lane");
    constexpr int CH = 32 * IPT;
    extern __shared__ __align__(16) unsigned char smem[];  // per warp: K buffers of CH*12 bytes
    __shared__ ChunkState s_state[NWB][K];                 // lane 0's scalars of each chunk
    __shared__ unsigned s_mask[NWB][K][IPT];
    __shared__ int s_rowbase[NWB][K][IPT];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* buf0 = smem + (size_t)warp * K * CH * 12;
    while (true) {
        long long g = 0;
        if (lane == 0) g = (long long)atomicAdd(&a.ctl->tile_counter, (unsigned long long)K);
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g >= a.nchunks) break;
        const int nq = (int)min((long long)K, a.nchunks - g);
        for (int q = 0; q < nq; ++q) {
            ChunkState cs;
            list_compute<IPT>(a, g + q, buf0 + q * CH * 12, cs);
            if (lane == 0) {
                if (!(a.debug & 1)) lookback_publish(a.status, g + q, cs.count);
                s_state[warp][q] = cs;
            }
            if (lane < IPT) {
                s_mask[warp][q][lane] = cs.mask;
                s_rowbase[warp][q][lane] = cs.rowbase;
            }
        }
        __syncwarp();
        for (int q = 0; q < nq; ++q) {
            ChunkState cs = s_state[warp][q];
            cs.mask = lane < IPT ? s_mask[warp][q][lane] : 0u;
            cs.rowbase = lane < IPT ? s_rowbase[warp][q][lane] : 0;
            list_finish<IPT>(a, cs, buf0 + q * CH * 12);
        }
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
template <int NWB, int IPT, int K, int MINB>
static cudaError_t launch_list_t(const ListArgs& a, cudaStream_t s) {
    const size_t smem = (size_t)NWB * K * 32 * IPT * 12;
    static int grid_cap = 0;
    if (!grid_cap) {
        cudaFuncSetAttribute(emit_list_kernel<NWB, IPT, K, MINB>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, emit_list_kernel<NWB, IPT, K, MINB>,
                                                      NWB * 32, smem);
        grid_cap = sms * (per_sm > 0 ? per_sm : 1);
    }
    const long long groups = (a.nchunks + (long long)NWB * K - 1) / ((long long)NWB * K);
    const int grid = (int)(groups < grid_cap ? groups : grid_cap);
    emit_list_kernel<NWB, IPT, K, MINB><<<grid > 0 ? grid : 1, NWB * 32, smem, s>>>(a);
    return cudaGetLastError();
}

// variant -> (warps per block, rows per chunk, chunks per claim, min blocks per SM):
//   0 = 4 x 16 x 2 x 4 (512-sample chunks, 12 KB smem per warp, 16 warps/SM)
//   1 = 4 x 8 x 4 x 4  (256-sample chunks, 12 KB per warp, 16 warps/SM)
//   2 = 4 x 8 x 2 x 8  (256, 6 KB per warp, 32 warps/SM, 64 registers)
//   3 = 8 x 16 x 2 x 2 (512, 12 KB per warp, 16 warps/SM)
//   4 = 4 x 16 x 1 x 8 (512, 6 KB per warp, one claim per chunk, 32 warps/SM)
int list_chunk_log2(int variant) {
    switch (variant) {
        case 1: return 8;
        case 2: return 8;
        default: return 9;
    }
}

cudaError_t launch_emit_list(const ListArgs& a, int variant, cudaStream_t s) {
    switch (variant) {
        case 1: return launch_list_t<4, 8, 4, 4>(a, s);
        case 2: return launch_list_t<4, 8, 2, 8>(a, s);
        case 3: return launch_list_t<8, 16, 2, 2>(a, s);
        case 4: return launch_list_t<4, 16, 1, 8>(a, s);
        default: return launch_list_t<4, 16, 2, 4>(a, s);
    }
}

int bitmap_tile_log2() { return 12; }

cudaError_t launch_emit_bitmap(const BitmapArgs& a, bool clip, cudaStream_t s) {
    if (clip) emit_bitmap_kernel<8, 16, true><<<(unsigned)a.ntiles, 256, 0, s>>>(a);
    else emit_bitmap_kernel<8, 16, false><<<(unsigned)a.ntiles, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace vxg
