// vxg_bitmap.cu -- occupancy bitmap of a batch's samples, tile-binned through shared memory.
//
// The bitmap (bit b = x + V*(y + V*(z - z_lo)) of 64-bit words, include/voxgpu.h) of a 4096^3
// volume is 8 GiB, far beyond L2, and every sector of it is hit by dozens of unrelated segments:
// a global atomicOr per sample turns the write into random DRAM read-modify-write. Instead the
// volume is cut into tiles of TX x TY x TZ voxels (TX = 256: a tile row is one 32-B sector) that
// fit one CTA's shared memory, and the work is binned by tile:
//
//   tiles_count_kernel   walk every segment through the tiles it visits (each axis' rounded
//                        coordinate is monotone in k, so a segment's in-tile samples are one
//                        k-range, a "piece"), count pieces per tile and in-volume samples
//   tiles_scan_kernel    exclusive prefix of the per-tile piece counts
//   tiles_scatter_kernel walk again and write every piece into its tile's bin
//   tiles_fill_kernel    persistent CTAs claim tiles: OR every piece's sample voxels into the
//                        tile's shared-memory bits (shared atomics, no DRAM traffic), then OR the
//                        tile into the bitmap with full-sector 16-B accesses, once per tile
//
// Samples are evaluated exactly as the list path does (include/voxline/parametric.hpp:41-48,
// FMA-free, llround), so the set of bits equals the set of chain voxels of the reference.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "vxg_device.cuh"
#include "vxg_internal.h"

namespace vxg {

// Tile shape: 128 x 120 x 120 voxels (225.5 KB with the padding): near-cubic, so a segment crosses ~14
// tile faces instead of the ~17 of a 256 x 80 x 80 tile -- fewer pieces to bin and to fill
// (cfg5: binning 38.4 -> 32.6 ms, fill 86.7 -> 83.1 ms; 128 x 112 x 112 and 256 x 88 x 80 were
// in between). A row is 16 B of the bitmap, each tile's own (x0 is a multiple of 128).
constexpr int kTX = 128, kTY = 120, kTZ = 120;
constexpr int kRW = kTX / 32;          // 32-bit words per row
constexpr int kSS = kRW * kTY + 1;     // words per z-slice (padded by one: bank skew per z step)
constexpr int kTileWords = kSS * kTZ;

// 1/w (0 for w == 0) for the crossing guesses only -- every guess is verified by exact samples,
// so an approximate reciprocal will do: MUFU.RCP64H's ~20 bits and one Newton step (~40 bits),
// instead of the IEEE division sequence.
__device__ __forceinline__ double guess_rcp(double w) {
    if (w == 0.0) return 0.0;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(w));
    return __dmul_rn(r, __fma_rn(-w, r, 2.0));
}

// Exact rounded coordinate of sample k < N on one axis (any sign).
__device__ __forceinline__ long long axis_round(double s, double w, long long k) {
    return (long long)round_fast(sample_axis(s, w, __ll2double_rn(k)));
}

// First k in [lo, hi) with pred(k), hi if none; pred monotone (false...true) on [lo, hi).
// pred(k): dir > 0 -> round(s + w*k) >= B, dir < 0 -> round(s + w*k) < B.
// An analytic guess from the reciprocal (any error is fixed up exactly), a few exact steps, and a
// binary-search fallback.
__device__ __forceinline__ long long axis_cross(double s, double w, double inv_w, long long lo,
                                                long long hi, long long B, int dir) {
    if (lo >= hi) return hi;
    auto pred = [&](long long k) {
        const long long r = axis_round(s, w, k);
        return dir > 0 ? r >= B : r < B;
    };
    if (w == 0.0) return pred(lo) ? lo : hi;
    double gd = ((double)B - 0.5 - s) * inv_w;  // real k where s + w*k crosses B - 0.5
    gd = ceil(gd);
    gd = fmin(fmax(gd, (double)lo), (double)hi);
    long long g = (long long)gd;
    // the guess is almost always exact: two evaluations confirm it
    if ((g == hi || pred(g)) && (g == lo || !pred(g - 1))) return g;
    int steps = 0;
    while (g > lo && pred(g - 1) && steps < 3) {
        --g;
        ++steps;
    }
    while (g < hi && !pred(g) && steps < 6) {
        ++g;
        ++steps;
    }
    if ((g == hi || pred(g)) && (g == lo || !pred(g - 1))) return g;
    long long a = lo, b = hi;  // exact fallback
    while (a < b) {
        const long long m = a + ((b - a) >> 1);
        if (pred(m)) b = m;
        else a = m + 1;
    }
    return a;
}

// k-range [klo, khi) of samples k < N whose rounded coordinate on one axis lies in [lo, hi).
__device__ __forceinline__ void axis_range(double s, double w, double inv_w, long long N,
                                           long long lo, long long hi, long long& klo,
                                           long long& khi) {
    if (w >= 0.0) {
        klo = axis_cross(s, w, inv_w, 0, N, lo, +1);
        khi = axis_cross(s, w, inv_w, klo, N, hi, +1);
    } else {
        klo = axis_cross(s, w, inv_w, 0, N, hi, -1);
        khi = axis_cross(s, w, inv_w, klo, N, lo, -1);
    }
}

// Inside the box every coordinate is >= 0 (rounds > -0.5): the one-DADD rounding applies.
__device__ __forceinline__ long long axis_round_pos(double s, double w, long long k) {
    return (long long)round_pos(sample_axis(s, w, __ll2double_rn(k)));
}

// axis_cross for the tile walk: the samples of [lo, hi) are inside the box. The analytic guess is
// verified with two exact evaluations (it is right unless (B - 0.5 - s)/w is within a few ulp of
// an integer); anything else falls back to the exact search.
// 32-bit form of walk_cross for the tile walk (every N < 2^31 on the tile path).
__device__ __forceinline__ int walk_cross32(double s, double w, double inv_w, int lo, int hi, int B,
                                            int dir) {
    // ceil + a saturating conversion in one (NaN -> 0), clamped as integers; the samples' k as
    // doubles through the magic-number add (no I2F: the conversion pipe is the walk's slowest)
    const int g = min(max(__double2int_ru(__dmul_rn(small_to_double(B) - 0.5 - s, inv_w)), lo), hi);
    const int rg = g < hi ? round_pos(sample_axis(s, w, small_to_double(g))) : 0;
    const int rp = g > lo ? round_pos(sample_axis(s, w, small_to_double(g - 1))) : 0;
    const bool at = g == hi || (dir > 0 ? rg >= B : rg < B);
    const bool before = g == lo || !(dir > 0 ? rp >= B : rp < B);
    if (at && before) return g;
    return (int)axis_cross(s, w, inv_w, lo, hi, B, dir);
}

__device__ __forceinline__ long long walk_cross(double s, double w, double inv_w, long long lo,
                                                long long hi, long long B, int dir) {
    double gd = ceil(((double)B - 0.5 - s) * inv_w);
    gd = fmin(fmax(gd, (double)lo), (double)hi);
    const long long g = (long long)gd;
    const long long rg = g < hi ? axis_round_pos(s, w, g) : 0;
    const long long rp = g > lo ? axis_round_pos(s, w, g - 1) : 0;
    const bool at = g == hi || (dir > 0 ? rg >= B : rg < B);
    const bool before = g == lo || !(dir > 0 ? rp >= B : rp < B);
    if (at && before) return g;
    return axis_cross(s, w, inv_w, lo, hi, B, dir);
}

constexpr int kWalkThreads = 256;  // block size of the kernels that walk (the shared columns)

// Visit the pieces of one segment inside the box [0,V)^2 x [z_lo,z_hi): sink(tile, ka, len, hasE)
// for every maximal k-range in one tile (hasE: its last sample is k = N, i.e. E itself).
// Also returns the number of the segment's samples inside [0, V)^3 (for the outside count).
// Written to keep a warp's lanes (one segment each) on one instruction stream: every step
// advances exactly one axis through one verified crossing, with the axis chosen by selects.
template <typename Sink>
__device__ __forceinline__ long long walk_pieces(const SegRec& r, long long N, const TileArgs& g,
                                                 Sink&& sink) {
    const double invx = guess_rcp(r.wx);
    const double invy = guess_rcp(r.wy);
    const double invz = guess_rcp(r.wz);
    const bool e_vol = r.ex >= 0 && r.ex < g.V && r.ey >= 0 && r.ey < g.V && r.ez >= 0 &&
                       r.ez < g.V;
    // S itself is sample 0 (S + W*0 == S); sample N-1 (not E, which may sit a rounding away)
    // bounds the monotone k < N samples on every axis.
    const long long nl = N > 0 ? N - 1 : 0;
    const long long s0x = axis_round(r.sx, r.wx, 0), s0y = axis_round(r.sy, r.wy, 0),
                    s0z = axis_round(r.sz, r.wz, 0);
    const long long slx = axis_round(r.sx, r.wx, nl), sly = axis_round(r.sy, r.wy, nl),
                    slz = axis_round(r.sz, r.wz, nl);
    const bool s_vol = s0x >= 0 && s0x < g.V && s0y >= 0 && s0y < g.V && s0z >= 0 && s0z < g.V;
    const bool l_vol = slx >= 0 && slx < g.V && sly >= 0 && sly < g.V && slz >= 0 && slz < g.V;
    long long klo, khi, inside;
    long long az0 = 0, az1 = N;
    if (s_vol && l_vol && e_vol) {  // the whole segment is inside the volume
        inside = N + 1;
        if (g.z_lo > 0 || g.z_hi < g.V) axis_range(r.sz, r.wz, invz, N, g.z_lo, g.z_hi, az0, az1);
        klo = az0;
        khi = az1;
    } else {
        long long ax0, ax1, ay0, ay1;
        axis_range(r.sx, r.wx, invx, N, 0, g.V, ax0, ax1);
        axis_range(r.sy, r.wy, invy, N, 0, g.V, ay0, ay1);
        klo = max(ax0, ay0);
        khi = min(ax1, ay1);
        inside = 0;
        if (klo < khi) {
            long long v0, v1;
            axis_range(r.sz, r.wz, invz, N, 0, g.V, v0, v1);
            inside = max(0ll, min(khi, v1) - max(klo, v0));
            if (g.z_lo == 0 && g.z_hi == g.V) {
                az0 = v0;
                az1 = v1;
            } else {
                axis_range(r.sz, r.wz, invz, N, g.z_lo, g.z_hi, az0, az1);
            }
            klo = max(klo, az0);
            khi = min(khi, az1);
        }
        if (e_vol) ++inside;
    }
    const bool e_in = e_vol && r.ez >= g.z_lo && r.ez < g.z_hi;
    long long last_tile = -1, last_ka = 0, last_end = -1;
    if (klo < khi) {
        // 32-bit walk (the tile path requires every N < 2^31): per axis the direction, the next
        // tile boundary B and the first k past it (khi: none); the tile id moves by strides.
        const int k0 = (int)klo, k1 = (int)khi;
        constexpr int tsz[3] = {kTX, kTY, kTZ};  // (compile-time: divisions by constants)
        const int org[3] = {0, 0, (int)g.z_lo};
        const int stride[3] = {1, (int)g.ntx, (int)(g.ntx * g.nty)};
        const double sa[3] = {r.sx, r.sy, r.sz}, wa[3] = {r.wx, r.wy, r.wz},
                     ia[3] = {invx, invy, invz};
        // Per-axis state in shared memory, this thread's column: the step below picks the axis
        // that crosses next by index (3 shared loads) instead of selecting among registers
        // (~20 selects per step, a quarter of the walk's instructions).
        __shared__ double sh_d[3][3][kWalkThreads];  // [axis][s, w, 1/w][thread]
        __shared__ int sh_i[3][3][kWalkThreads];     // [axis][next boundary, boundary step, tile step]
        const int tt = threadIdx.x;
        int nx[3];
        int tile = 0;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const int q = (int)(axis_round_pos(sa[i], wa[i], k0) - org[i]) / tsz[i];
            const int qe = (int)(axis_round_pos(sa[i], wa[i], k1 - 1) - org[i]) / tsz[i];
            const int dr = qe > q ? 1 : (qe < q ? -1 : 0);  // (an axis that stays never crosses)
            tile += q * stride[i];
            const int Bn = org[i] + (dr > 0 ? q + 1 : q) * tsz[i];
            nx[i] = dr != 0 ? walk_cross32(sa[i], wa[i], ia[i], k0, k1, Bn, dr) : k1;
            sh_d[i][0][tt] = sa[i];
            sh_d[i][1][tt] = wa[i];
            sh_d[i][2][tt] = ia[i];
            sh_i[i][0][tt] = Bn;
            sh_i[i][1][tt] = dr * tsz[i];
            sh_i[i][2][tt] = dr * stride[i];
        }
        int k = k0;
        while (true) {
            const int kn = min(nx[0], min(nx[1], nx[2]));
            if (kn > k) {  // (kn == k: two axes cross at once, the piece is empty)
                if (last_tile >= 0) sink(last_tile, last_ka, last_end - last_ka, false);
                last_tile = tile;
                last_ka = k;
                last_end = kn;
                k = kn;
            }
            if (k >= k1) break;
            // advance the (first) axis crossing at k: one crossing per step
            const int i = nx[0] == k ? 0 : (nx[1] == k ? 1 : 2);
            const int bstep = sh_i[i][1][tt];
            const int B = sh_i[i][0][tt] + bstep;
            sh_i[i][0][tt] = B;
            tile += sh_i[i][2][tt];
            const int nn = walk_cross32(sh_d[i][0][tt], sh_d[i][1][tt], sh_d[i][2][tt], k, k1, B,
                                        bstep > 0 ? 1 : -1);
            if (i == 0) nx[0] = nn;
            else if (i == 1) nx[1] = nn;
            else nx[2] = nn;
        }
    }
    if (e_in) {
        const long long tE = ((long long)((int)(r.ez - g.z_lo) / kTZ) * g.nty + r.ey / kTY) * g.ntx +
                             r.ex / kTX;
        if (last_tile == tE && last_end == N) {
            sink(last_tile, last_ka, last_end - last_ka + 1, true);
            last_tile = -1;
        } else {
            if (last_tile >= 0) sink(last_tile, last_ka, last_end - last_ka, false);
            last_tile = -1;
            sink(tE, N, 1, true);
        }
    }
    if (last_tile >= 0) sink(last_tile, last_ka, last_end - last_ka, false);
    return inside;
}

// Bins are (tile, length class): a tile's pieces are stored grouped by length (classes of 4
// samples), so the fill's warp steps, which run as long as their longest piece, get pieces of
// nearly equal length. A tile's bins are consecutive: its pieces are still one CSR range.
// (Round 1, exact fill: 8-sample classes 77.3 ms against 79.5 with 16-sample ones, for 1.7 ms
// more binning; round 2, fixed-point fill with one lane per piece: 4-sample classes 57.4 ms
// against 58.4 with 8, for 0.5 ms more binning.)
constexpr int kLenShift = 2;                   // class width 2^kLenShift samples
constexpr int kLenClasses = 256 >> kLenShift;  // (longer pieces share the last class)
__device__ __forceinline__ long long bin_of(long long tile, long long len) {
    return tile * kLenClasses + min((len - 1) >> kLenShift, (long long)(kLenClasses - 1));
}

__device__ __forceinline__ long long seg_steps(const TileArgs& g, long long i) {
    return __ldg(g.off + i + 1) - __ldg(g.off + i) - 1;
}
// N of a loaded record: records copied into walk order carry it above their flag bits.
__device__ __forceinline__ long long rec_steps(const TileArgs& g, const SegRec& r, long long i) {
    return g.rec_n ? (long long)(r.flags >> kRecNShift) : seg_steps(g, i);
}

// Walk order: segments grouped by length (8 buckets of N / 256; on a slab, of the estimated
// in-slab share, scaled to the slab's depth), so the 32 segments a warp walks in lock step have
// similar piece counts (the warp runs as long as its longest walk), and by coarse start cell
// (16^3). The perm pass copies the records into this order (perm_scatter_kernel). Swept on cfg5 (binning ms): no sort 41.5; 16^3 cells x {1, 2, 4, 8,
// 16, 32} length buckets 41.8, 35.4, 32.6, 32.2, 32.6, 33.5; {1, 4, 8, 12, 32}^3 cells x 32
// buckets 57.8, 36.2, 33.4, 33.4, 35.5; {20, 24}^3 cells x 16 buckets 32.8, 33.0.
constexpr int kLenBucketShift = 8;
constexpr int kLenBuckets = 2048 >> kLenBucketShift;
constexpr int kCellsPerAxis = 16;  // coarse spatial cells (16^3) of the box
constexpr int kPermKeys = kLenBuckets * kCellsPerAxis * kCellsPerAxis * kCellsPerAxis;
__device__ __forceinline__ int len_bucket(long long N) {
    return (int)min(N >> kLenBucketShift, (long long)kLenBuckets - 1);
}

// Walk-order key: length bucket (major) then the coarse cell of round(S) (minor). Lanes of a
// warp then walk equally long segments (the warp runs as long as its longest walk) that start
// near each other, so their pieces land in neighbouring bins (the scatter's writes and atomics
// stay L2-local).
__device__ __forceinline__ int perm_key(const TileArgs& g, long long i) {
    // (the order only steers performance: S's coarse cell from the record's first sector)
    const double2 sxy = __ldg(reinterpret_cast<const double2*>(g.rec + i));
    const double sz = __ldg(&g.rec[i].sz);
    auto cell = [](double v, double lo, double ext) {
        const int c = __double2int_rz(__dmul_rn(v - lo, (double)kCellsPerAxis / ext));
        return min(max(c, 0), kCellsPerAxis - 1);
    };
    const double V = (double)g.V;
    const int c = (cell(sz, (double)g.z_lo, (double)(g.z_hi - g.z_lo)) * kCellsPerAxis +
                   cell(sxy.y, 0.0, V)) * kCellsPerAxis + cell(sxy.x, 0.0, V);
    long long N = seg_steps(g, i);
    if (g.z_lo > 0 || g.z_hi < g.V) {
        // A slab: what a lane walks is the segment's share inside it -- estimate it from the z
        // overlap, in buckets scaled to the slab's depth (the shares are short), so a warp's
        // lanes walk alike.
        const double wz = __ldg(&g.rec[i].wz);
        const double z1 = sz + wz * (double)N;
        const double lo = fmin(sz, z1), hi = fmax(sz, z1);
        if (hi - lo > 1.0) {
            const double ov = fmin(hi, (double)g.z_hi) - fmax(lo, (double)g.z_lo);
            N = (long long)((double)N * fmax(ov, 0.0) / (hi - lo));
        }
        const long long depth = g.z_hi - g.z_lo;
        N <<= depth <= 256 ? 3 : depth <= 512 ? 2 : depth <= 1024 ? 1 : 0;
    }
    return len_bucket(N) * (kCellsPerAxis * kCellsPerAxis * kCellsPerAxis) + c;
}

__global__ void __launch_bounds__(256) perm_hist_kernel(TileArgs g) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= g.n) return;
    const long long i = g.sel ? (long long)g.sel[t] : t;  // (over a thin slab's selection)
    const int k = perm_key(g, i);
    // warp-aggregated: lanes with the same key add once
    const unsigned peers = __match_any_sync(__activemask(), k);
    if ((threadIdx.x & 31) == __ffs(peers) - 1)
        atomicAdd(reinterpret_cast<unsigned long long*>(g.perm_cur) + k,
                  (unsigned long long)__popc(peers));
}

// perm_cur[key] holds the bucket start on entry (perm_scan_kernel): positions by atomics.
__global__ void __launch_bounds__(256) perm_scatter_kernel(TileArgs g) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= g.n) return;
    const long long i = g.sel ? (long long)g.sel[t] : t;
    const int k = perm_key(g, i);
    const unsigned peers = __match_any_sync(__activemask(), k);
    const int leader = __ffs(peers) - 1;
    unsigned long long base = 0;
    if ((threadIdx.x & 31) == leader)
        base = atomicAdd(reinterpret_cast<unsigned long long*>(g.perm_cur) + k,
                         (unsigned long long)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    const unsigned below = peers & ((1u << (threadIdx.x & 31)) - 1u);
    const unsigned long long pos = base + __popc(below);
    if (g.prec) {  // the record itself moves: the passes after read it sequentially
        const uint4* q = reinterpret_cast<const uint4*>(g.rec + i);
        uint4* d = reinterpret_cast<uint4*>(g.prec + pos);
        const uint4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
        uint4 e = __ldg(q + 3);
        e.w = (e.w & ((1u << kRecNShift) - 1u)) | ((uint32_t)seg_steps(g, i) << kRecNShift);
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(d),
                     "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                     : "memory");
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(d + 2),
                     "r"(c.x), "r"(c.y), "r"(c.z), "r"(c.w), "r"(e.x), "r"(e.y), "r"(e.z), "r"(e.w)
                     : "memory");
    } else {
        g.perm[pos] = (int)i;
    }
}

// Exclusive prefix of the kPermKeys bucket counts, in place (one CTA).
__global__ void __launch_bounds__(1024) perm_scan_kernel(TileArgs g) {
    __shared__ long long s_warp[33];
    __shared__ long long s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int base = 0; base < kPermKeys; base += 1024) {
        const int i = base + tid;
        const long long v = g.perm_cur[i];
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
        g.perm_cur[i] = s_carry + s_warp[warp] + incl - v;
        __syncthreads();
        if (tid == 0) s_carry += s_warp[32];
        __syncthreads();
    }
}

__device__ __forceinline__ long long walk_segment(const TileArgs& g, long long t) {
    return g.perm ? (long long)__ldg(g.perm + t) : t;
}

// Thin z-slabs (one rank's share): the segments whose samples can reach [z_lo, z_hi), appended
// to a list the count and scatter passes walk instead of every segment (a conservative test:
// a few segments near the slab are walked for nothing). A skipped segment still adds its
// in-volume samples to the outside count (Control::total), as the count pass would have: N + 1
// when S and E are well inside the volume, else the same arithmetic as walk_pieces.
__global__ void __launch_bounds__(256) slab_select_kernel(TileArgs g, int* sel,
                                                          unsigned long long* nsel) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool keep = false;
    long long inside = 0;
    if (i < g.n) {
        // S and E only (no rounding): every sample lies between them (k < N: S + W*k with
        // |W*k| <= |E - S|, up to a few ulp) or is E itself, so its rounded z is within 1 of
        // [min(S.z, E.z), max(S.z, E.z)]; 2 planes of slack make the test conservative.
        const SegRec* p = g.rec + i;
        const double2 a = __ldg(reinterpret_cast<const double2*>(p));      // sx, sy
        const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);  // sz, wx
        const uint4 e = __ldg(reinterpret_cast<const uint4*>(p) + 3);      // ex, ey, ez, flags
        const double sx = a.x, sy = a.y, sz = b.x;
        const int ex = (int)e.x, ey = (int)e.y, ez = (int)e.z;
        const double zmin = fmin(sz, (double)ez), zmax = fmax(sz, (double)ez);
        keep = (zmax + 2.0 >= (double)g.z_lo && zmin - 2.0 < (double)g.z_hi) ||
               (e.w & (REC_CHECK | REC_WIDE));  // (caller plans: keep, the walk decides)
        if (!keep) {
            const double lo = 1.0, hi = (double)(g.V - 2);
            const bool s_in = sx >= lo && sx <= hi && sy >= lo && sy <= hi && sz >= lo && sz <= hi;
            const bool e_in = ex >= 1 && ex <= g.V - 2 && ey >= 1 && ey <= g.V - 2 && ez >= 1 &&
                              ez <= g.V - 2;
            const long long N = seg_steps(g, i);
            if (s_in && e_in) {
                inside = N + 1;  // every sample rounds into [0, V)^3
            } else {  // exactly, as walk_pieces does
                const SegRec r = load_rec(p);
                const long long nl = N > 0 ? N - 1 : 0;
                const bool e_vol = r.ex >= 0 && r.ex < g.V && r.ey >= 0 && r.ey < g.V &&
                                   r.ez >= 0 && r.ez < g.V;
                const long long s0x = axis_round(r.sx, r.wx, 0), s0y = axis_round(r.sy, r.wy, 0),
                                s0z = axis_round(r.sz, r.wz, 0);
                const long long slx = axis_round(r.sx, r.wx, nl), sly = axis_round(r.sy, r.wy, nl),
                                slz = axis_round(r.sz, r.wz, nl);
                const bool s_vol = s0x >= 0 && s0x < g.V && s0y >= 0 && s0y < g.V && s0z >= 0 &&
                                   s0z < g.V;
                const bool l_vol = slx >= 0 && slx < g.V && sly >= 0 && sly < g.V && slz >= 0 &&
                                   slz < g.V;
                if (s_vol && l_vol && e_vol) {
                    inside = N + 1;
                } else {
                    const double invx = guess_rcp(r.wx);
                    const double invy = guess_rcp(r.wy);
                    const double invz = guess_rcp(r.wz);
                    long long ax0, ax1, ay0, ay1, v0, v1;
                    axis_range(r.sx, r.wx, invx, N, 0, g.V, ax0, ax1);
                    axis_range(r.sy, r.wy, invy, N, 0, g.V, ay0, ay1);
                    const long long klo = max(ax0, ay0), khi = min(ax1, ay1);
                    if (klo < khi) {
                        axis_range(r.sz, r.wz, invz, N, 0, g.V, v0, v1);
                        inside = max(0ll, min(khi, v1) - max(klo, v0));
                    }
                    if (e_vol) ++inside;
                }
            }
        }
    }
    // one list append per block (a per-warp atomic on the single counter serialises: 2M of them)
    __shared__ unsigned s_cnt[8];
    __shared__ unsigned s_base;
    __shared__ unsigned long long s_inside;
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_inside = 0;
    if (lane == 0) s_cnt[warp] = __popc(m);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) inside += __shfl_xor_sync(0xffffffffu, inside, o);
    __syncthreads();
    if (lane == 0 && inside) atomicAdd(&s_inside, (unsigned long long)inside);
    if (threadIdx.x == 0) {
        unsigned tot = 0;
        for (int w = 0; w < 8; ++w) {
            const unsigned c = s_cnt[w];
            s_cnt[w] = tot;
            tot += c;
        }
        s_base = tot ? (unsigned)atomicAdd(nsel, (unsigned long long)tot) : 0u;
    }
    __syncthreads();
    if (keep) sel[s_base + s_cnt[warp] + __popc(m & ((1u << lane) - 1u))] = (int)i;
    if (threadIdx.x == 0 && s_inside)
        atomicAdd(reinterpret_cast<unsigned long long*>(&g.ctl->total), s_inside);
}

// Pass A: pieces per tile, in-volume samples.
// (256, 3): at most 80 registers, 3 CTAs per SM -- 84 registers round to 88 and leave 2 CTAs,
// 64 (4 CTAs) spill: cfg5 binning 35.5 / 32.3 / 33.2 ms for 2 / 3 / 4 CTAs (round 2)
#ifndef VXG_COUNT_MINB
#define VXG_COUNT_MINB 3
#endif
#ifndef VXG_SCATTER_MINB
#define VXG_SCATTER_MINB 4
#endif
__global__ void __launch_bounds__(256, VXG_COUNT_MINB) tiles_count_kernel(TileArgs g) {
    const long long tix = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long inside = 0, inbox = 0;
    if (tix < g.n) {
        const long long i = walk_segment(g, tix);
        const SegRec r = load_rec(g.rec + i);
        inside = walk_pieces(r, rec_steps(g, r, i), g, [&](long long t, long long, long long len, bool) {
            atomicAdd(reinterpret_cast<unsigned long long*>(g.tile_cnt) + bin_of(t, len), 1ull);
            inbox += len;
        });
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        inside += __shfl_xor_sync(0xffffffffu, inside, o);
        inbox += __shfl_xor_sync(0xffffffffu, inbox, o);
    }
    // block totals first: a per-warp atomic on the two single counters serialises in L2
    __shared__ unsigned long long s_sum[2];
    if (threadIdx.x == 0) s_sum[0] = s_sum[1] = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        if (inbox) atomicAdd(&s_sum[0], (unsigned long long)inbox);
        if (inside) atomicAdd(&s_sum[1], (unsigned long long)inside);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_sum[0]) atomicAdd(&g.ctl->outside, s_sum[0]);
        if (s_sum[1]) atomicAdd(reinterpret_cast<unsigned long long*>(&g.ctl->total), s_sum[1]);
    }
}

// Exclusive prefix of the (tile, class) piece counts (one CTA); tile_off[nbins] = total pieces.
__global__ void __launch_bounds__(1024) tiles_scan_kernel(TileArgs g) {
    __shared__ long long s_warp[33];
    __shared__ long long s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long nbins = g.ntiles * kLenClasses;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (long long base = 0; base < nbins; base += 1024) {
        const long long i = base + tid;
        const long long v = i < nbins ? g.tile_cnt[i] : 0;
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
        if (i < nbins) {
            g.tile_off[i] = s_carry + s_warp[warp] + incl - v;
            g.tile_cur[i] = (unsigned)(s_carry + s_warp[warp] + incl - v);  // scatter cursor
        }
        __syncthreads();
        if (tid == 0) s_carry += s_warp[32];
        __syncthreads();
    }
    if (tid == 0) {
        g.tile_off[nbins] = s_carry;
        g.ctl->n_entries = s_carry;
    }
}

// The same exclusive prefix over all GPUs' worth of bins at once: 4096 bins per CTA, tiles
// claimed in order by ticket (Control::pad0), the prefix by decoupled look-back (a one-CTA scan
// was 0.75 ms for config 5's 627K bins).
constexpr int kScanBlock = 1024, kScanIPT = 4, kScanTile = kScanBlock * kScanIPT;
__global__ void __launch_bounds__(kScanBlock) tiles_scan_lb_kernel(TileArgs g) {
    __shared__ long long s_warp[kScanBlock / 32 + 1];
    __shared__ long long s_tile, s_prefix;
    const int tid = threadIdx.x;
    if (tid == 0)
        s_tile = (long long)atomicAdd(reinterpret_cast<unsigned long long*>(&g.ctl->pad0), 1ull);
    __syncthreads();
    const long long tile = s_tile, base = tile * kScanTile + (long long)tid * kScanIPT;
    const long long nbins = g.ntiles * kLenClasses;
    long long v[kScanIPT], sum = 0;
#pragma unroll
    for (int q = 0; q < kScanIPT; ++q) {
        v[q] = base + q < nbins ? g.tile_cnt[base + q] : 0;
        sum += v[q];
    }
    long long agg;
    const long long excl = block_excl_scan<kScanBlock>(sum, s_warp, agg);
    if (tid < 32) {
        const long long pre = lookback_warp(g.scan_status, tile, agg, g.ctl);
        if (tid == 0) s_prefix = pre;
    }
    __syncthreads();
    long long run = s_prefix + excl;
#pragma unroll
    for (int q = 0; q < kScanIPT; ++q) {
        if (base + q < nbins) {
            g.tile_off[base + q] = run;
            g.tile_cur[base + q] = (unsigned)run;  // scatter cursor
        }
        run += v[q];
    }
    if (tid == 0 && (tile + 1) * kScanTile >= nbins) {  // the last tile: the total
        g.tile_off[nbins] = s_prefix + agg;
        g.ctl->n_entries = s_prefix + agg;
    }
}

// Pass B: write the pieces into their tiles' bins. tile_cur holds every bin's start on entry (the
// scan wrote it), so the slot is one atomicAdd; the store of a piece is deferred to the next
// piece so the atomic's round trip overlaps the walk instead of stalling it.
// (Deeper software pipelines -- 2 to 4 pieces in flight, their slots held in registers -- were
// measured slower: 93 registers instead of 77 cost more warps than the overlap gained; cfg5
// scatter 19.8 ms at depth 1, 21.3 at 2, 25.3 at 3. Batching 4-16 pieces per thread in shared
// memory and issuing their atomics back to back did not pay either: 19.9 / 20.0 / 21.5 ms.)
__global__ void __launch_bounds__(256, VXG_SCATTER_MINB) tiles_scatter_kernel(TileArgs g);


__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// OR a bit into the tile through a 32-bit shared address.
__device__ __forceinline__ void red_or_shared(uint32_t saddr, uint32_t bit) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(saddr), "r"(bit) : "memory");
}

// ------------------------------------------------------------------------ piece records
// A piece (one segment's samples k in [ka, ka + n) inside one tile, plus E when hasE) is a
// 32-B record -- one 256-bit store in the scatter pass, one 256-bit load in the fill -- written in
// the fill's own terms, so that the fill reads its pieces sequentially and gathers no segment
// record (except E's voxel, once per segment, and S/W in the rare exact redo):
//
//   fixed-point piece (REC_FX segment, n <= 255, ka < 2^24):
//     w0..w2  A0 per axis (x, y, z): a 31-bit value v = rn(2^23 (c_ka - o)) + 2^23 (0.5 + M),
//             i.e. the tile-local voxel coordinate of sample ka in bits 23-30 (0..128) and its
//             23-bit fraction below
//     w3..w5  D per axis: rn(2^30 W) as int32 (|W| <= 1)
//     w6      segment | hasE << 31
//     w7      ka | n << 24
//   exact piece (every other segment -- caller plans, |coordinates| >= 2^24 -- or a long one):
//     w0 segment, w1 ka, w2 (n + hasE) | hasE << 31, w3 = 0x80000000 (no D is that value)
//
// c_ka = fl(S + fl(W ka)) is the exact FP64 sample (include/voxline/parametric.hpp:44-47) and o
// the tile origin; c_ka - o is exact (a multiple of ulp(c_ka) below 2^7).
//
// Exactness of the fixed-point samples. The fill works in 32.32 fixed point: A0 = v 2^9,
// D = rn(2^30 W) 2^2, A_t = A0 + t D for sample k = ka + t. Sample k's voxel is floor(c_k + 0.5)
// (llround: every in-tile sample is > -0.5), and
//   |A_t / 2^32 - (c_k + 0.5 + M - o)| <= 2^-24 + t 2^-31 + 2 e1,
// e1 = max |fl(S + fl(W k)) - (S + W k)| <= (|W k| + |c_k|) 2^-53 < 2^-27 for |S|, |E| < 2^24
// (REC_FX) and in-volume samples. With t < 256 that is below 2^-24 + 2^-23 + 2^-26 < M = 2^-22.
// So whenever the 32-bit fraction of A_t is >= 2M, floor(A_t / 2^32) = floor(c_k + 0.5) - o: the
// high word IS the tile-local voxel coordinate, bit-exactly. A sample whose fraction is below 2M
// on some axis (probability ~3 * 2^-21) makes its lane redo the piece in exact FP64.
constexpr uint32_t kFxNear = 1u << 11;                      // 2M in units of 2^-32, M = 2^-22
constexpr uint32_t kFxBias23 = (1u << 22) + (1u << 1);      // 2^23 (0.5 + M)
constexpr uint32_t kPieceExact = 0x80000000u;               // w3 of an exact-format piece


struct Piece {
    uint32_t w[8];
};
__device__ __forceinline__ void st_piece(uint4* p, const Piece& q) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(q.w[0]),
                 "r"(q.w[1]), "r"(q.w[2]), "r"(q.w[3]), "r"(q.w[4]), "r"(q.w[5]), "r"(q.w[6]),
                 "r"(q.w[7])
                 : "memory");
}
__device__ __forceinline__ Piece ld_piece(const uint4* p) {
    Piece q;
    asm volatile("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(q.w[0]), "=r"(q.w[1]), "=r"(q.w[2]), "=r"(q.w[3]), "=r"(q.w[4]),
                   "=r"(q.w[5]), "=r"(q.w[6]), "=r"(q.w[7])
                 : "l"(p));
    return q;
}

// Build the piece record of (ka, len samples incl. E when hasE) of segment i (scatter pass).
// D[]: rn(2^30 W) per axis (the segment's, computed once); fx: REC_FX and fixed-point enabled.
__device__ __forceinline__ Piece make_piece(const SegRec& r, const uint32_t (&D)[3], bool fx,
                                            long long z_lo, long long i, long long ka,
                                            long long len, bool hasE) {
    const long long n = len - (hasE ? 1 : 0);
    Piece q;
    if (!fx || n > 255 || ka >= (1ll << 24)) {
        q.w[0] = (uint32_t)i;
        q.w[1] = (uint32_t)ka;
        q.w[2] = (uint32_t)len | (hasE ? 0x80000000u : 0u);
        q.w[3] = kPieceExact;
        q.w[4] = q.w[5] = q.w[6] = q.w[7] = 0u;
        return q;
    }
    const double sa[3] = {r.sx, r.sy, r.sz}, wa[3] = {r.wx, r.wy, r.wz};
    const int tsz[3] = {kTX, kTY, kTZ};
    const double t = small_to_double(ka);
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        q.w[ax] = 0u;
        if (n > 0) {  // the tile origin from the anchor sample's voxel (it lies in the tile)
            const long long org = ax == 2 ? z_lo : 0;
            const double c = sample_axis(sa[ax], wa[ax], t);
            const int v = round_pos(c);
            const int o = (int)((v - org) / tsz[ax] * tsz[ax] + org);
            q.w[ax] = rn_low(__dmul_rn(__dsub_rn(c, small_to_double(o)), 0x1p23)) + kFxBias23;
        }
        q.w[3 + ax] = D[ax];
    }
    q.w[6] = (uint32_t)i | (hasE ? 0x80000000u : 0u);
    q.w[7] = (uint32_t)ka | (uint32_t)n << 24;
    return q;
}

// Fixed-point helpers of the fill
__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

// Exact FP64 samples k = k0, k0 + G, ... (steps of them) of segment seg into the tile.
template <int G>
__device__ __forceinline__ void fill_exact(const TileArgs& g, uint32_t sbase, unsigned seg,
                                           long long k0, int steps) {
    const double2* rp = reinterpret_cast<const double2*>(g.rec + seg);
    const double2 ra = __ldg(rp), rb = __ldg(rp + 1), rc = __ldg(rp + 2);
    const double sx = ra.x, sy = ra.y, sz = rb.x, wx = rb.y, wy = rc.x, wz = rc.y;
    double t = __ll2double_rn(k0);
    auto one = [&]() {
        const int32_t x = round_pos(sample_axis(sx, wx, t));
        const int32_t y = round_pos(sample_axis(sy, wy, t));
        const int32_t z = round_pos(sample_axis(sz, wz, t));
        red_or_shared(sbase + 4u * (uint32_t)(z * kSS + y * kRW + (x >> 5)), 1u << (x & 31));
        t = __dadd_rn(t, (double)G);
    };
    for (int st = steps >> 2; st > 0; --st) {
        one();
        one();
        one();
        one();
    }
    for (int st = steps & 3; st > 0; --st) one();
}

// The fixed-point sample loop of a piece's lane (steps samples from A0 + gl D by G D, D = w << 2
// in 32.32): OR each sample's bit into the tile; returns false if some sample lay near a rounding
// boundary (from that sample on, the lane ORed into its spare word instead; the caller redoes the
// lane exactly). Per sample: per axis a 64-bit add as LEA/IADD3 (alu) + IMAD.X (fma-heavy), a
// 3-way min of the fractions and the near test (one predicate carries all samples' tests), the
// shared address (IMADs), a select, the bit, the reduction: ~15.75 issue slots, the alu and
// fma-heavy pipes (a warp instruction every 2 cycles each) about equally loaded.
// Measured alternatives (cfg5 fill, round 2): ptxas fuses a visible 64-bit step into one
// IMAD.WIDE, which holds the fma-heavy pipe 4 cycles -- 72.5 ms against 61.3 (hence the opaque
// zero in the step's high word); FP64 accumulators 2^52 + A stepped by exact integer DADDs on the
// idle FP64 pipe (12.75 slots per sample, the bit pattern's low word is the fraction): 63.7 ms,
// latency-bound on the DADD -> address -> reduction chain; the same with two chains per axis:
// 70.3 ms (register pressure at the 64-register cap).
template <int G>
__device__ __forceinline__ bool fx_loop_int(const TileArgs& g, const Piece& pc, int gl, int steps,
                                            uint32_t sloc, uint32_t spare) {
    constexpr int kSh = 2 + (G >= 32 ? 5 : G >= 16 ? 4 : G >= 8 ? 3 : G >= 4 ? 2 : G >= 2 ? 1 : 0);
    const int32_t wx = (int32_t)pc.w[3], wy = (int32_t)pc.w[4], wz = (int32_t)pc.w[5];
    const unsigned long long ax = ((unsigned long long)pc.w[0] << 9) + (unsigned long long)((long long)gl * wx * 4),
                             ay = ((unsigned long long)pc.w[1] << 9) + (unsigned long long)((long long)gl * wy * 4),
                             az = ((unsigned long long)pc.w[2] << 9) + (unsigned long long)((long long)gl * wz * 4);
    const uint32_t zero = (uint32_t)g.zero;  // 0, opaque to ptxas
    const uint32_t dxl = (uint32_t)wx << kSh, dxh = (uint32_t)(wx >> (32 - kSh)) + zero,
                   dyl = (uint32_t)wy << kSh, dyh = (uint32_t)(wy >> (32 - kSh)) + zero,
                   dzl = (uint32_t)wz << kSh, dzh = (uint32_t)(wz >> (32 - kSh)) + zero;
    uint32_t xl = (uint32_t)ax, yl = (uint32_t)ay, zl = (uint32_t)az;
    uint32_t xh = (uint32_t)(ax >> 32), yh = (uint32_t)(ay >> 32), zh = (uint32_t)(az >> 32);
    bool ok = true;
    auto one_sample = [&]() {
        ok = __vimin3_u32(xl, yl, zl) >= kFxNear && ok;
        uint32_t a = mad_u32(zh, 4u * kSS, sloc) + (yh << 4);
        a += __umulhi(xh, 1u << 27) << 2;
        red_or_shared(ok ? a : spare, 1u << (xh & 31));
        asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(xl), "+r"(xh) : "r"(dxl), "r"(dxh));
        asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(yl), "+r"(yh) : "r"(dyl), "r"(dyh));
        asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(zl), "+r"(zh) : "r"(dzl), "r"(dzh));
    };
    for (int st = steps >> 2; st > 0; --st) {
        one_sample();
        one_sample();
        one_sample();
        one_sample();
    }
    for (int st = steps & 3; st > 0; --st) one_sample();
    return ok;
}

// Set the bits of one piece (G lanes per piece, 32/G pieces per warp step): lane gl takes the
// samples ka + gl, ka + gl + G, ... Every lane runs its own trip count (lanes whose piece is done
// idle until the warp's longest piece is). sbase: the shared byte address of the tile's word 0
// minus 4 * (the tile's global word base); sloc: the shared byte address of word 0; spare: this
// lane's scratch word after the tile.
//
// The fixed-point loop per sample: 3 x (64-bit add), a 3-way min of the fractions with the
// near-boundary test (one predicate carries every sample's test: from the first near sample on,
// the lane ORs into its spare word and redoes the piece exactly afterwards), the shared address
// and the reduction (fx_loop_int / fx_loop_dadd above).
template <int G, bool LATE_E>
__device__ __forceinline__ void fill_piece(const TileArgs& g, uint32_t sbase, uint32_t sloc,
                                           uint32_t spare, const Piece& pc, int gl) {
    if (pc.w[3] == kPieceExact) {  // exact-format piece: gather S and W, FP64 samples
        const unsigned seg = pc.w[0];
        const bool hasE = (pc.w[2] >> 31) != 0;
        const int n = (int)(pc.w[2] & 0x7fffffffu) - (hasE ? 1 : 0);
        const int steps = n > gl ? (n - gl + G - 1) / G : 0;
        if (steps > 0) fill_exact<G>(g, sbase, seg, (long long)pc.w[1] + gl, steps);
        __syncwarp();
        if (hasE && gl == 0) {
            const SegRec* r = g.rec + seg;
            const int32_t ex = __ldg(&r->ex), ey = __ldg(&r->ey), ez = __ldg(&r->ez);
            red_or_shared(sbase + 4u * (uint32_t)(ez * kSS + ey * kRW + (ex >> 5)), 1u << (ex & 31));
        }
        return;
    }
    const unsigned seg = pc.w[6] & 0x7fffffffu;
    const bool hasE = (pc.w[6] >> 31) != 0;
    int32_t ex = 0, ey = 0, ez = 0;
    if (hasE && gl == 0) {  // issued now, used after the samples
        const SegRec* r = g.rec + seg;
        ex = __ldg(&r->ex);
        ey = __ldg(&r->ey);
        ez = __ldg(&r->ez);
    }
    const int n = (int)(pc.w[7] >> 24);
    const int steps = n > gl ? (n - gl + G - 1) / G : 0;
    if (steps > 0) {
        const bool ok = fx_loop_int<G>(g, pc, gl, steps, sloc, spare);
        if (!ok)  // (rare) a sample near a rounding boundary: redo this lane's samples exactly
            fill_exact<G>(g, sbase, seg, (long long)(pc.w[7] & 0xffffffu) + gl, steps);
    }
    // LATE_E: E's address is computed here, not hoisted above the loop by the compiler, so the
    // gather's latency hides behind the samples instead of stalling the warp before them (cfg5,
    // 76 samples per piece: fill 57.30 -> 56.95 ms; with cfg3's ~43-sample pieces the early
    // form is faster: 1.17 against 1.30 ms)
    if (LATE_E) asm volatile("" : "+r"(ex), "+r"(ey), "+r"(ez));
    __syncwarp();
    if (hasE && gl == 0)
        red_or_shared(sbase + 4u * (uint32_t)(ez * kSS + ey * kRW + (ex >> 5)), 1u << (ex & 31));
}

// Pass B: write every piece's record (make_piece) into its tile's bin. tile_cur holds every bin's
// start on entry (the scan wrote it), so the slot is one atomicAdd; the store of a piece is
// deferred to the next piece so the atomic's round trip overlaps the walk instead of stalling it.
// (Deeper software pipelines -- 2 to 4 pieces in flight, their slots held in registers -- were
// measured slower in round 1: cfg5 scatter 19.8 ms at depth 1, 21.3 at 2, 25.3 at 3. Batching
// 4-16 pieces per thread in shared memory and issuing their atomics back to back did not pay
// either: 19.9 / 20.0 / 21.5 ms.)
__global__ void __launch_bounds__(256, VXG_SCATTER_MINB) tiles_scatter_kernel(TileArgs g) {
    const long long tix = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (tix >= g.n) return;
    const long long i = walk_segment(g, tix);
    const SegRec r = load_rec(g.rec + i);
    const bool fx = (r.flags & REC_FX) != 0u && !(g.pf & 8);  // (pf bit 3: tests, A/B)
    uint32_t D[3] = {0u, 0u, 0u};  // rn(2^30 W)
    if (fx) {
        D[0] = rn_low(__dmul_rn(r.wx, 0x1p30));
        D[1] = rn_low(__dmul_rn(r.wy, 0x1p30));
        D[2] = rn_low(__dmul_rn(r.wz, 0x1p30));
    }
    // the pending piece is held as (ka, len | hasE << 31) and built when it is stored
    bool pending = false;
    unsigned pslot = 0, pka = 0, plen = 0;
    auto store = [&]() {
        st_piece(g.pieces + 2 * (size_t)pslot,
                 make_piece(r, D, fx, g.z_lo, i, pka, plen & 0x7fffffffu, (plen >> 31) != 0u));
    };
    walk_pieces(r, rec_steps(g, r, i), g, [&](long long t, long long ka, long long len, bool hasE) {
        // store the previous piece first: its slot arrived while this piece was being walked;
        // the new atomic's result lands directly in pslot and is not read until the next piece
        if (pending) store();
        pslot = atomicAdd(g.tile_cur + bin_of(t, len), 1u);  // 32-bit: one register
        pka = (uint32_t)ka;
        plen = (uint32_t)len | (hasE ? 0x80000000u : 0u);
        pending = true;
    });
    if (pending) store();
}

// Tile claimed by fill ticket r: tiles are handed out in blocks of bx x by x bz tiles (x fastest
// inside a block, blocks x-, then y-, then z-major; partial blocks at the far edges), so the tiles
// in flight at any time are spatially compact and the pieces of one segment in neighbouring tiles
// are filled close together in time (their records' second and later gathers hit L2).
__device__ __forceinline__ long long fill_tile_of(const TileArgs& g, long long r) {
    if (g.bx <= 0) return r;
    const long long ntx = g.ntx, nty = g.nty, ntz = g.ntz;
    const long long per_zl = (long long)g.bz * nty * ntx;
    const long long z0 = r / per_zl * g.bz;
    r %= per_zl;
    const long long dz = min((long long)g.bz, ntz - z0);
    const long long per_yr = (long long)g.by * ntx * dz;
    const long long y0 = r / per_yr * g.by;
    r %= per_yr;
    const long long dy = min((long long)g.by, nty - y0);
    const long long per_b = (long long)g.bx * dy * dz;
    const long long x0 = r / per_b * g.bx;
    r %= per_b;
    const long long dx = min((long long)g.bx, ntx - x0);
    const long long x = x0 + r % dx, y = y0 + (r / dx) % dy, z = z0 + r / (dx * dy);
    return (z * nty + y) * ntx + x;
}

// Persistent CTAs: claim a tile, set its samples' bits in shared memory, OR it into the bitmap.
//
// Shared layout: a row of kTX bits is kRW words; a z-slice of kTY rows is padded by one word so
// a step in z moves to the next bank (without the pad, samples of a segment running along z hit
// the same bank with different words: up to 32-way conflicts on the shared atomics).
// Work split: a warp takes 32/G pieces at a time, G lanes per piece (G from the mean piece
// length); piece entries run two steps ahead, their records are prefetched one step ahead.
// Streamed readback: count a finished tile of z-layer tzi on the device; the tile that completes
// the layer raises the layer's flag in mapped host memory (one plain store per layer, after a
// system fence: the host then copies the layer while the fill goes on).
__device__ __forceinline__ void layer_tile_done(const TileArgs& g, long long tzi) {
    if (atomicAdd(g.layer_cnt + tzi, 1u) + 1u == (unsigned)(g.ntx * g.nty)) {
        __threadfence_system();
        *reinterpret_cast<volatile unsigned*>(g.layer_done + tzi) = 1u;
    }
}

template <int NW, int G, bool STREAM, bool LATE_E>
__global__ void __launch_bounds__(NW * 32) tiles_fill_kernel(TileArgs g) {
    extern __shared__ __align__(16) uint32_t bits[];
    __shared__ long long s_tile[2];
    constexpr int PPW = 32 / G;      // pieces per warp step
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned long long V = (unsigned long long)g.V;
    const int grp = lane / G, gl = lane % G;
    for (int w = tid; w < kTileWords; w += NW * 32) bits[w] = 0u;
    for (int it = 0;; ++it) {
        // (parity-buffered ticket: a fast thread 0 may claim the next tile before a slow thread
        // has read this one's)
        if (tid == 0) s_tile[it & 1] = (long long)atomicAdd(&g.ctl->tile_counter, 1ull);
        __syncthreads();  // (also orders the clearing of the previous tile's bits)
        if (s_tile[it & 1] >= g.ntiles) break;
        const long long tile = fill_tile_of(g, s_tile[it & 1]);
        const long long p0 = __ldg(g.tile_off + tile * kLenClasses),
                        p1 = __ldg(g.tile_off + (tile + 1) * kLenClasses);
        const long long txi = tile % g.ntx, tyi = (tile / g.ntx) % g.nty, tzi = tile / (g.ntx * g.nty);
        const int x0 = (int)(txi * kTX), y0 = (int)(tyi * kTY), z0 = (int)(g.z_lo + tzi * kTZ);
        if (p0 == p1) {  // no samples: the bitmap keeps its words (overwrite: zeros)
            if (g.overwrite) {
                const int xw = (int)min((unsigned long long)kTX, V - x0) / 64;
                for (int r = tid; r < kTY * kTZ * (kRW / 4); r += NW * 32) {
                    const int half = r % (kRW / 4), row = r / (kRW / 4);
                    const long long y = y0 + row % kTY, z = z0 + row / kTY;
                    if (y >= (long long)V || z >= g.z_hi || 2 * half >= xw) continue;
                    *reinterpret_cast<ulonglong2*>(
                        g.words + ((((unsigned long long)(z - g.z_lo) * V + y) * V + x0) >> 6) +
                        2 * half) = make_ulonglong2(0ull, 0ull);
                }
                if (STREAM) {
                    __threadfence();
                    __syncthreads();
                }
            }
            if (STREAM && tid == 0) layer_tile_done(g, tzi);
            continue;
        }
        const int base = z0 * kSS + y0 * kRW + (x0 >> 5);  // (x0 is a multiple of 32)
        const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(bits) - 4u * (uint32_t)base;
        const uint32_t sloc = (uint32_t)__cvta_generic_to_shared(bits);
        const uint32_t spare = (uint32_t)__cvta_generic_to_shared(bits + kTileWords + lane);
        // warp steps of 32/G pieces (G lanes per piece); the next step's records (sequential
        // 32-B reads) load while this step's are filled
        constexpr long long step = (long long)NW * PPW;
        long long pb = p0 + (long long)warp * PPW;
        const uint4* pcs = g.pieces;
        Piece cur{};
        if (pb + grp < p1) cur = ld_piece(pcs + 2 * (pb + grp));
        for (; pb < p1; pb += step) {
            const long long pn = pb + step + grp;
            Piece nxt{};
            if (pn < p1) nxt = ld_piece(pcs + 2 * pn);
            fill_piece<G, LATE_E>(g, sbase, sloc, spare, cur, gl);
            cur = nxt;
        }
        __syncthreads();
        // OR the tile into the bitmap: a row of kTX bits is 4 words = 2 x 16 B; each thread
        // handles rows r = tid, tid + NW*32, ... with all loads issued before the stores.
        const int xw = (int)min((unsigned long long)kTX, V - x0) / 64;  // words inside the volume
        constexpr int kRows = kTY * kTZ;
        constexpr int kBatch = 4;  // rows per thread in flight
        for (int half = 0; half < kRW / 4; ++half) {  // the row's 16-B chunks
            for (int r0 = tid; r0 < kRows; r0 += kBatch * NW * 32) {
                ulonglong2 cur[kBatch];
                unsigned long long wa[kBatch], wb[kBatch];
                ulonglong2* dst[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    const int row = r0 + u * NW * 32;
                    wa[u] = wb[u] = 0;
                    dst[u] = nullptr;
                    if (row >= kRows) continue;
                    const int ly = row % kTY, lz = row / kTY;
                    uint32_t* sw = bits + lz * kSS + ly * kRW + 4 * half;
                    wa[u] = (unsigned long long)sw[0] | ((unsigned long long)sw[1] << 32);
                    wb[u] = (unsigned long long)sw[2] | ((unsigned long long)sw[3] << 32);
                    sw[0] = sw[1] = sw[2] = sw[3] = 0u;
                    const long long y = y0 + ly, z = z0 + lz;
                    if (y >= (long long)V || z >= g.z_hi || 2 * half >= xw ||
                        ((wa[u] | wb[u]) == 0 && !g.overwrite))
                        continue;
                    // (rows are 16-B aligned: V and x0 are multiples of 128)
                    dst[u] = reinterpret_cast<ulonglong2*>(
                        g.words + ((((unsigned long long)(z - g.z_lo) * V + y) * V + x0) >> 6) +
                        2 * half);
                    cur[u] = g.overwrite ? make_ulonglong2(0ull, 0ull) : *dst[u];
                }
#pragma unroll
                for (int u = 0; u < kBatch; ++u)
                    if (dst[u]) *dst[u] = make_ulonglong2(cur[u].x | wa[u], cur[u].y | wb[u]);
            }
        }
        // (the next iteration's __syncthreads orders these clears before new atomics)
        if (STREAM) {  // streamed readback: this tile's words are final
            __threadfence();
            __syncthreads();
            if (tid == 0) layer_tile_done(g, tzi);
        }
    }
}

// =============================================================================== launchers
int tile_len_classes() { return kLenClasses; }

int tile_perm_keys() { return kPermKeys; }

int tile_dims(long long V, long long depth, int& tx, int& ty, int& tz) {
    tx = kTX;
    ty = kTY;
    tz = kTZ;
    (void)V;
    (void)depth;
    return kTileWords * 4;  // shared-memory bytes of the tile (padded z-slices)
}

void launch_tiles_perm(const TileArgs& g, cudaStream_t s) {
    const unsigned grid = (unsigned)((g.n + 255) / 256);
    perm_hist_kernel<<<grid, 256, 0, s>>>(g);
    perm_scan_kernel<<<1, 1024, 0, s>>>(g);
    perm_scatter_kernel<<<grid, 256, 0, s>>>(g);
}

void launch_slab_select(const TileArgs& g, int* sel, unsigned long long* nsel, cudaStream_t s) {
    slab_select_kernel<<<(unsigned)((g.n + 255) / 256), 256, 0, s>>>(g, sel, nsel);
}

void launch_tiles_count(const TileArgs& g, cudaStream_t s) {
    if (g.n <= 0) return;  // (a slab no segment reaches)
    tiles_count_kernel<<<(unsigned)((g.n + 255) / 256), 256, 0, s>>>(g);
}
int tile_scan_tiles(long long nbins) { return (int)((nbins + kScanTile - 1) / kScanTile); }
void launch_tiles_scan(const TileArgs& g, cudaStream_t s) {
    if (g.scan_status)
        tiles_scan_lb_kernel<<<(unsigned)tile_scan_tiles(g.ntiles * kLenClasses), kScanBlock, 0, s>>>(g);
    else
        tiles_scan_kernel<<<1, 1024, 0, s>>>(g);
}
void launch_tiles_scatter(const TileArgs& g, cudaStream_t s) {
    if (g.n <= 0) return;
    TileArgs gg = g;
    if (const char* e = getenv("VXG_FILL_PF")) gg.pf = atoi(e);  // bit 3: exact pieces only
    tiles_scatter_kernel<<<(unsigned)((gg.n + 255) / 256), 256, 0, s>>>(gg);
}
template <int NW, int G, bool STREAM, bool LATE_E>
static cudaError_t launch_fill_nw(const TileArgs& g, int num_sms, cudaStream_t s) {
    const size_t smem = (size_t)(kTileWords + 32) * 4;  // the tile + 32 per-lane spare words
    cudaFuncSetAttribute(tiles_fill_kernel<NW, G, STREAM, LATE_E>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tiles_fill_kernel<NW, G, STREAM, LATE_E>,
                                                  NW * 32, smem);
    if (per_sm < 1) per_sm = 1;
    long long grid = (long long)per_sm * num_sms;
    if (grid > g.ntiles) grid = g.ntiles;
    tiles_fill_kernel<NW, G, STREAM, LATE_E><<<(unsigned)grid, NW * 32, smem, s>>>(g);
    return cudaGetLastError();
}

template <int G, bool STREAM>
static cudaError_t launch_fill_gs(const TileArgs& g, int num_sms, cudaStream_t s) {
    // 32 warps per CTA at 64 registers (one CTA per SM: the tile takes the shared memory);
    // round 2, cfg5 fill: 61.35 ms at 32 warps, 61.45 at 24 (85 registers), 64.1 at 16.
    // Pieces of one lane (G = 1) averaging >= 60 samples: E's address after the samples.
    if constexpr (G == 1) {
        if (g.late_e) return launch_fill_nw<32, G, STREAM, true>(g, num_sms, s);
    }
    return launch_fill_nw<32, G, STREAM, false>(g, num_sms, s);
}

// (the streamed-readback signalling is a separate instantiation: the plain kernel stays as lean)
template <int G>
static cudaError_t launch_fill_g(const TileArgs& g, int num_sms, cudaStream_t s) {
    return g.layer_done ? launch_fill_gs<G, true>(g, num_sms, s) : launch_fill_gs<G, false>(g, num_sms, s);
}

static cudaError_t launch_tiles_fill_g(const TileArgs& g, int num_sms, int G, cudaStream_t s);

// mean_len: mean samples per piece -> lanes per piece (VXG_FILL_G overrides: 4, 8, 16 or 32)
cudaError_t launch_tiles_fill(const TileArgs& g, int num_sms, double mean_len, cudaStream_t s) {
    // (round 2, fixed-point fill: G = 1 is best for the config-3 and config-5 piece lengths --
    // cfg5 fill 58.3 ms against 61.3 (G = 2) and 67.1 (G = 4); cfg3 1.18 / 1.29 / 1.67 ms. The
    // exact FP64 fill of round 1 preferred G = 2: profiles/r1_fill_G)
    int G = mean_len < 160.0 ? 1 : (mean_len < 320.0 ? 16 : 32);
    if (const char* e = getenv("VXG_FILL_G")) G = atoi(e);
    TileArgs gg = g;
    gg.late_e = mean_len >= 60.0 ? 1 : 0;
    if (const char* e = getenv("VXG_FILL_LATE_E")) gg.late_e = atoi(e);
    gg.pf = 1;
    if (const char* e = getenv("VXG_FILL_PF")) gg.pf = atoi(e);
    if (const char* e = getenv("VXG_FILL_ORDER")) {  // "bx,by,bz" (experiments)
        gg.bx = gg.by = gg.bz = 0;
        sscanf(e, "%d,%d,%d", &gg.bx, &gg.by, &gg.bz);
        if (gg.bx <= 0 || gg.by <= 0 || gg.bz <= 0) gg.bx = gg.by = gg.bz = 0;
    }
    return launch_tiles_fill_g(gg, num_sms, G, s);
}

static cudaError_t launch_tiles_fill_g(const TileArgs& g, int num_sms, int G, cudaStream_t s) {
    if (G == 1) return launch_fill_g<1>(g, num_sms, s);
    if (G == 2) return launch_fill_g<2>(g, num_sms, s);
    if (G == 4) return launch_fill_g<4>(g, num_sms, s);
    if (G == 8) return launch_fill_g<8>(g, num_sms, s);
    if (G == 16) return launch_fill_g<16>(g, num_sms, s);
    return launch_fill_g<32>(g, num_sms, s);
}

}  // namespace vxg
