// vxg_device.cuh -- device arithmetic shared by every kernel.
//
// Bit-exact parity with the reference CPU path hinges on evaluating exactly the reference's
// IEEE-754 operation sequence with round-to-nearest and NO fused multiply-add (nvcc contracts
// `s + w*t` to DFMA by default). Every FP64 operation below is therefore an
// explicit _rn intrinsic (DMUL / DADD / DSQRT / DDIV), and the library is also built with
// --fmad=false as a second line of defence.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace vxg {

// Packed per-segment record consumed by the emit kernels (64 B: one half cache line).
struct alignas(16) SegRec {
    double sx, sy, sz;   // S
    double wx, wy, wz;   // W = (E - S) / N
    int32_t ex, ey, ez;  // round_point(E): the k == N sample (include/voxline/parametric.hpp:43)
    uint32_t flags;      // REC_* below
};
static_assert(sizeof(SegRec) == 64, "SegRec must be 64 B");

enum : uint32_t {
    REC_CHECK = 1u,  // samples can approach the int32 edge -> checked rounding, generic path
    REC_WIDE = 2u,   // some |W| > 1 (only from caller-supplied plans) -> exact dedup, generic path
    REC_POS = 4u,    // every coordinate of S and E >= 1: samples are positive, round = trunc(x+.5)
    REC_FX = 8u,     // plan-kernel W and every |coordinate| of S and E < 2^24: the bitmap fill may
                     // step samples in 32.32 fixed point (vxg_bitmap.cu, fill_piece)
};
// The bitmap passes' walk-order copy of the records keeps N in the flag word's upper bits.
constexpr int kRecNShift = 4;

// Voxel key for consecutive-duplicate tests: x + 8y + 64z (mod 2^32). Consecutive samples of one
// segment differ by |W| <= 1 per axis plus a few ulp, so their voxels differ by at most 2 per
// axis, and dx + 8dy + 64dz with |d| <= 3 vanishes only for d == 0: within a segment the key
// equality is exactly voxel equality. (Records with |W| > 1 carry REC_WIDE and compare exactly.)
__device__ __forceinline__ int32_t voxel_key(int32_t x, int32_t y, int32_t z) {
    return x + 8 * y + 64 * z;
}

// llround for samples known to lie in (-0.5, 2^31): one DADD in round-toward-minus-infinity
// against K = 2^51 + 0.5. The sum lies in [2^51, 2^52), whose ulp is 0.5, so
// RM(c + K) = 2^51 + floor(2c + 1) / 2 exactly and the 52-bit mantissa field is F = floor(2c + 1);
// llround(c) = floor(c + 0.5) = F >> 1 (one funnel shift on the ALU pipe). One FP64 op instead of
// the two of an RZ add + magic-number extraction, and no F2I (quarter-rate conversion pipe).
// (K lives in the constant bank: DADD takes it as a c[][] operand, so hot loops neither hold it
// in two registers nor rematerialise it with two moves per iteration)
static __constant__ double kRoundPosK = 0x1.0000000000001p51;

__device__ __forceinline__ int32_t round_pos(double c) {
    const double d = __dadd_rd(c, kRoundPosK);
    return (int32_t)__funnelshift_r((unsigned)__double2loint(d), (unsigned)__double2hiint(d), 1);
}

// Endpoints whose magnitude exceeds this get per-sample range checks in the emit kernels;
// below it every sample S + W*k (k < N) provably rounds inside the int32 lattice because it lies
// between S and E up to a relative error of a few ulp.
constexpr double kCheckThreshold = 2147483000.0;

// Run-control block shared by the kernels of one batch (one cudaMemsetAsync resets it).
struct Control {
    unsigned long long max_steps;   // N_max (atomicMax)
    long long err_seg;              // error key (see record_error), 0 = none
    long long pad0;
    long long total;                // emit: total voxels (or capacity for the plan)
    unsigned long long tile_counter;// dynamic tile ids (look-back forward progress)
    unsigned long long outside;     // bitmap: samples outside the volume
    long long n_entries;            // clip: non-empty entries
    int abort;                      // look-back watchdog fired (see lookback_resolve)
    int pad1[3];
};

// ----------------------------------------------------------------------------- rounding
// llround (src/geometry.cpp:21): half away from zero == trunc(RZ(c + copysign(0.5, c))).
// Proof sketch: for c >= 0, floor(RZ(c + 0.5)) == floor(c + 0.5) because the integer
// floor(c + 0.5) is representable and <= c + 0.5, so RZ cannot round below it; c < 0 mirrors.
__device__ __forceinline__ double round_bias(double c) {
    return __dadd_rz(c, copysign(0.5, c));
}

__device__ __forceinline__ int32_t round_fast(double c) {
    return __double2int_rz(round_bias(c));
}

// Checked variant: false if c is non-finite or llround(c) falls outside int32
// (src/geometry.cpp:16-26). NaN fails both comparisons.
__device__ __forceinline__ bool round_checked(double c, int32_t& out) {
    const double h = round_bias(c);
    if (!(h > -2147483649.0 && h < 2147483648.0)) {
        out = 0;
        return false;
    }
    out = __double2int_rz(h);
    return true;
}

// L1 prefetch (no register); callers keep p in bounds.
__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// cnt += (a != b) as one compare + one predicated add (the compiler's select-and-add form is
// three instructions; this sits in the count loops' per-sample body)
__device__ __forceinline__ void count_ne(int& cnt, int32_t a, int32_t b) {
    asm("{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %1, %2;\n\t@p add.s32 %0, %0, 1;\n\t}"
        : "+r"(cnt)
        : "r"(a), "r"(b));
}

// S + W*t with separate multiply and add (include/voxline/parametric.hpp:44-47).
__device__ __forceinline__ double sample_axis(double s, double w, double t) {
    return __dadd_rn(s, __dmul_rn(w, t));
}

// ----------------------------------------------------------------------------- magic numbers
// Integer <-> double conversions on the FP64 pipe (one DADD each) instead of the slow conversion
// pipe (I2F / F2I): x + 1.5 2^52 rounds x to an integer (round to nearest) for |x| < 2^51, and the
// low 52 bits of its bit pattern hold 2^51 + rn(x).
constexpr double kMagic52 = 0x1.8p52;
__device__ __forceinline__ double small_to_double(long long v) {  // exact for |v| < 2^51
    return __dadd_rn(__longlong_as_double(0x4338000000000000ll + v), -kMagic52);
}
__device__ __forceinline__ uint32_t rn_low(double x) {  // rn(x) mod 2^32, |x| < 2^51
    return (uint32_t)__double2loint(__dadd_rn(x, kMagic52));
}
__device__ __forceinline__ long long rn_i64(double x) {  // rn(x), |x| < 2^50
    const long long b = __double_as_longlong(__dadd_rn(x, kMagic52));
    return (b & 0xfffffffffffffll) - (1ll << 51);
}

// ----------------------------------------------------------------------------- fixed point
// 32.32 fixed-point stepping of a segment's samples (the bitmap fill and the list fast runs).
// Sample k is c_k = fl(S + fl(W k)) per axis (include/voxline/parametric.hpp:44-47); its voxel
// is llround(c_k) = floor(c_k + 0.5) for c_k > -0.5. A lane starts from an exact FP64 sample c_t0:
//   A_0 = round(c_t0) 2^32 + rn(2^32 (c_t0 - round(c_t0))) + (0.5 + M) 2^32,  D = rn(2^32 W),
// (c_t0 - round(c_t0) is exact by Sterbenz for c_t0 >= 0.5) and steps A_j = A_0 + j m D for a
// step of m samples. Then
//   |A_j / 2^32 - (c_k + 0.5 + M)| <= 2^-33 + j m 2^-33 + 2 e1,
// e1 = max |fl(S + fl(W k)) - (S + W k)| <= (|W k| + |c_k|) 2^-53 < 2^-26 for coordinates below
// 2^24 (REC_FX). For j m <= 1023 that is below 2^-23 + 2^-25 < M = 2^-22, so whenever the 32-bit
// fraction of A_j is >= 2M, its high word is llround(c_k) exactly. A sample whose fraction is
// below 2M on some axis (probability ~3 * 2^-21) is evaluated in FP64 instead.
constexpr uint32_t kFxNear22 = 1u << 11;                  // 2M in units of 2^-32, M = 2^-22
constexpr long long kFxBias22 = (1ll << 31) + (1ll << 10);  // (0.5 + M) 2^32

__device__ __forceinline__ void fx_start(double s, double w, double t, uint32_t& lo, uint32_t& hi) {
    const double c = sample_axis(s, w, t);
    const int32_t o = round_pos(c);
    const long long A = ((long long)o << 32) +
                        rn_i64(__dmul_rn(__dsub_rn(c, small_to_double(o)), 0x1p32)) + kFxBias22;
    lo = (uint32_t)A;
    hi = (uint32_t)((unsigned long long)A >> 32);
}
// m D = m rn(2^32 w) as (lo, hi), m a power of two
__device__ __forceinline__ void fx_delta(double w, int shift, uint32_t& lo, uint32_t& hi) {
    const long long d = rn_i64(__dmul_rn(w, 0x1p32)) << shift;
    lo = (uint32_t)d;
    hi = (uint32_t)((unsigned long long)d >> 32);
}
// (lo, hi) += (dlo, dhi): LEA/IADD3 (alu) + IMAD.X (fma) -- a 64-bit add that ptxas cannot fuse
// into one IMAD.WIDE (which holds the fma-heavy pipe 4 cycles)
__device__ __forceinline__ void fx_add(uint32_t& lo, uint32_t& hi, uint32_t dlo, uint32_t dhi) {
    asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(lo), "+r"(hi) : "r"(dlo), "r"(dhi));
}

// ----------------------------------------------------------------------------- plan
// make_plan (src/parametric.cpp:8-26). Returns false on a range error of either endpoint.
struct Plan {
    long long n;
    double wx, wy, wz;
    int32_t ex, ey, ez;
};

__device__ __forceinline__ bool make_plan(double sx, double sy, double sz, double ex, double ey,
                                          double ez, Plan& p) {
    int32_t vsx, vsy, vsz;
    bool ok = round_checked(sx, vsx) & round_checked(sy, vsy) & round_checked(sz, vsz);
    ok &= round_checked(ex, p.ex) & round_checked(ey, p.ey) & round_checked(ez, p.ez);
    if (!ok) {
        p.n = 0;
        p.wx = p.wy = p.wz = 0.0;
        return false;
    }
    if (vsx == p.ex && vsy == p.ey && vsz == p.ez) {
        p.n = 0;
        p.wx = p.wy = p.wz = 0.0;
        return true;
    }
    const double dx = __dsub_rn(ex, sx), dy = __dsub_rn(ey, sy), dz = __dsub_rn(ez, sz);
    // sqrt((dx*dx + dy*dy) + dz*dz), left to right (src/geometry.cpp:10)
    const double len =
        __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    long long n = static_cast<long long>(floor(len));
    const double ext = fmax(fabs(dx), fmax(fabs(dy), fabs(dz)));
    const long long ce = static_cast<long long>(ceil(ext));
    n = n > ce ? n : ce;
    n = n > 1 ? n : 1;
    const double nd = __ll2double_rn(n);
    p.n = n;
    p.wx = __ddiv_rn(dx, nd);
    p.wy = __ddiv_rn(dy, nd);
    p.wz = __ddiv_rn(dz, nd);
    return true;
}

__device__ __forceinline__ uint32_t rec_flags(double sx, double sy, double sz, double ex,
                                              double ey, double ez) {
    const double m = fmax(fmax(fmax(fabs(sx), fabs(sy)), fmax(fabs(sz), fabs(ex))),
                          fmax(fabs(ey), fabs(ez)));
    const double lo = fmin(fmin(fmin(sx, sy), fmin(sz, ex)), fmin(ey, ez));
    // samples lie between S and E up to a few ulp: all >= 1 - tiny > -0.5 when lo >= 1
    return (m > kCheckThreshold ? REC_CHECK : 0u) | (lo >= 1.0 ? REC_POS : 0u) |
           (m < 0x1p24 ? REC_FX : 0u);
}

// ----------------------------------------------------------------------------- SplitMix64
// include/voxline/bench.hpp:20-37
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
__host__ __device__ __forceinline__ uint64_t splitmix_draw(uint64_t seed, uint64_t j) {
    return mix64(seed + (j + 1) * kGamma);
}

struct SplitMix {
    uint64_t state;
    __device__ __forceinline__ uint64_t next() {
        state += kGamma;
        return mix64(state);
    }
    __device__ __forceinline__ double uniform01() {
        return __dmul_rn(__ull2double_rn(next() >> 11), 0x1.0p-53);
    }
    __device__ __forceinline__ double uniform(double lo, double hi) {
        return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), uniform01()));
    }
};

// ----------------------------------------------------------------------------- memory order
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// ----------------------------------------------------------------------------- look-back
// Decoupled look-back (single-pass prefix scan): tile t publishes its aggregate (flag A) as soon
// as it is known, then accumulates predecessors' values until it meets an inclusive prefix
// (flag P), and publishes its own inclusive prefix. Values are 62-bit and packed with the flag
// into one 64-bit word, so a relaxed single-copy-atomic access carries both.
constexpr unsigned long long kFlagA = 1ull << 62;
constexpr unsigned long long kFlagP = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

// Publish a tile's aggregate (tile 0 publishes its inclusive prefix directly). One lane.
__device__ __forceinline__ void lookback_publish(unsigned long long* status, long long tile,
                                                 long long aggregate) {
    st_relaxed_u64(&status[tile], (tile == 0 ? kFlagP : kFlagA) | (unsigned long long)aggregate);
}

// Resolve a tile whose aggregate was already published: accumulate predecessors back to the
// nearest inclusive prefix, publish this tile's inclusive prefix, return the exclusive one.
// Called by all 32 lanes of one warp. Each round examines a window of 32*LB predecessors (lane i
// holds tiles end-1-LB*i-q, q < LB), so a prefix that lies a few hundred tiles back -- the
// number of tiles in flight -- is reached in one or two L2 round trips.
// Watchdog: a spin that outlives kSpinLimit polls (~seconds) raises Control::abort, which makes
// every other spinning warp give up too; the kernel then terminates with a logic error instead
// of hanging the GPU.
constexpr unsigned kSpinLimit = 1u << 22;
constexpr int kLookbackItems = 4;

__device__ __forceinline__ long long lookback_resolve(unsigned long long* status, long long tile,
                                                      long long aggregate, Control* ctl) {
    constexpr int LB = kLookbackItems;
    const int lane = threadIdx.x & 31;
    if (tile == 0) return 0;
    long long excl = 0;
    long long end = tile;  // window: tiles [end - 32*LB, end)
    while (true) {
        unsigned long long s[LB];
#pragma unroll
        for (int q = 0; q < LB; ++q) {
            const long long j = end - 1 - (long long)(LB * lane + q);
            s[q] = j >= 0 ? ld_relaxed_u64(&status[j]) : kFlagP;  // virtual P before tile 0
        }
        unsigned spins = 0;
        int qp;          // this lane's first item with an inclusive prefix (LB if none)
        unsigned pmask;  // lanes holding one
        while (true) {
            qp = LB;
#pragma unroll
            for (int q = LB - 1; q >= 0; --q)
                if ((s[q] >> 62) == 2) qp = q;
            pmask = __ballot_sync(0xffffffffu, qp < LB);
            const int plane = pmask ? __ffs(pmask) - 1 : 32;
            // items that matter: everything nearer than the nearest prefix, and that prefix
            const int lim = lane < plane ? LB : (lane == plane ? qp + 1 : 0);
            bool missing = false;
#pragma unroll
            for (int q = 0; q < LB; ++q) missing |= q < lim && (s[q] >> 62) == 0;
            if (!__any_sync(0xffffffffu, missing)) {
                long long v = 0;
#pragma unroll
                for (int q = 0; q < LB; ++q)
                    if (q < lim) v += (long long)(s[q] & kValMask);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                excl += v;
                break;
            }
            // back off: a spinning warp must not steal issue slots from the warps whose
            // aggregates it is waiting for
            __nanosleep(spins < 64 ? 20u : 200u);
#pragma unroll
            for (int q = 0; q < LB; ++q) {
                if (q < lim && (s[q] >> 62) == 0) {
                    const long long j = end - 1 - (long long)(LB * lane + q);
                    s[q] = ld_relaxed_u64(&status[j]);
                }
            }
            if ((++spins & 63u) == 0) {  // (spins is warp-uniform)
                if (spins >= (kSpinLimit >> 4) && lane == 0) atomicExch(&ctl->abort, 1);
                const int ab = *reinterpret_cast<volatile int*>(&ctl->abort);
                if (__any_sync(0xffffffffu, ab != 0)) {  // give up: the call fails (logic error)
                    pmask = 1u;
                    break;
                }
            }
        }
        if (pmask) break;
        end -= 32 * LB;
    }
    if (lane == 0) st_relaxed_u64(&status[tile], kFlagP | (unsigned long long)(excl + aggregate));
    return excl;
}

// ----------------------------------------------------------------------------- errors / samples
// Error key ((2^59 - 1 - seg) << 3) | kind: atomicMax keeps the lowest failing segment, so the
// reported segment matches the reference's serial preprocess loop (src/batch.cpp:61-66).
__device__ __forceinline__ void record_error(Control* ctl, long long seg, int kind) {
    const long long key = ((((1ll << 59) - 1) - seg) << 3) | (long long)kind;
    atomicMax(&ctl->err_seg, key);
}

// Voxel of sample k of a segment (include/voxline/parametric.hpp:41-48 + src/geometry.cpp:32).
__device__ __forceinline__ void eval_sample(const SegRec& r, long long k, long long N, int32_t& x,
                                            int32_t& y, int32_t& z, bool& bad) {
    if (k >= N) {  // the final sample is E itself
        x = r.ex;
        y = r.ey;
        z = r.ez;
        return;
    }
    const double t = __ll2double_rn(k);
    const double gx = sample_axis(r.sx, r.wx, t);
    const double gy = sample_axis(r.sy, r.wy, t);
    const double gz = sample_axis(r.sz, r.wz, t);
    if (r.flags & REC_CHECK) {
        bool ok = round_checked(gx, x);
        ok &= round_checked(gy, y);
        ok &= round_checked(gz, z);
        bad |= !ok;
    } else {
        x = round_fast(gx);
        y = round_fast(gy);
        z = round_fast(gz);
    }
}

__device__ __forceinline__ SegRec load_rec(const SegRec* p) {
    const uint4* q = reinterpret_cast<const uint4*>(p);
    SegRec r;
    uint4* d = reinterpret_cast<uint4*>(&r);
    d[0] = __ldg(q + 0);
    d[1] = __ldg(q + 1);
    d[2] = __ldg(q + 2);
    d[3] = __ldg(q + 3);
    return r;
}

// ----------------------------------------------------------------------------- block scan
// Exclusive scan of one long long per thread over the block; returns the thread's exclusive
// prefix and (in every thread, after the call) the block total via `total`.
template <int BLOCK>
__device__ __forceinline__ long long block_excl_scan(long long v, long long* s_warp,
                                                     long long& total) {
    constexpr int NW = BLOCK / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        long long x = lane < NW ? s_warp[lane] : 0;
        long long xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += t;
        }
        if (lane < NW) s_warp[lane] = xi - x;
        if (lane == 31) s_warp[NW] = xi;
    }
    __syncthreads();
    total = s_warp[NW];
    return s_warp[warp] + incl - v;
}

// Publish + resolve in one go (called by all 32 lanes of one warp).
__device__ __forceinline__ long long lookback_warp(unsigned long long* status, long long tile,
                                                   long long aggregate, Control* ctl) {
    if ((threadIdx.x & 31) == 0) lookback_publish(status, tile, aggregate);
    return lookback_resolve(status, tile, aggregate, ctl);
}

}  // namespace vxg
