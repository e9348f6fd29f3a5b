/*
 * round_pos_check.c -- host check of the one-DADD rounding identity the GPU hot loops use
 * (paper_2009_09500_b200/csrc/vxg_device.cuh round_pos) against llround, the reference's
 * rounding (src/geometry.cpp:21, ties away from zero).
 *
 * TEST INFRASTRUCTURE (built into oracle/_build/liboracle.so, called by tests/ only).
 *
 * The identity: for c in (-0.5, 2^31), RM(c + (2^51 + 0.5)) lies in [2^51, 2^52) where the ulp is
 * 0.5, so its 52-bit mantissa field F equals floor(2c + 1) and llround(c) = floor(c + 0.5) =
 * F >> 1. The GPU computes RM(...) with __dadd_rd and takes bits 1..32 of the double with one
 * funnel shift; this file performs the same IEEE-754 addition in round-toward-minus-infinity on
 * the host (fesetround(FE_DOWNWARD); built with -frounding-math so nothing is folded at compile
 * time) and extracts the same bits.
 */
#include <fenv.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

static int32_t round_pos_emul(double c) {
    volatile double k = 0x1.0000000000001p51; /* 2^51 + 0.5 */
    volatile double cc = c;
    /* (current rounding mode: downward; the volatile store keeps the addition before the
     * caller restores the mode -- GCC may otherwise move FP arithmetic across fesetround) */
    volatile double d = cc + k;
    const double dv = d;
    uint64_t bits;
    memcpy(&bits, &dv, sizeof bits);
    return (int32_t)(uint32_t)(bits >> 1); /* __funnelshift_r(lo, hi, 1) */
}

static uint64_t sm_next(uint64_t* s) {
    uint64_t z = (*s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* Checks: every tie k + 0.5 for k < ties and both its neighbouring doubles; `rnd` random values
 * uniform in [0, 2^31 - 1) and as many near-ties (k + 0.5 +- up to 8 ulp, k random < 2^31 - 1);
 * a fixed list of small values in (-0.5, 1] and near 2^31. Returns the number of mismatches; *checked gets
 * the number of values tested and *first_bad the first mismatching value (if any). */
int64_t vo_check_round_pos(int64_t ties, int64_t rnd, uint64_t seed, int mode, int64_t* checked,
                           double* first_bad) {
    /* mode 1: the addition in round-to-nearest instead (a deliberately wrong variant: the
     * check must catch it) */
    const int rm = mode == 1 ? FE_TONEAREST : FE_DOWNWARD;
    const int old = fegetround();
    fesetround(FE_DOWNWARD);
    int64_t bad = 0, n = 0;
    double fb = 0.0;
#define CHECK(v)                                              \
    do {                                                      \
        const double c_ = (v);                                \
        fesetround(rm);                                       \
        const int32_t got_ = round_pos_emul(c_);              \
        fesetround(FE_TONEAREST);                             \
        const long long want_ = llround(c_);                  \
        ++n;                                                  \
        if (got_ != want_) {                                  \
            if (!bad) fb = c_;                                \
            ++bad;                                            \
        }                                                     \
    } while (0)
    for (int64_t k = 0; k < ties; ++k) {
        const double t = (double)k + 0.5;
        CHECK(t);
        CHECK(nextafter(t, 0.0));
        CHECK(nextafter(t, INFINITY));
    }
    uint64_t s = seed;
    const double top = 2147483647.0 - 1.0;
    for (int64_t i = 0; i < rnd; ++i) {
        const double u = (double)(sm_next(&s) >> 11) * 0x1.0p-53;
        CHECK(u * top);
        const double t = floor(u * top) + 0.5;
        const int j = (int)(sm_next(&s) % 17) - 8;
        double v = t;
        for (int q = 0; q < (j < 0 ? -j : j); ++q) v = nextafter(v, j < 0 ? 0.0 : INFINITY);
        CHECK(v);
    }
    static const double small[] = {-0.49999999999999994, -0.25, -1e-300, -0.0, 0.0, 1e-300,
                                   0.25, 0.49999999999999994, 0.5, 0.5000000000000001,
                                   0.9999999999999999, 1.0, 1.4999999999999998, 1.5,
                                   2147483646.4999998, 2147483646.5, 2147483645.5};
    for (size_t i = 0; i < sizeof small / sizeof small[0]; ++i) CHECK(small[i]);
#undef CHECK
    fesetround(old);
    if (checked) *checked = n;
    if (first_bad) *first_bad = fb;
    return bad;
}
