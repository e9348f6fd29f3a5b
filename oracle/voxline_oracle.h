/*
 * voxline_oracle.h -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity checker for the B200 path. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. The product library
 * (libvoxgpu.so) never links or calls it.
 *
 * Parity pinning: the restatement is checked against (1) the reference's own golden
 * vectors / known-answer tests (tests/golden/*.json, produced by tests/golden/make_golden.py)
 * and (2) the reference implementation itself, compiled unmodified from /root/reference into
 * oracle/_ref/libref_voxline.so by oracle/Makefile (see oracle/ref_wrapper.cpp).
 *
 * Build flags matter: the reference's canonical build is CMake Release without -march, which
 * emits separate mulsd/addsd (no FMA).  This file is compiled with -ffp-contract=off.
 *
 * Error codes follow the reference's exception classes (include/voxgpu.h mirrors them):
 *   0 ok, 1 std::invalid_argument, 2 std::range_error, 3 std::out_of_range, 4 std::logic_error.
 */
#ifndef VOXLINE_ORACLE_H
#define VOXLINE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { VO_OK = 0, VO_INVALID_ARGUMENT = 1, VO_RANGE_ERROR = 2, VO_OUT_OF_RANGE = 3, VO_LOGIC_ERROR = 4 };

/* SplitMix64 (include/voxline/bench.hpp:20-37). */
uint64_t vo_splitmix_next(uint64_t* state);
double vo_uniform01(uint64_t* state);
double vo_uniform(uint64_t* state, double lo, double hi);

/* geometry (src/geometry.cpp:8-34). Segment = 6 doubles {sx,sy,sz,ex,ey,ez}. */
double vo_segment_length(const double seg[6]);
int vo_round_point(const double p[3], int32_t out[3]);

/* parametric (src/parametric.cpp:8-26, include/voxline/parametric.hpp:41-48). */
int vo_make_plan(const double seg[6], int64_t* n, double w[3]);
void vo_sample(const double seg[6], int64_t n, const double w[3], int64_t k, double out[3]);
int vo_voxelize_parametric(const double seg[6], int32_t* out, int64_t cap, int64_t* count);
int vo_chain_length_bounds(const double seg[6], int64_t* lo, int64_t* hi);

/* batch (src/batch.cpp:57-73, 75-90, 92-152, 164-170). */
int vo_batch_preprocess(const double* segs, int64_t n, int64_t* steps, double* w3,
                        int64_t* offsets, int64_t* max_steps, int64_t* capacity);
int vo_kernel_work_item(const double* segs, int64_t n, const int64_t* steps, const double* w3,
                        int64_t max_steps, int64_t i, int64_t k, int32_t out[3], int* live);
/* Flat batch result: chain i is out[chain_off[i] .. chain_off[i+1]) (voxels of 3 int32).
 * out may be NULL to only count. nthreads<=0 -> all cores. */
int vo_run_batch(const double* segs, int64_t n, int32_t* out, int64_t out_cap,
                 int64_t* chain_off, int64_t* total, int nthreads);
/* Per-segment chain lengths only (no voxel output). */
int vo_chain_lengths(const double* segs, int64_t n, int64_t* lengths, int nthreads);

/* Occupancy bitmap of every sample voxel (no reference counterpart; the set of rounded
 * samples == the set of chain voxels). Layout: bit b = x + V*(y + V*(z - z_lo)), 64-bit
 * little-endian words, only planes z_lo <= z < z_hi. Samples outside the volume [0,V)^3 are
 * counted in *outside; in-volume samples outside the slab are skipped. */
int vo_bitmap(const double* segs, int64_t n, uint64_t* bits, int64_t V, int64_t z_lo,
              int64_t z_hi, int64_t* outside, int nthreads);

/* The same bitmap and outside count, computed z-partitioned for large batches: the volume's
 * planes are cut into chunks and each task owns one chunk's words (plain ORs, no atomics),
 * walking only the k-range of each segment whose rounded z falls in its chunk (found by
 * bisection: the rounded z of S + W*k is monotone in k). Pinned against vo_bitmap. */
int vo_bitmap_zpart(const double* segs, int64_t n, uint64_t* bits, int64_t V, int64_t z_lo,
                    int64_t z_hi, int64_t* outside, int nthreads);

/* Per-chain order-sensitive hash + length (checks multi-GB GPU outputs without storing them):
 * h_i = sum_j (x_j*P1 + y_j*P2 + z_j*P3) * (j+1) mod 2^64, constants in voxline_oracle.c. */
int vo_chain_hashes(const double* segs, int64_t n, uint64_t* hashes, int64_t* lengths,
                    int nthreads);

/* Generators. vo_gen_segment_of_length follows src/bench.cpp:62-83 exactly.
 * vo_gen_segment_in_volume is the volume-fitted variant used by the BASELINE configs
 * (direction first, then start drawn so that both endpoints lie in [1, V-2]^3). */
int vo_gen_segment_of_length(int64_t target, uint64_t seed, double out[6]);
int vo_gen_segment_in_volume(int64_t target, uint64_t seed, int64_t V, double out[6]);
/* Batch generator: segment i uses master draws (jumpable SplitMix64 stream).
 *   fixed length (len_max == 0): L_i = len_fixed, seed_i = draw(i)
 *   arbitrary    (len_max  > 0): L_i = 1 + draw(2i) % len_max, seed_i = draw(2i+1)
 * V == 0 -> reference generator (start in [-50,50]^3), else volume generator. */
int vo_gen_batch(int64_t n, int64_t len_fixed, int64_t len_max, int64_t V, uint64_t seed,
                 double* out, int nthreads);
uint64_t vo_splitmix_draw(uint64_t seed, uint64_t j);
/* src/bench.cpp:85-136 (log-uniform lengths rescaled to an exact total). */
int vo_gen_arbitrary_batch(int64_t total, int64_t count, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif
#endif
