/*
 * voxgpu.h -- C ABI of the B200 parametric segment voxelizer (libvoxgpu.so).
 *
 * The reference (voxline, /root/reference/proj) exposes its hot path only as a C++ header API,
 * statically linked; it has no C ABI or plugin registry. This header is the thin
 * C layer the north_star puts under that API: plain pointers and sizes, no C++ or torch types, no
 * exceptions.  Each entry point names the reference interface it replaces (file:line relative to
 * /root/reference/proj).  The C++ shim (paper_2009_09500_b200/shim/voxline_gpu_core.cpp) and the
 * Python package (paper_2009_09500_b200/_lib.py) are both written on top of it.
 *
 * Memory layouts are byte-identical to the reference's value types:
 *   vxg_segment      == voxline::Segment      (include/voxline/geometry.hpp:35-40, 48 B)
 *   vxg_voxel        == voxline::Voxel        (include/voxline/geometry.hpp:25-32, 12 B)
 *   vxg_segment_plan == voxline::SegmentPlan  (include/voxline/batch.hpp:20-24, 40 B)
 *   vxg_timing       == voxline::BatchTiming  (include/voxline/batch.hpp:42-46)
 *
 * Errors: every call returns a vxg_status; the codes map 1:1 onto the reference's exception
 * classes (SURVEY.md §8b "Error conventions"). vxg_last_error() gives the message and
 * vxg_last_error_segment() the lowest offending segment index (or -1).
 *
 * Pointer spaces: functions taking VXG_MEM flags accept device pointers (VXG_MEM_DEVICE; enqueued
 * on the context stream, no host synchronisation unless a scalar result is returned) or host
 * pointers (VXG_MEM_HOST; staged through pinned buffers, synchronous).
 *
 * Bitmap layout (no reference counterpart): bit b = x + V*(y + V*(z - z_lo)) of little-endian
 * 64-bit words, i.e. x fastest; a z-slab [z_lo, z_hi) is a contiguous piece of the full bitmap.
 */
#ifndef VOXGPU_H
#define VOXGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define VXG_API __attribute__((visibility("default")))
#else
#define VXG_API
#endif

#define VXG_ABI_VERSION 1

typedef enum vxg_status {
    VXG_OK = 0,
    VXG_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    VXG_RANGE_ERROR = 2,      /* std::range_error (non-finite / outside the int32 lattice) */
    VXG_OUT_OF_RANGE = 3,     /* std::out_of_range (kernel_work_item indices) */
    VXG_LOGIC_ERROR = 4,      /* std::logic_error (malformed plan, capacity mismatch) */
    VXG_CUDA_ERROR = 5,       /* CUDA runtime failure */
    VXG_OUT_OF_MEMORY = 6,    /* device or pinned allocation failed */
    VXG_IO_ERROR = 7          /* file cannot be opened / read / written (the CLI's IoError) */
} vxg_status;

typedef enum vxg_mem { VXG_MEM_HOST = 0, VXG_MEM_DEVICE = 1 } vxg_mem;

typedef struct vxg_segment {
    double sx, sy, sz; /* start S */
    double ex, ey, ez; /* end E */
} vxg_segment;

typedef struct vxg_voxel {
    int32_t x, y, z;
} vxg_voxel;

typedef struct vxg_segment_plan {
    int64_t step_count;    /* N_i */
    double wx, wy, wz;     /* W_i */
    int64_t output_offset; /* exclusive prefix sum of N_j + 1 */
} vxg_segment_plan;

typedef struct vxg_timing {
    int64_t preprocess_ns;
    int64_t kernel_ns;
    int64_t assemble_ns;
} vxg_timing;

typedef struct vxg_context vxg_context; /* device, stream, events, pinned staging */
typedef struct vxg_batch vxg_batch;     /* device-resident segments + plan (a voxline::BatchPlan) */

/* ---------------------------------------------------------------- context */
VXG_API int vxg_abi_version(void);
VXG_API vxg_status vxg_create(int device, vxg_context** out);
VXG_API void vxg_destroy(vxg_context* ctx);
/* Use a caller-owned cudaStream_t (NULL = the context's own stream). */
VXG_API vxg_status vxg_set_stream(vxg_context* ctx, void* cuda_stream);
VXG_API void* vxg_get_stream(vxg_context* ctx);
VXG_API const char* vxg_last_error(const vxg_context* ctx);
VXG_API int64_t vxg_last_error_segment(const vxg_context* ctx);
/* Number of this library's kernels launched on ctx so far (evidence counter for bench.py). */
VXG_API int64_t vxg_launch_count(const vxg_context* ctx);
VXG_API vxg_status vxg_synchronize(vxg_context* ctx);
/* Pinned host memory for fast staging (cudaHostAlloc / cudaFreeHost). */
VXG_API void* vxg_host_alloc(size_t bytes);
VXG_API void vxg_host_free(void* p);

/* ---------------------------------------------------------------- geometry / parametric */
/* round_point (src/geometry.cpp:32-34) for n points (3 doubles each) on the GPU. */
VXG_API vxg_status vxg_round_points(vxg_context* ctx, const double* pts, int64_t n, int32_t* out);
/* segment_length (src/geometry.cpp:8-11) for n segments on the GPU. */
VXG_API vxg_status vxg_segment_lengths(vxg_context* ctx, const vxg_segment* segs, int64_t n,
                                       double* out);
/* make_plan (src/parametric.cpp:8-26) for n host segments; steps/w3 host outputs. */
VXG_API vxg_status vxg_make_plans(vxg_context* ctx, const vxg_segment* segs, int64_t n,
                                  int64_t* steps, double* w3);
/* voxelize_parametric (src/parametric.cpp:28-40) of one host segment: the chain goes to host
 * `out` (capacity `cap` voxels; N+1 always suffices), its length to *count. A chain longer than
 * `cap` -> LOGIC_ERROR with the true length in *count and the first `cap` voxels written.
 * Chains up to 2^14 samples take one launch and one synchronisation (single_chain_kernel, the
 * latency regime); longer ones up to 2^30 one multi-CTA launch into device memory and a copy
 * back (long_chain_kernel); longer still the batch passes. */
VXG_API vxg_status vxg_voxelize_parametric(vxg_context* ctx, const vxg_segment* seg,
                                           vxg_voxel* out, int64_t cap, int64_t* count);
/* voxelize_parametric (src/parametric.cpp:28-40) into DEVICE memory: the segment (host memory,
 * passed as launch arguments) is planned and voxelized by one launch over as many CTAs as its
 * length asks for (long_chain_kernel; chains beyond 2^30 samples take the batch passes), then
 * one readback of the count. At most `cap` voxels are written; a longer chain -> LOGIC_ERROR
 * with *count set to its length. */
VXG_API vxg_status vxg_voxelize_parametric_device(vxg_context* ctx, const vxg_segment* seg,
                                                  vxg_voxel* d_out, int64_t cap, int64_t* count);
/* GPU time (CUDA events) of the last long_chain_kernel launch on this context (kernel_ns; the
 * other fields 0; all 0 before the first). */
VXG_API vxg_status vxg_voxelize_parametric_timing(vxg_context* ctx, vxg_timing* t);
/* chain_length_bounds (src/parametric.cpp:42-50). */
VXG_API vxg_status vxg_chain_length_bounds(vxg_context* ctx, const vxg_segment* seg,
                                           int64_t* lo, int64_t* hi);

/* ---------------------------------------------------------------- batch engine */
/* batch_preprocess (src/batch.cpp:57-73): upload n segments (host or device pointer) and build
 * the plan on the GPU (plan kernel + decoupled look-back offset scan). Empty -> INVALID_ARGUMENT;
 * bad endpoint -> RANGE_ERROR (lowest segment index reported).
 * VXG_MEM_HOST: synchronous; plan errors are returned here. VXG_MEM_DEVICE: only enqueued -- the
 * plan's N_max / capacity and any plan error are read back by the first call that needs them
 * (vxg_batch_info, or the single readback of a device-pointer vxg_batch_emit_list on a batch of
 * fewer than 2^18 segments), which then returns the plan's error; every later call repeats it. */
VXG_API vxg_status vxg_batch_create(vxg_context* ctx, const vxg_segment* segs, int64_t n,
                                    vxg_mem where, vxg_batch** out);
/* A batch from a caller-supplied plan (batch_voxelize takes `const BatchPlan&`,
 * src/batch.cpp:92-105): validates like the reference (LOGIC_ERROR on mismatch). */
VXG_API vxg_status vxg_batch_from_plan(vxg_context* ctx, const vxg_segment* segs,
                                       const vxg_segment_plan* plans, int64_t n,
                                       int64_t max_steps, int64_t capacity, vxg_batch** out);
VXG_API void vxg_batch_destroy(vxg_batch* b);
/* BatchPlan scalars: N_P, N_max, total_voxel_capacity (src/batch.cpp:67-71). */
VXG_API vxg_status vxg_batch_info(const vxg_batch* b, int64_t* n, int64_t* max_steps,
                                  int64_t* capacity);
/* Per-segment plans to host (BatchPlan::per_segment). */
VXG_API vxg_status vxg_batch_plans(vxg_batch* b, vxg_segment_plan* out);
/* effective_item_count (src/batch.cpp:164-170). */
VXG_API vxg_status vxg_batch_item_count(const vxg_batch* b, int64_t* live, int64_t* redundant);
/* kernel_work_item (src/batch.cpp:75-90): *live = 0 for redundant items (k > N_i),
 * OUT_OF_RANGE outside [0,N_P) x [0,N_max]. Evaluated on the GPU. */
VXG_API vxg_status vxg_batch_work_item(vxg_batch* b, int64_t i, int64_t k, int32_t out[3],
                                       int* live);
/* Kernel + assemble phases of batch_voxelize (src/batch.cpp:107-150) on the GPU: every sample of
 * the flat (segment, k) space is evaluated by a warp row of 32, consecutive duplicates are dropped
 * in registers, and the kept voxels are compacted into the list (a count task per range, a prefix,
 * an emit task per range; fused into one kernel for large batches). Chain i is
 * out[chain_off[i] .. chain_off[i+1]); *total = BatchResult.total_voxels.
 * `out` needs room for `total` voxels (capacity always suffices); chain_off has n+1 entries.
 * where == VXG_MEM_HOST: out/chain_off are host pointers (D2H included, synchronous).
 * where == VXG_MEM_DEVICE: device pointers; *total still returned (one 8-byte readback). */
VXG_API vxg_status vxg_batch_emit_list(vxg_batch* b, vxg_voxel* out, int64_t out_cap,
                                       int64_t* chain_off, int64_t* total, vxg_mem where);
/* BatchResult.total_voxels (src/batch.cpp:148-150) without materialising the list: the count
 * pass of vxg_batch_emit_list (every sample evaluated, consecutive duplicates dropped) and its
 * range prefix; one 8-byte readback. Sizes a host list exactly, and is the voxel count of a
 * batch whose output is a bitmap. */
VXG_API vxg_status vxg_batch_count_voxels(vxg_batch* b, int64_t* total);
/* Occupancy bitmap of the batch's samples restricted to planes [z_lo, z_hi) of a V^3 volume.
 * Samples outside [0,V)^3 are skipped and counted in *outside (may be NULL). `words` holds
 * V*V*(z_hi-z_lo)/64 uint64 (rounded up) and is OR-ed into (caller zeroes it).
 * V % 128 == 0 (and every N_i < 2^31): the tile-binned path -- segments are walked through
 * 128x120x120-voxel tiles (clipped to the slab on the device, the z-slab partitioner), their
 * in-tile k-ranges binned, every tile filled in shared memory and OR-ed into `words` once.
 * Other volumes: one global atomic per sample; VXG_BITMAP_CLIP then clips every segment's
 * k-range to the slab first (work proportional to the slab's samples), without it every sample
 * is scanned. `flags` is a bit set of VXG_BITMAP_*; VXG_BITMAP_OVERWRITE zeroes `words` on the
 * device first instead of OR-ing into them (with VXG_MEM_HOST it also skips uploading the
 * caller's words: the host->device traffic is the segments only). */
#define VXG_BITMAP_CLIP 1
#define VXG_BITMAP_OVERWRITE 2
VXG_API vxg_status vxg_batch_emit_bitmap(vxg_batch* b, uint64_t* words, int64_t V, int64_t z_lo,
                                         int64_t z_hi, int flags, int64_t* outside, vxg_mem where);
/* Samples of the batch whose rounded z lies in [z_lo, z_hi) (the slab's work). */
/* The z-slab partitioner's filter (multi-GPU bitmaps): copy to `out` (device)
 * the segments of `segs` (device, n) whose samples can reach planes [z_lo, z_hi) -- a
 * conservative test on the endpoints' z (2 planes of slack; non-finite endpoints are kept, so
 * the plan still reports them) -- in an unspecified order; *n_out gets their count. A rank's
 * bitmap of its slab from the filtered batch equals the slab of the full batch's bitmap. */
VXG_API vxg_status vxg_select_slab_segments(vxg_context* ctx, const vxg_segment* segs, int64_t n,
                                            int64_t z_lo, int64_t z_hi, vxg_segment* out,
                                            int64_t* n_out);
VXG_API vxg_status vxg_batch_slab_samples(vxg_batch* b, int64_t z_lo, int64_t z_hi,
                                          int64_t* samples);
/* The caller states that every segment of the batch may reach planes [z_lo, z_hi) -- e.g. they
 * came out of vxg_select_slab_segments for that slab: bitmaps of slabs inside it then skip the
 * tile path's own slab filter (which would keep every segment). Purely a shortcut: the output is
 * the same either way. */
VXG_API vxg_status vxg_batch_set_slab(vxg_batch* b, int64_t z_lo, int64_t z_hi);
/* GPU time (ns, CUDA events) on this batch of the last plan kernel + offset scan (preprocess_ns),
 * the dominant output kernel (kernel_ns: list emit pass or bitmap tile fill) and the auxiliary
 * passes before it (assemble_ns: list count pass + range scan, or the bitmap binning passes). */
VXG_API vxg_status vxg_batch_timing(const vxg_batch* b, vxg_timing* t);

/* run_batch (src/batch.cpp:154-162) on DEVICE-resident segments into device buffers, for small
 * batches in ONE kernel launch: plan, count, output prefix (decoupled look-back over tiles of 64
 * segments) and emit fused (the latency regime, config 1). out: room for out_cap voxels;
 * chain_off: n + 1 entries. total != NULL: synchronous, *total = BatchResult.total_voxels.
 * total == NULL: only enqueued on the context's stream; vxg_run_batch_device_result reads the
 * result of the last such call (the segments must stay valid until then). Batches holding a
 * segment with more than 2^14 steps take the multi-pass path (same results). */
VXG_API vxg_status vxg_run_batch_device(vxg_context* ctx, const vxg_segment* segs, int64_t n,
                                        vxg_voxel* out, int64_t out_cap, int64_t* chain_off,
                                        int64_t* total);
/* Result of the last vxg_run_batch_device call enqueued without a total: synchronises; also
 * N_max and the capacity (sum of N_i + 1) of its plan (either may be NULL). */
VXG_API vxg_status vxg_run_batch_device_result(vxg_context* ctx, int64_t* total,
                                               int64_t* max_steps, int64_t* capacity);

/* run_batch (src/batch.cpp:154-162) with host buffers: upload, plan, emit, read back.
 * out needs room for the capacity (use vxg_batch_* for a two-step sized call). */
VXG_API vxg_status vxg_run_batch(vxg_context* ctx, const vxg_segment* segs, int64_t n,
                                 vxg_voxel* out, int64_t out_cap, int64_t* chain_off,
                                 int64_t* total, vxg_timing* timing);

/* ---------------------------------------------------------------- synthetic inputs */
/* SplitMix64-driven generators on the GPU (src/bench.cpp:62-83 rule: exact step count).
 * lens/seeds given (device or host per `where`): segment i = gen(lens[i], seeds[i]).
 * lens == NULL: master stream `seed`; len_max > 0 -> L_i = 1 + draw(2i) % len_max,
 *   seed_i = draw(2i+1); else L_i = len_fixed, seed_i = draw(i).
 * V == 0: gen_segment_of_length (start in [-50,50]^3); V > 0: volume-fitted (both endpoints in
 * [1, V-2]^3). Output `out` (n segments) in the same memory space as `where`. */
VXG_API vxg_status vxg_gen_segments(vxg_context* ctx, int64_t n, const int64_t* lens,
                                    const uint64_t* seeds, int64_t len_fixed, int64_t len_max,
                                    int64_t V, uint64_t seed, vxg_segment* out, vxg_mem where);
/* gen_arbitrary_batch (src/bench.cpp:85-136): host length planning, GPU segment generation. */
VXG_API vxg_status vxg_gen_arbitrary_batch(vxg_context* ctx, int64_t total, int64_t count,
                                           uint64_t seed, vxg_segment* out);

/* ---------------------------------------------------------------- formats (host, native) */
/* read_segments_csv (src/formats.cpp:92-132) of a file: six finite decimal fields per line
 * (sx,sy,sz,ex,ey,ez), '#' and blank lines skipped. On success *out holds *n segments (malloc'd:
 * release with vxg_free). A malformed line -> VXG_INVALID_ARGUMENT with its 1-based number in
 * *bad_line (the first one, as the reference's serial parser reports); no file -> VXG_IO_ERROR. */
VXG_API vxg_status vxg_read_segments_csv(const char* path, vxg_segment** out, int64_t* n,
                                         int64_t* bad_line);
VXG_API void vxg_free(void* p);
/* write_vox3_multi (format 0, VOX3 version 2) / write_xyz_multi (format 1)
 * (src/formats.cpp:140-185) of n chains given as a flat list + chain offsets (n + 1 entries), as
 * vxg_batch_emit_list returns them. Byte-identical to the reference's writers. */
VXG_API vxg_status vxg_write_chains(const char* path, int format, const vxg_voxel* voxels,
                                    const int64_t* chain_off, int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* VOXGPU_H */
