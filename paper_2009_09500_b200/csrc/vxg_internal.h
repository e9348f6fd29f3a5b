// vxg_internal.h -- kernel argument blocks and launchers shared by vxg_kernels.cu and vxg_api.cu.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/voxgpu.h"

namespace vxg {

struct SegRec;
struct Control;

struct ClipEntry {  // one segment's in-slab k-range: items k in [ka, kb) then (optionally) k = n
    long long seg, ka, kb, n;
};

struct PlanArgs {
    const double* segs;  // AoS, 6 doubles per segment, 16-B aligned
    long long n;
    SegRec* rec;
    long long* offsets;  // n + 1
    unsigned long long* status;
    Control* ctl;
};

struct ListArgs {
    const SegRec* rec;
    const long long* off;       // nseg + 1 sample offsets
    long long nseg, total_samples;
    long long nranges;          // contiguous sample ranges, one per resident emit warp
    long long range_len;        // samples per range (a multiple of the staging block)
    long long* range_cnt;       // kCountSplit * nranges: kept voxels per range part (count pass)
    long long* range_pre;       // nranges + 1: exclusive prefix (range scan)
    int32_t* out;               // 3 int32 per voxel, 4-B aligned
    long long out_cap;
    long long* chain_off;       // nseg + 1
    Control* ctl;
    unsigned long long* status; // fused kernel: nranges look-back words (zeroed)
    long long lookahead;        // fused kernel: max count tasks ahead of the emit tasks
    // two-pass kernels with total_samples < 0 ("deferred"): the capacity is off[nseg], written by
    // the plan kernel earlier on the stream, range_len holds the block granularity and the
    // kernels do nothing if plan_ctl records a plan error
    const Control* plan_ctl;
    int fx_off;                 // 1: FP64 samples in the fast runs too (tests, A/B; VXG_LIST_FX=0)
};

struct SmallArgs {           // one-launch run_batch of a small batch (list_small_kernel)
    const double* segs;         // AoS, 6 doubles per segment, 16-B aligned
    long long n, ntiles;
    int32_t* out;               // 3 int32 per voxel
    long long out_cap;
    long long* chain_off;       // n + 1
    unsigned long long* status; // ntiles look-back words (zeroed)
    Control* ctl;               // total, max_steps, pad0 = capacity, n_entries = long segment
    int spw;                    // segments per warp tile (small_spw)
};

struct SingleArgs {          // one segment, one CTA (single_chain_kernel)
    double seg[6];
    long long cap;              // voxels `out` can hold (more are counted, not written)
    long long max_samples;      // the launch's bound on N + 1 (larger: nothing done, host reroutes)
    int32_t* out;               // 3 int32 per voxel (mapped pinned host memory)
    Control* ctl;               // mapped: total, max_steps (= N), err_seg, n_entries (reroute)
};

struct LongArgs {            // one segment over many CTAs (long_chain_kernel)
    double seg[6];
    long long cap;              // voxels `out` can hold (more are counted, not written)
    long long max_samples;      // samples the grid covers (more: nothing done, host reroutes)
    int32_t* out;               // 3 int32 per voxel (device)
    unsigned long long* status; // one look-back word per CTA (zeroed)
    Control* ctl;               // device: total, max_steps (= N), err_seg, n_entries (reroute),
                                // tile_counter (zeroed)
};

struct BitmapArgs {
    const SegRec* rec;
    const ClipEntry* entries;   // CLIP mode only
    const long long* off;       // n_entries + 1
    const long long* tile_seg;
    long long n_entries, total_samples, ntiles;
    unsigned long long* words;
    long long V, z_lo, z_hi;
    Control* ctl;
};

struct TileArgs {  // tile-binned bitmap (vxg_bitmap.cu)
    const SegRec* rec;
    const long long* off;  // n + 1 sample offsets (full plan)
    long long n;
    long long V, z_lo, z_hi;
    int tx, ty, tz;                   // tile size in voxels (tx = 256: one sector per row)
    long long ntx, nty, ntz, ntiles;  // tiles per axis of the box [0,V)^2 x [z_lo,z_hi)
    long long* tile_cnt;              // ntiles * classes (zeroed): pieces per bin, then cursor
    long long* tile_off;              // ntiles * classes + 1: exclusive prefix
    unsigned* tile_cur;               // ntiles * classes: scatter cursors (pieces < 2^32)
    uint4* pieces;                    // 32-B piece records (2 x uint4) binned by tile (vxg_bitmap.cu)
    unsigned long long* words;        // the slab's bitmap (OR-ed into)
    Control* ctl;                     // total: in-volume samples, n_entries: pieces
    int* perm;                        // walk order (segments grouped by length) or null
    SegRec* prec;                     // perm pass: records copied in walk order, or null
    int rec_n;                        // rec holds such copies: N = flags >> kRecNShift
    const int* sel;                   // thin slab: the segments reaching it (g.n of them) or null
    long long* perm_cur;              // tile_perm_keys(): bucket counts, then cursors (zeroed)
    unsigned long long* scan_status;  // bin scan: look-back words, one per 4096 bins (zeroed)
    unsigned* layer_cnt;              // fill (streamed readback): finished tiles per z-layer
    unsigned* layer_done;             // ... and per-layer done flags in mapped host memory, or null
    int bx, by, bz;                   // fill: tiles claimed in blocks of bx x by x bz (0: linear)
    int zero;                         // always 0: a value ptxas cannot see through (fill steps)
    int late_e;                       // fill: E's shared address computed after the samples
    int overwrite;                    // fill: store the tiles (zeros included), no read of the
                                      // old words (VXG_BITMAP_OVERWRITE: no memset either)
    int pf;                           // fill: record prefetch (bit 0: L1 at step start, bit 1: L2
                                      // at step start, bit 2: L1 before the last samples)
};

struct ClipArgs {
    const SegRec* rec;
    const long long* off;  // n + 1 (full plan)
    long long n;
    long long z_lo, z_hi;
    ClipEntry* entries;    // up to n
    long long* ent_off;    // up to n + 1
    unsigned long long* status;
    unsigned long long* status2;
    Control* ctl;
};

struct GenArgs {
    long long n;
    const long long* lens;
    const unsigned long long* seeds;
    long long len_fixed, len_max, V;
    unsigned long long seed;
    double* out;
    Control* ctl;
};

int plan_tile_count(long long n);
int clip_tile_count(long long n);
int list_block_samples();              // samples per staged block
long long list_ranges(int num_sms);     // warp ranges of the list passes
int bitmap_tile_log2();

void launch_plan(const PlanArgs& a, cudaStream_t s);
void launch_tile_index(const long long* off, long long n_entries, int ts_log2, long long* tile_seg,
                       cudaStream_t s);
cudaError_t launch_list_count(const ListArgs& a, cudaStream_t s);  // count pass + range scan
cudaError_t launch_list_emit(const ListArgs& a, cudaStream_t s);   // emit pass
cudaError_t launch_list_fused(const ListArgs& a, int num_sms, cudaStream_t s);  // both, overlapped
cudaError_t launch_single_chain(const SingleArgs& a, cudaStream_t s);
long long long_chain_samples_per_cta();
cudaError_t launch_long_chain(const LongArgs& a, long long ctas, cudaStream_t s);
long long small_tile_count(long long n, int spw);
int small_spw(long long n, int num_sms);
cudaError_t launch_list_small(const SmallArgs& a, int num_sms, cudaStream_t s);
int list_resident_warps(int num_sms);
int list_fused_block_samples();  // fused kernel's staged block
cudaError_t launch_emit_bitmap(const BitmapArgs& a, bool clip, cudaStream_t s);
void launch_clip(const ClipArgs& a, cudaStream_t s);
int tile_dims(long long V, long long depth, int& tx, int& ty, int& tz);  // -> smem bytes
int tile_len_classes();  // piece bins per tile (length classes)
int tile_perm_keys();    // walk-order buckets (length x coarse cell)
void launch_tiles_perm(const TileArgs& g, cudaStream_t s);  // length-grouped walk order
void launch_tiles_count(const TileArgs& g, cudaStream_t s);
void launch_slab_select(const TileArgs& g, int* sel, unsigned long long* nsel, cudaStream_t s);
void launch_select_slab(const double* segs, long long n, long long z_lo, long long z_hi,
                        double* out, unsigned long long* count, cudaStream_t s);
void launch_tiles_scan(const TileArgs& g, cudaStream_t s);  // (look-back scan if g.scan_status)
int tile_scan_tiles(long long nbins);
void launch_tiles_scatter(const TileArgs& g, cudaStream_t s);
cudaError_t launch_tiles_fill(const TileArgs& g, int num_sms, double mean_len, cudaStream_t s);
void launch_round_points(const double* p, long long n, int32_t* out, Control* ctl, cudaStream_t s);
void launch_segment_lengths(const double* segs, long long n, double* out, cudaStream_t s);
void launch_export_plans(const SegRec* rec, const long long* off, long long n,
                         vxg_segment_plan* out, cudaStream_t s);
void launch_pack_plan(const double* segs, const vxg_segment_plan* plans, long long n, SegRec* rec,
                      long long* off, Control* ctl, cudaStream_t s);
void launch_work_item(const SegRec* rec, const long long* off, long long i, long long k,
                      int32_t* out, Control* ctl, cudaStream_t s);
void launch_gen(const GenArgs& a, cudaStream_t s);

}  // namespace vxg
