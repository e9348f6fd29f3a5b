"""The reference's Python API, re-pointed at the B200 path.

Mirrors ``voxline`` (/root/reference/proj/python/voxline/__init__.py:8-48, bound in
bindings/pybind_module.cpp:77-273): same function names, argument meaning, return shapes and
exception classes, so ``import paper_2009_09500_b200 as voxline`` is a drop-in for the
segment-generation API. Every voxel is computed by libvoxgpu's CUDA kernels through the C ABI
(include/voxgpu.h); nothing here evaluates geometry on the CPU.

Out of scope: the candidate-walk oracle (voxelize_walk, candidate_voxels,
chains_equivalent) and point_line_distance, which are not on the parametric hot path.

Beyond the reference surface, flat NumPy entry points (``run_batch_flat``, ``voxelize_bitmap``,
``gen_segments``) return zero-copy arrays instead of lists of tuples.
"""
from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib
from ._lib import (MEM_DEVICE, MEM_HOST, InvalidArgument, default_context, vxg_segment_plan,
                   vxg_timing)

__all__ = [
    "BatchPlan", "batch_preprocess", "batch_voxelize", "chain_length_bounds", "compute_mvps",
    "effective_item_count", "gen_arbitrary_batch", "gen_segment_of_length", "kernel_work_item",
    "make_plan", "round_point", "run_batch", "segment_length", "voxelize_parametric",
    "run_batch_flat", "voxelize_bitmap", "gen_segments", "pinned_empty", "Batch",
    "read_segments_csv", "write_chains", "batch_to_file",
]


# ----------------------------------------------------------------------------- helpers
def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _segments_array(segments) -> np.ndarray:
    """(start, end) pairs / (n,2,3) / (n,6) -> contiguous float64 (n, 6) == vxg_segment[n]."""
    if isinstance(segments, np.ndarray):
        a = segments
    else:
        a = np.asarray(list(segments), dtype=np.float64)
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.size == 0:
        return a.reshape(0, 6)
    return a.reshape(-1, 6)


def _check_host_buffer(a, dtype, name: str, min_size: int = 0, shape_tail=None):
    """Caller-supplied host output buffers are written by the library through a raw pointer:
    check type, layout and size first (InvalidArgument instead of a native overflow)."""
    if not isinstance(a, np.ndarray):
        raise InvalidArgument(f"{name}: expected a numpy array", -1)
    if a.dtype != np.dtype(dtype):
        raise InvalidArgument(f"{name}: dtype {a.dtype}, expected {np.dtype(dtype)}", -1)
    if not a.flags["C_CONTIGUOUS"] or not a.flags["WRITEABLE"]:
        raise InvalidArgument(f"{name}: must be a writeable C-contiguous array", -1)
    if shape_tail is not None and (a.ndim != 1 + len(shape_tail) or a.shape[1:] != shape_tail):
        raise InvalidArgument(f"{name}: shape {a.shape}, expected (rows, {shape_tail[0]})", -1)
    if a.size < min_size:
        raise InvalidArgument(f"{name}: {a.size} elements, need {min_size}", -1)


def _one_segment(start, end) -> np.ndarray:
    s = np.asarray(start, dtype=np.float64).reshape(3)
    e = np.asarray(end, dtype=np.float64).reshape(3)
    return np.ascontiguousarray(np.concatenate([s, e]))


def pinned_empty(shape, dtype) -> np.ndarray:
    """A NumPy array in page-locked host memory (fast DMA); freed with the array."""
    lib = _lib.load()
    dtype = np.dtype(dtype)
    count = int(np.prod(shape)) if np.ndim(shape) else int(shape)
    nbytes = max(count * dtype.itemsize, 1)
    p = lib.vxg_host_alloc(nbytes)
    if not p:
        raise MemoryError(f"vxg_host_alloc({nbytes}) failed")
    buf = (C.c_char * nbytes).from_address(p)
    arr = np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)
    weakref.finalize(buf, lib.vxg_host_free, p)
    return arr


def _chains_from_flat(vox: np.ndarray, off: np.ndarray) -> list:
    rows = [tuple(v) for v in vox.tolist()]
    o = off.tolist()
    return [rows[o[i]:o[i + 1]] for i in range(len(o) - 1)]


def _check_cfg(workers: int, group_size: int):
    # src/batch.cpp:93-96 -- output never depends on the partitioning (one GPU grid)
    if group_size < 1 or workers < 1:
        raise InvalidArgument("batch_voxelize: group_size and worker_count must be >= 1")


# ----------------------------------------------------------------------------- geometry
def segment_length(start, end) -> float:
    """Euclidean length (src/geometry.cpp:8-11), on the GPU."""
    ctx = default_context()
    s = _one_segment(start, end)
    out = np.zeros(1)
    ctx.check(ctx.lib.vxg_segment_lengths(ctx.h, _ptr(s), 1, _ptr(out)))
    return float(out[0])


def round_point(point) -> tuple:
    """Nearest voxel, ties away from zero; ValueError outside int32 (src/geometry.cpp:15-34)."""
    ctx = default_context()
    p = np.ascontiguousarray(np.asarray(point, dtype=np.float64).reshape(3))
    out = np.zeros(3, np.int32)
    ctx.check(ctx.lib.vxg_round_points(ctx.h, _ptr(p), 1, _ptr(out)))
    return (int(out[0]), int(out[1]), int(out[2]))


# ----------------------------------------------------------------------------- parametric
def make_plan(start, end):
    """(N, [wx, wy, wz]) of src/parametric.cpp:8-26, computed by the plan kernel."""
    ctx = default_context()
    s = _one_segment(start, end)
    n = np.zeros(1, np.int64)
    w = np.zeros(3)
    ctx.check(ctx.lib.vxg_make_plans(ctx.h, _ptr(s), 1, _ptr(n), _ptr(w)))
    return int(n[0]), [float(w[0]), float(w[1]), float(w[2])]


def _voxelize_one(seg: np.ndarray) -> np.ndarray:
    ctx = default_context()
    d = np.asarray(seg[3:6], dtype=np.float64) - np.asarray(seg[0:3], dtype=np.float64)
    with np.errstate(all="ignore"):
        bound = max(float(np.sqrt(np.dot(d, d))), float(np.max(np.abs(d)))) + 5.0
    # (N + 1 <= bound: one call; otherwise the count of the first call sizes the second)
    cap = int(bound) if np.isfinite(bound) and bound < 2 ** 31 else 4096
    while True:
        out = np.zeros((cap, 3), np.int32)
        cnt = C.c_int64()
        st = ctx.lib.vxg_voxelize_parametric(ctx.h, _ptr(seg), _ptr(out), cap, C.byref(cnt))
        if st == _lib.VXG_LOGIC_ERROR and cnt.value > cap:
            cap = cnt.value
            continue
        ctx.check(st)
        return out[: cnt.value]


def voxelize_parametric(start, end) -> list:
    """Sample-and-round chain of one segment (src/parametric.cpp:28-40) as a list of tuples."""
    return [tuple(v) for v in _voxelize_one(_one_segment(start, end)).tolist()]


def voxelize_parametric_device(seg, out_ptr: int, cap: int, ctx=None) -> int:
    """voxelize_parametric (src/parametric.cpp:28-40) into device memory: `seg` is one segment
    (sx, sy, sz, ex, ey, ez) in host memory, at most `cap` voxels (3 x int32 each) go to the
    device address `out_ptr`; returns the chain's length (vxg_voxelize_parametric_device: one
    launch and one readback). A chain longer than `cap` raises LogicError."""
    ctx = ctx or default_context()
    s = np.ascontiguousarray(np.asarray(seg, dtype=np.float64).reshape(6))
    cnt = C.c_int64()
    ctx.check(ctx.lib.vxg_voxelize_parametric_device(ctx.h, _ptr(s), C.c_void_p(out_ptr), cap,
                                                     C.byref(cnt)))
    return cnt.value


def voxelize_parametric_host(seg, out: np.ndarray, ctx=None) -> int:
    """voxelize_parametric (src/parametric.cpp:28-40) into a caller's host buffer: `out` is a
    C-contiguous (cap, 3) int32 array (pinned memory makes the copy back direct); returns the
    chain's length. A chain longer than cap raises LogicError."""
    ctx = ctx or default_context()
    _check_host_buffer(out, np.int32, "out", 0, (3,))
    s = np.ascontiguousarray(np.asarray(seg, dtype=np.float64).reshape(6))
    cnt = C.c_int64()
    ctx.check(ctx.lib.vxg_voxelize_parametric(ctx.h, _ptr(s), _ptr(out), out.shape[0],
                                              C.byref(cnt)))
    return cnt.value


def voxelize_parametric_kernel_ns(ctx=None) -> int:
    """GPU time (ns) of the last voxelize_parametric_device launch on the context."""
    ctx = ctx or default_context()
    t = _lib.vxg_timing()
    ctx.check(ctx.lib.vxg_voxelize_parametric_timing(ctx.h, C.byref(t)))
    return t.kernel_ns


def chain_length_bounds(start, end):
    """(span + 1, N + 1) (src/parametric.cpp:42-50)."""
    ctx = default_context()
    s = _one_segment(start, end)
    lo, hi = C.c_int64(), C.c_int64()
    ctx.check(ctx.lib.vxg_chain_length_bounds(ctx.h, _ptr(s), C.byref(lo), C.byref(hi)))
    return (lo.value, hi.value)


# ----------------------------------------------------------------------------- batch engine
BITMAP_CLIP, BITMAP_OVERWRITE = 1, 2  # include/voxgpu.h VXG_BITMAP_*


def _bitmap_flags(clip: bool, overwrite: bool) -> int:
    return (BITMAP_CLIP if clip else 0) | (BITMAP_OVERWRITE if overwrite else 0)


class Batch:
    """A device-resident batch (vxg_batch): segments + plan kept in HBM between calls."""

    def __init__(self, segments, ctx=None, device_ptr: int | None = None, n: int | None = None):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        if device_ptr is not None:
            self._keep = None
            st = self.ctx.lib.vxg_batch_create(self.ctx.h, device_ptr, n, MEM_DEVICE, C.byref(h))
        else:
            a = _segments_array(segments)
            self._keep = a
            st = self.ctx.lib.vxg_batch_create(self.ctx.h, _ptr(a) if a.size else None,
                                               a.shape[0], MEM_HOST, C.byref(h))
        self.ctx.check(st)
        self.h = h
        self.n = int(n) if device_ptr is not None else int(self._keep.shape[0])
        self._info = None  # (max_steps, capacity): read back on first use (vxg_batch_info)
        self._plans = None

    def set_slab(self, z_lo: int, z_hi: int) -> "Batch":
        """State that every segment may reach planes [z_lo, z_hi) (e.g. the output of
        shard.select_slab_segments): bitmaps of slabs inside it skip the tile path's own slab
        filter (vxg_batch_set_slab). Returns self."""
        self.ctx.check(self.ctx.lib.vxg_batch_set_slab(self.h, z_lo, z_hi))
        return self

    def resolve(self):
        """Read the plan's N_max / capacity back (raises the plan's error, if any). A device-
        resident batch defers this; emit_list_device resolves it in its own readback."""
        if self._info is None:
            n_, mx, cap = C.c_int64(), C.c_int64(), C.c_int64()
            self.ctx.check(self.ctx.lib.vxg_batch_info(self.h, C.byref(n_), C.byref(mx),
                                                       C.byref(cap)))
            self._info = (mx.value, cap.value)
        return self._info

    @property
    def max_steps(self) -> int:
        return self.resolve()[0]

    @property
    def capacity(self) -> int:
        return self.resolve()[1]

    def plans(self) -> np.ndarray:
        if self._plans is None:
            arr = (vxg_segment_plan * self.n)()
            self.ctx.check(self.ctx.lib.vxg_batch_plans(self.h, arr))
            self._plans = np.ctypeslib.as_array(arr).copy()
        return self._plans

    def emit_list(self, out=None, chain_off=None):
        """-> (voxels (M,3) int32, chain_offsets (n+1,) int64, total) in host memory. Caller
        buffers must be C-contiguous: out int32 (rows, 3), chain_off int64 with n + 1 entries."""
        if out is None:
            out = pinned_empty((max(self.capacity, 1), 3), np.int32)
        else:
            _check_host_buffer(out, np.int32, "out", shape_tail=(3,))
        if chain_off is None:
            chain_off = pinned_empty((self.n + 1,), np.int64)
        else:
            _check_host_buffer(chain_off, np.int64, "chain_off", min_size=self.n + 1)
        total = C.c_int64()
        self.ctx.check(self.ctx.lib.vxg_batch_emit_list(self.h, _ptr(out), out.shape[0],
                                                        _ptr(chain_off), C.byref(total),
                                                        MEM_HOST))
        return out[: total.value], chain_off, total.value

    def emit_list_device(self, out_ptr: int, out_cap: int, chain_ptr: int) -> int:
        total = C.c_int64()
        self.ctx.check(self.ctx.lib.vxg_batch_emit_list(self.h, out_ptr, out_cap, chain_ptr,
                                                        C.byref(total), MEM_DEVICE))
        return total.value

    def count_voxels(self) -> int:
        """BatchResult.total_voxels without materialising the list (count pass only)."""
        total = C.c_int64()
        self.ctx.check(self.ctx.lib.vxg_batch_count_voxels(self.h, C.byref(total)))
        return total.value

    def emit_bitmap(self, V: int, z_lo: int = 0, z_hi: int | None = None, clip: bool = False,
                    words: np.ndarray | None = None, overwrite: bool | None = None):
        """Bitmap of planes [z_lo, z_hi) into `words` (host). The words are OR-ed into unless
        `overwrite` (default: True when `words` is None, so a fresh bitmap is zeroed on the
        device and nothing but the segments crosses PCIe host->device)."""
        z_hi = V if z_hi is None else z_hi
        nwords = (V * V * (z_hi - z_lo) + 63) // 64
        if overwrite is None:
            overwrite = words is None
        if words is None:
            words = np.empty(max(nwords, 1), np.uint64)
        else:
            _check_host_buffer(words, np.uint64, "words", min_size=nwords)
        outside = C.c_int64()
        self.ctx.check(self.ctx.lib.vxg_batch_emit_bitmap(self.h, _ptr(words), V, z_lo, z_hi,
                                                          _bitmap_flags(clip, overwrite),
                                                          C.byref(outside), MEM_HOST))
        return words[:nwords], outside.value

    def emit_bitmap_device(self, words_ptr: int, V: int, z_lo: int, z_hi: int,
                           clip: bool, overwrite: bool = False) -> int:
        outside = C.c_int64()
        self.ctx.check(self.ctx.lib.vxg_batch_emit_bitmap(self.h, words_ptr, V, z_lo, z_hi,
                                                          _bitmap_flags(clip, overwrite),
                                                          C.byref(outside), MEM_DEVICE))
        return outside.value

    def slab_samples(self, z_lo: int, z_hi: int) -> int:
        s = C.c_int64()
        self.ctx.check(self.ctx.lib.vxg_batch_slab_samples(self.h, z_lo, z_hi, C.byref(s)))
        return s.value

    def work_item(self, i: int, k: int):
        out = np.zeros(3, np.int32)
        live = C.c_int()
        self.ctx.check(self.ctx.lib.vxg_batch_work_item(self.h, i, k, _ptr(out), C.byref(live)))
        return (int(out[0]), int(out[1]), int(out[2])) if live.value else None

    def gpu_timing(self):
        """CUDA-event times (ns) of the last calls on this batch: (plan kernel + offset scan,
        dominant output kernel, auxiliary passes: list count pass + range scan, or the bitmap's
        binning passes)."""
        t = vxg_timing()
        self.ctx.check(self.ctx.lib.vxg_batch_timing(self.h, C.byref(t)))
        return t.preprocess_ns, t.kernel_ns, t.assemble_ns

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.vxg_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class BatchPlan:
    """voxline.BatchPlan (bindings/pybind_module.cpp:177-202): N_max, capacity, per-segment
    step counts and output offsets of a preprocessed batch. Its segments and plan stay in HBM."""

    def __init__(self, batch: Batch, preprocess_ns: int = 0):
        self._batch = batch
        self._preprocess_ns = preprocess_ns

    @property
    def max_steps(self) -> int:
        return self._batch.max_steps

    @property
    def total_voxel_capacity(self) -> int:
        return self._batch.capacity

    @property
    def step_counts(self) -> list:
        return self._batch.plans()["step_count"].tolist()

    @property
    def output_offsets(self) -> list:
        return self._batch.plans()["output_offset"].tolist()

    @property
    def step_vectors(self) -> np.ndarray:
        p = self._batch.plans()
        return np.stack([p["wx"], p["wy"], p["wz"]], axis=1)

    def __len__(self) -> int:
        return self._batch.n


def batch_preprocess(segments) -> BatchPlan:
    """Plans, N_max and offsets for a batch (src/batch.cpp:57-73): plan kernel + look-back scan."""
    import time
    t0 = time.perf_counter_ns()
    b = Batch(segments)
    b.resolve()
    return BatchPlan(b, time.perf_counter_ns() - t0)


def kernel_work_item(plan: BatchPlan, segment_index: int, k: int):
    """One work item; None when redundant (src/batch.cpp:75-90)."""
    return plan._batch.work_item(int(segment_index), int(k))


def _result_dict(vox, off, total, timing) -> dict:
    return {"chains": _chains_from_flat(vox, off), "total_voxels": int(total), "timing": timing}


def batch_voxelize(plan: BatchPlan, workers: int = 1, group_size: int = 64) -> dict:
    """Kernel + assemble phases (src/batch.cpp:92-152) as one GPU emit; preprocess_ns == 0."""
    import time
    _check_cfg(workers, group_size)
    t0 = time.perf_counter_ns()
    vox, off, total = plan._batch.emit_list()
    t1 = time.perf_counter_ns()
    _, emit_ns, aux_ns = plan._batch.gpu_timing()
    kernel_ns = emit_ns + aux_ns  # every GPU pass of the kernel phase
    timing = {"preprocess_ns": 0, "kernel_ns": int(kernel_ns),
              "assemble_ns": int(max(t1 - t0 - kernel_ns, 0))}
    return _result_dict(vox, off, total, timing)


def run_batch(segments, workers: int = 1, group_size: int = 64) -> dict:
    """Preprocess + batch-voxelize (src/batch.cpp:154-162)."""
    _check_cfg(workers, group_size)
    plan = batch_preprocess(segments)
    res = batch_voxelize(plan, workers, group_size)
    res["timing"]["preprocess_ns"] = int(plan._preprocess_ns)
    return res


def effective_item_count(plan: BatchPlan):
    """(live, redundant) items of the N_P x (N_max + 1) grid (src/batch.cpp:164-170)."""
    live, red = C.c_int64(), C.c_int64()
    b = plan._batch
    b.ctx.check(b.ctx.lib.vxg_batch_item_count(b.h, C.byref(live), C.byref(red)))
    return (live.value, red.value)


def run_batch_device(segs_ptr: int, n: int, out_ptr: int, out_cap: int, chain_ptr: int,
                     ctx=None, sync: bool = True):
    """run_batch on device-resident segments into device buffers in one kernel launch (small
    batches; vxg_run_batch_device). sync: return BatchResult.total_voxels; else only enqueue
    (run_batch_device_result() reads it)."""
    ctx = ctx or default_context()
    total = C.c_int64()
    ctx.check(ctx.lib.vxg_run_batch_device(ctx.h, segs_ptr, n, out_ptr, out_cap, chain_ptr,
                                           C.byref(total) if sync else None))
    return total.value if sync else None


def run_batch_device_result(ctx=None):
    """(total_voxels, max_steps, capacity) of the last asynchronous run_batch_device call."""
    ctx = ctx or default_context()
    t, m, c = C.c_int64(), C.c_int64(), C.c_int64()
    ctx.check(ctx.lib.vxg_run_batch_device_result(ctx.h, C.byref(t), C.byref(m), C.byref(c)))
    return t.value, m.value, c.value


def run_batch_flat(segments):
    """run_batch with flat outputs: (voxels int32 (M,3), chain_offsets int64 (n+1,), total)."""
    b = Batch(segments)
    try:
        return b.emit_list()
    finally:
        b.close()


def voxelize_bitmap(segments, V: int, z_lo: int = 0, z_hi: int | None = None,
                    clip: bool = True):
    """Occupancy bitmap (x-fastest bits in uint64 words) of every sample voxel of the batch in
    planes [z_lo, z_hi) of a V^3 volume -> (words, samples outside the volume)."""
    b = Batch(segments)
    try:
        return b.emit_bitmap(V, z_lo, z_hi, clip)
    finally:
        b.close()


# ----------------------------------------------------------------------------- generators
def gen_segment_of_length(target_voxels: int, seed: int):
    """Deterministic segment with exactly `target_voxels` steps (src/bench.cpp:62-83)."""
    if int(target_voxels) < 1:
        raise InvalidArgument("gen_segment_of_length: target must be >= 1")
    a = gen_segments(1, len_fixed=int(target_voxels), seeds=[int(seed)])
    s = a[0].tolist()
    return (s[:3], s[3:])


def gen_segments(n: int, len_fixed: int = 0, len_max: int = 0, V: int = 0, seed: int = 1,
                 seeds=None, lens=None) -> np.ndarray:
    """Synthetic batch on the GPU -> float64 (n, 6). See vxg_gen_segments."""
    ctx = default_context()
    out = np.zeros((max(n, 1), 6))
    if seeds is not None:
        sd = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64).reshape(-1))
        ln = (np.ascontiguousarray(np.asarray(lens, dtype=np.int64).reshape(-1)) if lens is not None
              else np.full(sd.shape[0], len_fixed, np.int64))
        ctx.check(ctx.lib.vxg_gen_segments(ctx.h, n, _ptr(ln), _ptr(sd), 0, 0, V, 0, _ptr(out),
                                           MEM_HOST))
    else:
        ctx.check(ctx.lib.vxg_gen_segments(ctx.h, n, None, None, len_fixed, len_max, V, seed,
                                           _ptr(out), MEM_HOST))
    return out[:n]


def gen_arbitrary_batch(total_voxels_target: int, segment_count: int, seed: int) -> list:
    """Batch whose step counts sum to the target (src/bench.cpp:85-136)."""
    ctx = default_context()
    n = int(segment_count)
    out = np.zeros((max(n, 1), 6))
    ctx.check(ctx.lib.vxg_gen_arbitrary_batch(ctx.h, int(total_voxels_target), n, int(seed),
                                              _ptr(out)))
    return [(r[:3], r[3:]) for r in out[:n].tolist()]


def compute_mvps(total_voxels: int, elapsed_ms: float) -> float:
    """Mega-voxels per second (src/bench.cpp:138-146)."""
    if not (elapsed_ms > 0.0):
        raise InvalidArgument("compute_mvps: elapsed time must be > 0 ms")
    if total_voxels < 0:
        raise InvalidArgument("compute_mvps: negative voxel count")
    return float(total_voxels) / (elapsed_ms / 1000.0) / 1e6


# ----------------------------------------------------------------------------- formats
def read_segments_csv(path: str) -> np.ndarray:
    """read_segments_csv (src/formats.cpp:92-132) -> float64 (n, 6). Malformed line ->
    InvalidArgument naming it (the reference's message); unreadable file -> IoError."""
    lib = _lib.load()
    out = C.c_void_p()
    n, bad = C.c_int64(), C.c_int64()
    st = lib.vxg_read_segments_csv(str(path).encode(), C.byref(out), C.byref(n), C.byref(bad))
    if st == _lib.VXG_INVALID_ARGUMENT:
        raise InvalidArgument(f"segments csv: line {bad.value}: expected 6 finite decimal fields "
                              "(sx,sy,sz,ex,ey,ez)")
    if st == _lib.VXG_IO_ERROR:
        raise _lib.IoError(f"cannot read input file: {path}")
    if st != _lib.VXG_OK:
        raise _lib.VoxGpuError(f"read_segments_csv: status {st}")
    try:
        if n.value == 0:
            return np.zeros((0, 6))
        buf = (C.c_double * (6 * n.value)).from_address(out.value)
        return np.frombuffer(buf, dtype=np.float64).reshape(n.value, 6).copy()
    finally:
        lib.vxg_free(out)


def write_chains(path: str, voxels: np.ndarray, chain_off: np.ndarray, format: str = "vox3"):
    """write_vox3_multi / write_xyz_multi (src/formats.cpp:140-185) of a flat list + offsets."""
    lib = _lib.load()
    v = np.ascontiguousarray(voxels, dtype=np.int32).reshape(-1, 3)
    o = np.ascontiguousarray(chain_off, dtype=np.int64)
    fmt = {"vox3": 0, "xyz": 1}[format]
    st = lib.vxg_write_chains(str(path).encode(), fmt, _ptr(v) if v.size else None, _ptr(o),
                              o.shape[0] - 1)
    if st == _lib.VXG_IO_ERROR:
        raise _lib.IoError(f"cannot open output file: {path}")
    if st != _lib.VXG_OK:
        raise _lib.VoxGpuError(f"write_chains: status {st}")


def batch_to_file(segments, path: str, format: str = "vox3") -> int:
    """The CLI's `batch` (tools/voxline_cli.cpp:101-129) on the GPU: voxelize the batch and
    write every chain; returns total_voxels."""
    vox, off, total = run_batch_flat(segments)
    write_chains(path, vox, off, format)
    return total

