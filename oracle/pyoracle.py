"""ctypes view of the parity checkers (TEST INFRASTRUCTURE ONLY).

``Oracle`` wraps ``oracle/_build/liboracle.so`` (the C restatement, voxline_oracle.c) and
``RefOracle`` wraps ``oracle/_ref/libref_voxline.so`` (the reference compiled unmodified from
/root/reference by oracle/Makefile).  Both expose the same numpy-level API so tests can pin one
against the other.  Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu-baseline legs
may import this module; the product package never does.

Error codes map to the reference's exception classes (voxline_oracle.h):
0 ok, 1 invalid_argument, 2 range_error, 3 out_of_range, 4 logic_error.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
HASH_P = (0x9E3779B97F4A7C15, 0xC2B2AE3D27D4EB4F, 0x165667B19E3779F9)  # vo_chain_hashes
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_voxline.so")

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_u64p = C.POINTER(C.c_uint64)

ERRORS = {1: ValueError, 2: ValueError, 3: IndexError, 4: RuntimeError, 5: RuntimeError}
ERROR_NAMES = {0: "ok", 1: "invalid_argument", 2: "range_error", 3: "out_of_range", 4: "logic_error"}


class OracleError(Exception):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {ERROR_NAMES.get(code, code)}")
        self.code = code


def _p(a, t):
    return a.ctypes.data_as(t)


def _check(code, where):
    if code:
        raise OracleError(code, where)


def build(ref: bool = True) -> None:
    """Compile the checkers (make -C oracle [ref])."""
    targets = ["all"]
    if ref and os.path.isdir("/root/reference/proj"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def as_segments(segs) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(segs, dtype=np.float64).reshape(-1, 6))
    return a


class Oracle:
    """The C restatement (oracle/voxline_oracle.c)."""

    prefix = "vo_"

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        self.lib = C.CDLL(path)
        L = self.lib
        L.vo_splitmix_next.restype = C.c_uint64
        L.vo_splitmix_next.argtypes = [_u64p]
        L.vo_splitmix_draw.restype = C.c_uint64
        L.vo_splitmix_draw.argtypes = [C.c_uint64, C.c_uint64]
        L.vo_segment_length.restype = C.c_double
        L.vo_segment_length.argtypes = [_f64p]
        L.vo_round_point.argtypes = [_f64p, _i32p]
        L.vo_make_plan.argtypes = [_f64p, _i64p, _f64p]
        L.vo_voxelize_parametric.argtypes = [_f64p, _i32p, C.c_int64, _i64p]
        L.vo_chain_length_bounds.argtypes = [_f64p, _i64p, _i64p]
        L.vo_batch_preprocess.argtypes = [_f64p, C.c_int64, _i64p, _f64p, _i64p, _i64p, _i64p]
        L.vo_kernel_work_item.argtypes = [_f64p, C.c_int64, _i64p, _f64p, C.c_int64, C.c_int64,
                                          C.c_int64, _i32p, C.POINTER(C.c_int)]
        L.vo_run_batch.argtypes = [_f64p, C.c_int64, _i32p, C.c_int64, _i64p, _i64p, C.c_int]
        L.vo_chain_lengths.argtypes = [_f64p, C.c_int64, _i64p, C.c_int]
        L.vo_bitmap.argtypes = [_f64p, C.c_int64, _u64p, C.c_int64, C.c_int64, C.c_int64, _i64p,
                                C.c_int]
        L.vo_bitmap_zpart.argtypes = L.vo_bitmap.argtypes
        L.vo_check_round_pos.restype = C.c_int64
        L.vo_check_round_pos.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_int, _i64p,
                                         C.POINTER(C.c_double)]
        L.vo_chain_hashes.argtypes = [_f64p, C.c_int64, _u64p, _i64p, C.c_int]
        L.vo_gen_segment_of_length.argtypes = [C.c_int64, C.c_uint64, _f64p]
        L.vo_gen_segment_in_volume.argtypes = [C.c_int64, C.c_uint64, C.c_int64, _f64p]
        L.vo_gen_batch.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, _f64p,
                                   C.c_int]
        L.vo_gen_arbitrary_batch.argtypes = [C.c_int64, C.c_int64, C.c_uint64, _f64p]

    # --- scalar API -----------------------------------------------------------------
    def splitmix(self, seed: int, count: int) -> list[int]:
        st = C.c_uint64(seed)
        return [self.lib.vo_splitmix_next(C.byref(st)) for _ in range(count)]

    def segment_length(self, seg) -> float:
        s = as_segments(seg)[0]
        return self.lib.vo_segment_length(_p(s, _f64p))

    def round_point(self, p):
        a = np.ascontiguousarray(np.asarray(p, dtype=np.float64))
        out = np.zeros(3, np.int32)
        _check(self.lib.vo_round_point(_p(a, _f64p), _p(out, _i32p)), "round_point")
        return tuple(int(v) for v in out)

    def make_plan(self, seg):
        s = as_segments(seg)[0]
        n = C.c_int64()
        w = np.zeros(3)
        _check(self.lib.vo_make_plan(_p(s, _f64p), C.byref(n), _p(w, _f64p)), "make_plan")
        return n.value, tuple(float(x) for x in w)

    def voxelize_parametric(self, seg) -> np.ndarray:
        s = as_segments(seg)[0]
        n, _ = self.make_plan(s)
        out = np.zeros((n + 1, 3), np.int32)
        cnt = C.c_int64()
        _check(self.lib.vo_voxelize_parametric(_p(s, _f64p), _p(out, _i32p), n + 1, C.byref(cnt)),
               "voxelize_parametric")
        return out[: cnt.value].copy()

    def chain_length_bounds(self, seg):
        s = as_segments(seg)[0]
        lo, hi = C.c_int64(), C.c_int64()
        _check(self.lib.vo_chain_length_bounds(_p(s, _f64p), C.byref(lo), C.byref(hi)),
               "chain_length_bounds")
        return lo.value, hi.value

    # --- batch API ------------------------------------------------------------------
    def batch_preprocess(self, segs):
        s = as_segments(segs)
        n = s.shape[0]
        steps = np.zeros(max(n, 1), np.int64)
        w = np.zeros((max(n, 1), 3))
        off = np.zeros(max(n, 1), np.int64)
        mx, cap = C.c_int64(), C.c_int64()
        _check(self.lib.vo_batch_preprocess(_p(s, _f64p), n, _p(steps, _i64p), _p(w, _f64p),
                                            _p(off, _i64p), C.byref(mx), C.byref(cap)),
               "batch_preprocess")
        return dict(steps=steps[:n], step_vectors=w[:n], offsets=off[:n], max_steps=mx.value,
                    capacity=cap.value)

    def run_batch(self, segs, nthreads: int = 0):
        """-> (voxels int32[M,3], chain_offsets int64[n+1], total)."""
        s = as_segments(segs)
        n = s.shape[0]
        off = np.zeros(n + 1, np.int64)
        total = C.c_int64()
        _check(self.lib.vo_run_batch(_p(s, _f64p), n, None, 0, _p(off, _i64p), C.byref(total),
                                     nthreads), "run_batch")
        out = np.zeros((max(total.value, 1), 3), np.int32)
        _check(self.lib.vo_run_batch(_p(s, _f64p), n, _p(out, _i32p), total.value, _p(off, _i64p),
                                     C.byref(total), nthreads), "run_batch")
        return out[: total.value], off, total.value

    def chain_lengths(self, segs, nthreads: int = 0) -> np.ndarray:
        s = as_segments(segs)
        n = s.shape[0]
        out = np.zeros(max(n, 1), np.int64)
        _check(self.lib.vo_chain_lengths(_p(s, _f64p), n, _p(out, _i64p), nthreads),
               "chain_lengths")
        return out[:n]

    def bitmap(self, segs, V: int, z_lo: int = 0, z_hi: int | None = None, nthreads: int = 0,
               zpart: bool = False):
        """-> (uint64 words, outside count); bit b = x + V*(y + V*(z - z_lo)).
        zpart: the z-partitioned evaluation (vo_bitmap_zpart) for large batches."""
        s = as_segments(segs)
        z_hi = V if z_hi is None else z_hi
        nbits = V * V * (z_hi - z_lo)
        words = np.zeros((nbits + 63) // 64, np.uint64)
        outside = C.c_int64()
        fn = self.lib.vo_bitmap_zpart if zpart else self.lib.vo_bitmap
        _check(fn(_p(s, _f64p), s.shape[0], _p(words, _u64p), V, z_lo, z_hi, C.byref(outside),
                  nthreads), "bitmap")
        return words, outside.value

    def check_round_pos(self, ties: int, rnd: int, seed: int = 7, mode: int = 0):
        """Host check of the GPU's one-DADD rounding (round_pos) against llround ->
        (mismatches, values checked, first mismatching value); see round_pos_check.c."""
        n, fb = C.c_int64(), C.c_double()
        bad = self.lib.vo_check_round_pos(ties, rnd, seed, mode, C.byref(n), C.byref(fb))
        return bad, n.value, fb.value

    def chain_hashes(self, segs, nthreads: int = 0):
        """-> (uint64 hash per chain, int64 length per chain); see vo_chain_hashes."""
        s = as_segments(segs)
        n = s.shape[0]
        h = np.zeros(max(n, 1), np.uint64)
        ln = np.zeros(max(n, 1), np.int64)
        _check(self.lib.vo_chain_hashes(_p(s, _f64p), n, _p(h, _u64p), _p(ln, _i64p), nthreads),
               "chain_hashes")
        return h[:n], ln[:n]

    # --- generators -----------------------------------------------------------------
    def gen_segment_of_length(self, target: int, seed: int) -> np.ndarray:
        out = np.zeros(6)
        _check(self.lib.vo_gen_segment_of_length(target, seed, _p(out, _f64p)),
               "gen_segment_of_length")
        return out

    def gen_segment_in_volume(self, target: int, seed: int, V: int) -> np.ndarray:
        out = np.zeros(6)
        _check(self.lib.vo_gen_segment_in_volume(target, seed, V, _p(out, _f64p)),
               "gen_segment_in_volume")
        return out

    def gen_batch(self, n: int, len_fixed: int = 0, len_max: int = 0, V: int = 0, seed: int = 1,
                  nthreads: int = 0) -> np.ndarray:
        out = np.zeros((n, 6))
        _check(self.lib.vo_gen_batch(n, len_fixed, len_max, V, seed, _p(out, _f64p), nthreads),
               "gen_batch")
        return out

    def gen_arbitrary_batch(self, total: int, count: int, seed: int) -> np.ndarray:
        out = np.zeros((max(count, 1), 6))
        _check(self.lib.vo_gen_arbitrary_batch(total, count, seed, _p(out, _f64p)),
               "gen_arbitrary_batch")
        return out[:count]


class RefOracle:
    """The reference implementation compiled unmodified (oracle/_ref/libref_voxline.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_round_point.argtypes = [_f64p, _i32p]
        L.ref_segment_length.restype = C.c_double
        L.ref_segment_length.argtypes = [_f64p]
        L.ref_make_plan.argtypes = [_f64p, _i64p, _f64p]
        L.ref_voxelize_parametric.argtypes = [_f64p, _i32p, C.c_int64, _i64p]
        L.ref_chain_length_bounds.argtypes = [_f64p, _i64p, _i64p]
        L.ref_batch_preprocess.argtypes = [_f64p, C.c_int64, _i64p, _f64p, _i64p, _i64p, _i64p,
                                           _i64p, _i64p]
        L.ref_kernel_work_item.argtypes = [_f64p, C.c_int64, C.c_int64, C.c_int64, _i32p,
                                           C.POINTER(C.c_int)]
        L.ref_run_batch.argtypes = [_f64p, C.c_int64, C.c_int, C.c_int, _i32p, C.c_int64, _i64p,
                                    _i64p, _i64p]
        L.ref_gen_segment_of_length.argtypes = [C.c_int64, C.c_uint64, _f64p]
        L.ref_gen_arbitrary_batch.argtypes = [C.c_int64, C.c_int64, C.c_uint64, _f64p]
        L.ref_splitmix_next.restype = C.c_uint64
        L.ref_splitmix_next.argtypes = [_u64p]
        L.ref_compute_mvps.restype = C.c_double
        L.ref_compute_mvps.argtypes = [C.c_int64, C.c_double, C.POINTER(C.c_int)]
        L.ref_read_segments_csv.argtypes = [C.c_char_p, _f64p, C.c_int64, _i64p, C.c_char_p,
                                            C.c_int64]
        L.ref_batch_write.argtypes = [_f64p, C.c_int64, C.c_char_p, C.c_int]
        L.ref_run_batch_bitmap.argtypes = [_f64p, C.c_int64, C.c_int, C.c_int, _u64p, C.c_int64,
                                           C.c_int64, C.c_int64, _i64p, _i64p, _i64p]
        L.ref_sequential_map.argtypes = [_f64p, C.c_int64, _i64p]

    def splitmix(self, seed: int, count: int) -> list[int]:
        st = C.c_uint64(seed)
        return [self.lib.ref_splitmix_next(C.byref(st)) for _ in range(count)]

    def segment_length(self, seg) -> float:
        s = as_segments(seg)[0]
        return self.lib.ref_segment_length(_p(s, _f64p))

    def round_point(self, p):
        a = np.ascontiguousarray(np.asarray(p, dtype=np.float64))
        out = np.zeros(3, np.int32)
        _check(self.lib.ref_round_point(_p(a, _f64p), _p(out, _i32p)), "round_point")
        return tuple(int(v) for v in out)

    def make_plan(self, seg):
        s = as_segments(seg)[0]
        n = C.c_int64()
        w = np.zeros(3)
        _check(self.lib.ref_make_plan(_p(s, _f64p), C.byref(n), _p(w, _f64p)), "make_plan")
        return n.value, tuple(float(x) for x in w)

    def voxelize_parametric(self, seg) -> np.ndarray:
        s = as_segments(seg)[0]
        cnt = C.c_int64()
        _check(self.lib.ref_voxelize_parametric(_p(s, _f64p), None, 0, C.byref(cnt)),
               "voxelize_parametric")
        out = np.zeros((max(cnt.value, 1), 3), np.int32)
        _check(self.lib.ref_voxelize_parametric(_p(s, _f64p), _p(out, _i32p), cnt.value,
                                                C.byref(cnt)), "voxelize_parametric")
        return out[: cnt.value]

    def chain_length_bounds(self, seg):
        s = as_segments(seg)[0]
        lo, hi = C.c_int64(), C.c_int64()
        _check(self.lib.ref_chain_length_bounds(_p(s, _f64p), C.byref(lo), C.byref(hi)),
               "chain_length_bounds")
        return lo.value, hi.value

    def batch_preprocess(self, segs):
        s = as_segments(segs)
        n = s.shape[0]
        steps = np.zeros(max(n, 1), np.int64)
        w = np.zeros((max(n, 1), 3))
        off = np.zeros(max(n, 1), np.int64)
        mx, cap, live, red = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        _check(self.lib.ref_batch_preprocess(_p(s, _f64p), n, _p(steps, _i64p), _p(w, _f64p),
                                             _p(off, _i64p), C.byref(mx), C.byref(cap),
                                             C.byref(live), C.byref(red)), "batch_preprocess")
        return dict(steps=steps[:n], step_vectors=w[:n], offsets=off[:n], max_steps=mx.value,
                    capacity=cap.value, live=live.value, redundant=red.value)

    def kernel_work_item(self, segs, i, k):
        s = as_segments(segs)
        out = np.zeros(3, np.int32)
        live = C.c_int()
        _check(self.lib.ref_kernel_work_item(_p(s, _f64p), s.shape[0], i, k, _p(out, _i32p),
                                             C.byref(live)), "kernel_work_item")
        return tuple(int(v) for v in out) if live.value else None

    def run_batch(self, segs, workers: int = 1, group_size: int = 64, with_voxels: bool = True):
        """-> (voxels int32[M,3] or None, chain_offsets int64[n+1], total, timing_ns[3])."""
        s = as_segments(segs)
        n = s.shape[0]
        off = np.zeros(n + 1, np.int64)
        total = C.c_int64()
        timing = np.zeros(3, np.int64)
        if not with_voxels:
            _check(self.lib.ref_run_batch(_p(s, _f64p), n, workers, group_size, None, 0,
                                          _p(off, _i64p), C.byref(total), _p(timing, _i64p)),
                   "run_batch")
            return None, off, total.value, timing
        # one pass to size, one to fill (the reference has no flat API)
        _check(self.lib.ref_run_batch(_p(s, _f64p), n, workers, group_size, None, 0,
                                      _p(off, _i64p), C.byref(total), None), "run_batch")
        out = np.zeros((max(total.value, 1), 3), np.int32)
        _check(self.lib.ref_run_batch(_p(s, _f64p), n, workers, group_size, _p(out, _i32p),
                                      total.value, _p(off, _i64p), C.byref(total),
                                      _p(timing, _i64p)), "run_batch")
        return out[: total.value], off, total.value, timing

    def run_batch_bitmap(self, segs, V: int, z_lo: int = 0, z_hi: int | None = None,
                         workers: int = 1, group_size: int = 64, words=None):
        """The bitmap configs' CPU arm: run_batch, then the harness bit-setting pass over its
        chains. -> (words, total_voxels, outside, (run_batch ns, bit-setting ns))."""
        s = as_segments(segs)
        z_hi = V if z_hi is None else z_hi
        nwords = (V * V * (z_hi - z_lo) + 63) // 64
        if words is None:
            words = np.zeros(nwords, np.uint64)
        total, outside = C.c_int64(), C.c_int64()
        t = np.zeros(2, np.int64)
        _check(self.lib.ref_run_batch_bitmap(_p(s, _f64p), s.shape[0], workers, group_size,
                                             _p(words, _u64p), V, z_lo, z_hi, C.byref(total),
                                             C.byref(outside), _p(t, _i64p)), "run_batch_bitmap")
        return words, total.value, outside.value, (int(t[0]), int(t[1]))

    def sequential_map(self, segs) -> int:
        """src/bench.cpp:188-205: voxelize_parametric per segment on this thread -> total."""
        s = as_segments(segs)
        total = C.c_int64()
        _check(self.lib.ref_sequential_map(_p(s, _f64p), s.shape[0], C.byref(total)),
               "sequential_map")
        return total.value

    def gen_segment_of_length(self, target: int, seed: int) -> np.ndarray:
        out = np.zeros(6)
        _check(self.lib.ref_gen_segment_of_length(target, seed, _p(out, _f64p)),
               "gen_segment_of_length")
        return out

    def gen_arbitrary_batch(self, total: int, count: int, seed: int) -> np.ndarray:
        out = np.zeros((max(count, 1), 6))
        _check(self.lib.ref_gen_arbitrary_batch(total, count, seed, _p(out, _f64p)),
               "gen_arbitrary_batch")
        return out[:count]

    def compute_mvps(self, total: int, ms: float) -> float:
        err = C.c_int()
        v = self.lib.ref_compute_mvps(total, ms, C.byref(err))
        _check(err.value, "compute_mvps")
        return v

    # --- formats (src/formats.cpp) ------------------------------------------------
    def read_segments_csv(self, path: str):
        """-> (float64 (n, 6), None) or (None, the reference's invalid_argument message)."""
        n = C.c_int64()
        msg = C.create_string_buffer(512)
        rc = self.lib.ref_read_segments_csv(str(path).encode(), None, 0, C.byref(n), msg, 512)
        if rc:
            return None, msg.value.decode()
        out = np.zeros((max(n.value, 1), 6))
        rc = self.lib.ref_read_segments_csv(str(path).encode(), _p(out, _f64p), n.value,
                                            C.byref(n), msg, 512)
        return out[: n.value], None

    def batch_write(self, segs, path: str, fmt: str = "vox3"):
        """The reference CLI's batch output: run_batch + write_vox3_multi / write_xyz_multi."""
        s = as_segments(segs)
        _check(self.lib.ref_batch_write(_p(s, _f64p), s.shape[0], str(path).encode(),
                                        {"vox3": 0, "xyz": 1}[fmt]), "batch_write")
