"""ctypes binding of libvoxgpu.so (the C ABI in include/voxgpu.h).

This is the only way the Python package reaches the GPU. There is no CPU fallback: if the
library is missing or no CUDA device is present the calls raise. Status codes map onto the
exception classes the reference's pybind11 module raises: invalid_argument and
range_error -> ValueError, out_of_range -> IndexError, logic_error -> RuntimeError.
"""
from __future__ import annotations

import ctypes as C
import os
import re
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VXG_LIBRARY", os.path.join(HERE, "lib", "libvoxgpu.so"))
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "voxgpu.h")

VXG_OK = 0
VXG_INVALID_ARGUMENT = 1
VXG_RANGE_ERROR = 2
VXG_OUT_OF_RANGE = 3
VXG_LOGIC_ERROR = 4
VXG_CUDA_ERROR = 5
VXG_OUT_OF_MEMORY = 6
VXG_IO_ERROR = 7
MEM_HOST = 0
MEM_DEVICE = 1


class VoxGpuError(Exception):
    """Base of every libvoxgpu failure; `code` is the vxg_status, `segment` the lowest index."""

    code = -1

    def __init__(self, message: str, segment: int = -1):
        super().__init__(message)
        self.segment = segment


class InvalidArgument(VoxGpuError, ValueError):  # std::invalid_argument
    code = VXG_INVALID_ARGUMENT


class RangeError(VoxGpuError, ValueError):  # std::range_error
    code = VXG_RANGE_ERROR


class OutOfRange(VoxGpuError, IndexError):  # std::out_of_range
    code = VXG_OUT_OF_RANGE


class LogicError(VoxGpuError, RuntimeError):  # std::logic_error
    code = VXG_LOGIC_ERROR


class CudaError(VoxGpuError, RuntimeError):
    code = VXG_CUDA_ERROR


class DeviceOutOfMemory(VoxGpuError, MemoryError):
    code = VXG_OUT_OF_MEMORY


class IoError(VoxGpuError, OSError):  # the CLI's IoError (tools/voxline_cli.cpp:237-240)
    code = VXG_IO_ERROR


_EXC = {c.code: c for c in (InvalidArgument, RangeError, OutOfRange, LogicError, CudaError,
                            DeviceOutOfMemory, IoError)}


class vxg_segment(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("sx", "sy", "sz", "ex", "ey", "ez")]


class vxg_voxel(C.Structure):
    _fields_ = [("x", C.c_int32), ("y", C.c_int32), ("z", C.c_int32)]


class vxg_segment_plan(C.Structure):
    _fields_ = [("step_count", C.c_int64), ("wx", C.c_double), ("wy", C.c_double),
                ("wz", C.c_double), ("output_offset", C.c_int64)]


class vxg_timing(C.Structure):
    _fields_ = [("preprocess_ns", C.c_int64), ("kernel_ns", C.c_int64),
                ("assemble_ns", C.c_int64)]


_vp = C.c_void_p
_i64 = C.c_int64
_i64p = C.POINTER(C.c_int64)

# name -> (restype, argtypes); every symbol declared in include/voxgpu.h
SIGNATURES = {
    "vxg_abi_version": (C.c_int, []),
    "vxg_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "vxg_destroy": (None, [_vp]),
    "vxg_set_stream": (C.c_int, [_vp, _vp]),
    "vxg_get_stream": (_vp, [_vp]),
    "vxg_last_error": (C.c_char_p, [_vp]),
    "vxg_last_error_segment": (_i64, [_vp]),
    "vxg_launch_count": (_i64, [_vp]),
    "vxg_synchronize": (C.c_int, [_vp]),
    "vxg_host_alloc": (_vp, [C.c_size_t]),
    "vxg_host_free": (None, [_vp]),
    "vxg_round_points": (C.c_int, [_vp, _vp, _i64, _vp]),
    "vxg_segment_lengths": (C.c_int, [_vp, _vp, _i64, _vp]),
    "vxg_make_plans": (C.c_int, [_vp, _vp, _i64, _vp, _vp]),
    "vxg_voxelize_parametric": (C.c_int, [_vp, _vp, _vp, _i64, _i64p]),
    "vxg_voxelize_parametric_device": (C.c_int, [_vp, _vp, _vp, _i64, _i64p]),
    "vxg_voxelize_parametric_timing": (C.c_int, [_vp, C.POINTER(vxg_timing)]),
    "vxg_chain_length_bounds": (C.c_int, [_vp, _vp, _i64p, _i64p]),
    "vxg_batch_create": (C.c_int, [_vp, _vp, _i64, C.c_int, C.POINTER(_vp)]),
    "vxg_batch_set_slab": (C.c_int, [_vp, _i64, _i64]),
    "vxg_batch_from_plan": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, C.POINTER(_vp)]),
    "vxg_batch_destroy": (None, [_vp]),
    "vxg_batch_info": (C.c_int, [_vp, _i64p, _i64p, _i64p]),
    "vxg_batch_plans": (C.c_int, [_vp, _vp]),
    "vxg_batch_item_count": (C.c_int, [_vp, _i64p, _i64p]),
    "vxg_batch_work_item": (C.c_int, [_vp, _i64, _i64, _vp, C.POINTER(C.c_int)]),
    "vxg_batch_emit_list": (C.c_int, [_vp, _vp, _i64, _vp, _i64p, C.c_int]),
    "vxg_batch_count_voxels": (C.c_int, [_vp, _i64p]),
    "vxg_run_batch_device": (C.c_int, [_vp, _vp, _i64, _vp, _i64, _vp, _i64p]),
    "vxg_run_batch_device_result": (C.c_int, [_vp, _i64p, _i64p, _i64p]),
    "vxg_batch_emit_bitmap": (C.c_int, [_vp, _vp, _i64, _i64, _i64, C.c_int, _i64p, C.c_int]),
    "vxg_batch_slab_samples": (C.c_int, [_vp, _i64, _i64, _i64p]),
    "vxg_select_slab_segments": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64p]),
    "vxg_batch_timing": (C.c_int, [_vp, C.POINTER(vxg_timing)]),
    "vxg_run_batch": (C.c_int, [_vp, _vp, _i64, _vp, _i64, _vp, _i64p, C.POINTER(vxg_timing)]),
    "vxg_gen_segments": (C.c_int, [_vp, _i64, _vp, _vp, _i64, _i64, _i64, C.c_uint64, _vp,
                                   C.c_int]),
    "vxg_gen_arbitrary_batch": (C.c_int, [_vp, _i64, _i64, C.c_uint64, _vp]),
    "vxg_read_segments_csv": (C.c_int, [C.c_char_p, C.POINTER(_vp), _i64p, _i64p]),
    "vxg_free": (None, [_vp]),
    "vxg_write_chains": (C.c_int, [C.c_char_p, C.c_int, _vp, _vp, _i64]),
}

_lib = None
_lib_lock = threading.Lock()


def header_symbols(path: str = HEADER_PATH) -> list[str]:
    """Function names declared VXG_API in include/voxgpu.h."""
    text = open(path).read()
    return re.findall(r"VXG_API\s+[\w\s\*]+?\b(vxg_\w+)\s*\(", text)


def load():
    """Load libvoxgpu.so (raises if it was not built: there is no fallback)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libvoxgpu.so not found at {LIB_PATH}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (make -C "
                "paper_2009_09500_b200/csrc)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class Context:
    """One vxg_context: a device, a stream and a caching allocator. Not thread-safe; use one per
    thread (the reference's functions are re-entrant)."""

    def __init__(self, device: int | None = None):
        lib = load()
        if device is None:
            device = int(os.environ.get("VXG_DEVICE", "0"))
        h = _vp()
        st = lib.vxg_create(device, C.byref(h))
        if st != VXG_OK:
            raise CudaError(f"vxg_create(device={device}) failed with status {st}: no usable "
                            "CUDA device (libvoxgpu has no CPU fallback)")
        self.lib = lib
        self.h = h
        self.device = device

    def check(self, status: int):
        if status == VXG_OK:
            return
        msg = (self.lib.vxg_last_error(self.h) or b"").decode(errors="replace")
        seg = self.lib.vxg_last_error_segment(self.h)
        raise _EXC.get(status, VoxGpuError)(msg or f"libvoxgpu status {status}", seg)

    def set_stream(self, stream_handle: int | None):
        """Enqueue on a caller's cudaStream_t. None = the context's own stream; 0 (torch's
        handle for the legacy default stream) maps to cudaStreamLegacy."""
        if stream_handle == 0:
            stream_handle = 1  # cudaStreamLegacy
        self.check(self.lib.vxg_set_stream(self.h, stream_handle))

    def use_torch_stream(self):
        """Order device-pointer calls after work torch queued on its current stream."""
        import torch
        self.set_stream(torch.cuda.current_stream(self.device).cuda_stream)

    @property
    def launches(self) -> int:
        return self.lib.vxg_launch_count(self.h)

    def synchronize(self):
        self.check(self.lib.vxg_synchronize(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.vxg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default: dict[int, Context] = {}


def default_context() -> Context:
    tid = threading.get_ident()
    ctx = _default.get(tid)
    if ctx is None:
        ctx = Context()
        _default[tid] = ctx
    return ctx
