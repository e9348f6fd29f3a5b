"""B200-native parametric 3D segment voxelization (arxiv 2009.09500 hot path).

Drop-in for the reference's ``voxline`` segment-generation API: ``import paper_2009_09500_b200
as voxline``. Every call goes through libvoxgpu.so (include/voxgpu.h) to hand-written sm_100a
CUDA kernels; there is no CPU fallback.
"""
from . import _lib
from ._lib import (CudaError, InvalidArgument, LogicError, OutOfRange, RangeError,
                   VoxGpuError, Context, default_context)
from .api import (Batch, BatchPlan, batch_preprocess, batch_voxelize, chain_length_bounds,
                  compute_mvps, effective_item_count, gen_arbitrary_batch, gen_segment_of_length,
                  gen_segments, kernel_work_item, make_plan, pinned_empty, round_point, run_batch,
                  run_batch_flat, run_batch_device, run_batch_device_result, segment_length,
                  voxelize_bitmap, voxelize_parametric, voxelize_parametric_device,
                  voxelize_parametric_host, voxelize_parametric_kernel_ns,
                  read_segments_csv, write_chains, batch_to_file)
from ._lib import IoError

__all__ = [
    "BatchPlan", "batch_preprocess", "batch_voxelize", "chain_length_bounds", "compute_mvps",
    "effective_item_count", "gen_arbitrary_batch", "gen_segment_of_length", "kernel_work_item",
    "make_plan", "round_point", "run_batch", "segment_length", "voxelize_parametric",
    "Batch", "run_batch_flat", "voxelize_bitmap", "gen_segments", "pinned_empty", "Context",
    "default_context", "VoxGpuError", "InvalidArgument", "RangeError", "OutOfRange", "LogicError",
    "CudaError", "IoError", "read_segments_csv", "write_chains", "batch_to_file",
    "run_batch_device", "run_batch_device_result", "voxelize_parametric_device",
    "voxelize_parametric_host", "voxelize_parametric_kernel_ns",
]


def library_path() -> str:
    return _lib.LIB_PATH
