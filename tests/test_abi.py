"""The C-ABI library loads and exports every symbol include/voxgpu.h declares (CPU only: no
compute calls), its value types are byte-compatible with the reference's, and the product fails
loudly (no CPU fallback) when no GPU is present."""
import ctypes as C
import os
import subprocess

import pytest

from paper_2009_09500_b200 import _lib

pytestmark = pytest.mark.filterwarnings("ignore")


def test_library_built():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build()"


def test_exports_every_header_symbol():
    declared = set(_lib.header_symbols())
    assert len(declared) >= 28
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert declared <= exported, declared - exported
    # nothing else leaks from the library's C++ internals
    assert {s for s in exported if s.startswith("vxg_")} == declared
    # the ctypes binding declares exactly the header's functions
    assert set(_lib.SIGNATURES) == declared
    lib = _lib.load()
    for name in declared:
        assert getattr(lib, name)


def test_value_type_layouts():
    # voxline::Segment 48 B, Voxel 12 B, SegmentPlan 40 B
    assert C.sizeof(_lib.vxg_segment) == 48
    assert C.sizeof(_lib.vxg_voxel) == 12
    assert C.sizeof(_lib.vxg_segment_plan) == 40
    assert _lib.vxg_segment_plan.output_offset.offset == 32
    assert C.sizeof(_lib.vxg_timing) == 24


def test_abi_version():
    assert _lib.load().vxg_abi_version() == 1


def test_sm100a_cubin_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    funcs = {}
    for chunk in sass.split("Function : ")[1:]:
        funcs[chunk.split()[0]] = chunk
    # every kernel that evaluates samples S + W*k must be free of fused multiply-adds (the
    # reference's FMA-free arithmetic); each must be present. (Kernels that also run make_plan
    # -- plan_kernel, single_chain_kernel -- contain the DFMAs of the correctly rounded
    # __ddiv_rn / __dsqrt_rn sequences, so they are not in this list.)
    hot = ["list_fused_kernel", "list_count_kernel", "list_emit_kernel", "tiles_fill_kernel",
           "emit_bitmap_kernel"]
    for k in hot:
        bodies = [body for name, body in funcs.items() if k in name]
        assert bodies, f"{k} missing from the library"
        for body in bodies:
            assert "DMUL" in body and "DADD" in body, k
            assert "DFMA" not in body, k
    # and the one-DADD rounding (round_pos, DADD.RM) is what the hot loops use
    assert "DADD.RM" in funcs[next(n for n in funcs if "tiles_fill_kernel" in n)]
    assert "DADD.RM" in funcs[next(n for n in funcs if "list_fused_kernel" in n)]


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2009_09500_b200 as vx
    with pytest.raises(vx.CudaError):
        vx.round_point((0.5, 0.5, 0.5))
    with pytest.raises(vx.CudaError):
        vx.run_batch([((0, 0, 0), (5, 0, 0))])
