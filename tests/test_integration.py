"""The drop-in boundary: the reference's OWN pybind module (bindings/pybind_module.cpp) and
acceptance gate (tests/acceptance_main.cpp), compiled unchanged against
integration/voxline_gpu_core.cpp + libvoxgpu.so by integration/Makefile.

The checks mirror the reference's tests/python/test_smoke.py (same calls, same expected values
and exception classes), with the oracle as the parity checker. The built artefacts live in
integration/_build (made in the container that has /root/reference); without them the tests
skip, since the reference sources are needed to build them.
"""
import glob
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "integration", "_build")
MODULE = glob.glob(os.path.join(BUILD, "_voxline*.so"))
ACCEPT = os.path.join(BUILD, "acceptance")

needs_build = pytest.mark.skipif(not MODULE, reason="integration/_build not built "
                                 "(make -C integration needs /root/reference)")


def _mod():
    if BUILD not in sys.path:
        sys.path.insert(0, BUILD)
    import _voxline
    return _voxline


REF_API = ["BatchPlan", "batch_preprocess", "batch_voxelize", "candidate_voxels",
           "chain_length_bounds", "chains_equivalent", "compute_mvps", "effective_item_count",
           "gen_arbitrary_batch", "gen_segment_of_length", "kernel_work_item", "make_plan",
           "point_line_distance", "round_point", "run_batch", "segment_length",
           "voxelize_parametric", "voxelize_walk"]


@needs_build
def test_module_loads_and_exports_reference_api():
    m = _mod()
    for name in REF_API:  # python/voxline/__init__.py:8-48
        assert hasattr(m, name), name
    out = subprocess.run(["ldd", MODULE[0]], capture_output=True, text=True).stdout
    assert "libvoxgpu.so" in out and "not found" not in out


@needs_build
def test_no_cpu_fallback_without_gpu():
    """Without a device the hot path raises instead of computing on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    m = _mod()
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        m.make_plan((0.0, 0.0, 0.0), (5.0, 0.0, 0.0))
    with pytest.raises(RuntimeError):
        m.run_batch([((0.0, 0.0, 0.0), (5.0, 0.0, 0.0))])


# ----------------------------------------------------------------------------- on the GPU
@needs_build
@pytest.mark.gpu
def test_reference_smoke_through_gpu_core(oracle):
    """tests/python/test_smoke.py:26-117, through the reference module on the GPU core."""
    m = _mod()
    n, w = m.make_plan((0.0, 0.0, 0.0), (5.0, 0.0, 0.0))
    assert n == 5 and tuple(w) == (1.0, 0.0, 0.0)
    chain = m.voxelize_parametric((0.0, 0.0, 0.0), (3.0, 3.0, 3.0))
    assert chain == [(0, 0, 0), (1, 1, 1), (2, 2, 2), (3, 3, 3)]
    with pytest.raises(ValueError):
        m.round_point((3e9, 0.0, 0.0))
    chain = m.voxelize_parametric((0.1, 0.3, 0.7), (12.45, 4.9, 0.2))  # FMA-sensitive
    assert len(chain) == 14 and chain[12] == (11, 5, 0)
    plan = m.batch_preprocess([((0.0, 0.0, 0.0), (5.0, 0.0, 0.0)),
                               ((0.0, 0.0, 0.0), (3.0, 3.0, 3.0))])
    assert plan.step_counts == [5, 5] and plan.output_offsets == [0, 6]
    assert plan.max_steps == 5 and plan.total_voxel_capacity == 12 and len(plan) == 2
    plan = m.batch_preprocess([((0.0, 0.0, 0.0), (5.0, 0.0, 0.0)),
                               ((0.0, 0.0, 0.0), (2.0, 1.0, 0.0))])
    assert m.kernel_work_item(plan, 1, 2) == (2, 1, 0)
    assert m.kernel_work_item(plan, 1, 5) is None
    with pytest.raises(IndexError):
        m.kernel_work_item(plan, 2, 0)
    assert m.effective_item_count(plan) == (9, 3)
    res = m.batch_voxelize(plan, workers=4, group_size=1)
    assert res["chains"][1] == [(0, 0, 0), (1, 1, 0), (2, 1, 0)]
    assert res["timing"]["preprocess_ns"] == 0
    assert set(res["timing"]) == {"preprocess_ns", "kernel_ns", "assemble_ns"}
    with pytest.raises(ValueError):
        m.batch_preprocess([])
    with pytest.raises(ValueError):
        m.batch_voxelize(plan, workers=0)
    with pytest.raises(ValueError):  # range_error raised during preprocess
        m.run_batch([((0.0, 0.0, 0.0), (3e9, 0.0, 0.0))])


@needs_build
@pytest.mark.gpu
def test_reference_module_batch_matches_oracle(oracle):
    """run_batch through the reference module == oracle chains (bit-exact), and == the
    sequential voxelize_parametric map (tests/python/test_smoke.py:85-96)."""
    m = _mod()
    segs = m.gen_arbitrary_batch(200000, 512, 99)
    arr = np.asarray([list(s) + list(e) for s, e in segs], dtype=np.float64)
    res = m.run_batch(segs, workers=8, group_size=7)
    ovox, ooff, ototal = oracle.run_batch(arr)
    assert res["total_voxels"] == ototal
    flat = np.asarray([v for c in res["chains"] for v in c], dtype=np.int32).reshape(-1, 3)
    assert np.array_equal(flat, ovox)
    lens = np.asarray([len(c) for c in res["chains"]])
    assert np.array_equal(np.diff(ooff), lens)
    for i in range(0, 512, 61):
        assert m.voxelize_parametric(*segs[i]) == res["chains"][i]
    # generators: the reference's bench.cpp over the GPU make_plan == oracle generator
    s, e = m.gen_segment_of_length(1000, 5)
    np.testing.assert_array_equal(np.asarray(list(s) + list(e)),
                                  oracle.gen_segment_of_length(1000, 5))
    arr2 = np.asarray([list(s) + list(e) for s, e in m.gen_arbitrary_batch(10**6, 256, 3)])
    np.testing.assert_array_equal(arr2, oracle.gen_arbitrary_batch(10**6, 256, 3))


@needs_build
@pytest.mark.gpu
@pytest.mark.parametrize("criterion", [4, 5, 6])
def test_reference_acceptance_gate(criterion):
    """The reference's acceptance criteria that pin the batch path (c4 partition independence,
    c5 exact work-item accounting, c6 throughput arithmetic), run by its own binary."""
    r = subprocess.run([ACCEPT, str(criterion)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "[PASS]" in r.stdout, r.stdout + r.stderr
