"""Formats around the hot path: CSV segment ingest, VOX3 v2 / xyz
chain output and the `voxgpu` CLI, checked byte for byte against the reference's own
src/formats.cpp (oracle/_ref, compiled unmodified) and its CLI contract
(tools/voxline_cli.cpp: batch output, exit codes 0/2/3)."""
import os
import subprocess

import numpy as np
import pytest

import paper_2009_09500_b200 as vx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2009_09500_b200", "bin", "voxgpu")

GOOD = """# header comment
0,0,0,5,3,1

  1.5 , -2.25,3e1,0x1p3,+4,  -0.0
# another
-50.125,12,7.5,3.75,-8,100\r
1,2,3,4,5,6,
   \t
0.1,0.3,0.7,12.45,4.9,0.2"""

BAD = [
    "0,0,0,5,3\n",                    # five fields
    "0,0,0,5,3,1,2\n",                # seven
    "0,0,0,5,nan,1\n",                # not finite
    "0,0,0,5,inf,1\n",
    "0,0,0,1e400,3,1\n",              # overflow (std::stod: out_of_range)
    "0,0,0,1e-400,3,1\n",             # underflow (ERANGE)
    "0,0,0,5,3x,1\n",                 # trailing text
    "0,,0,5,3,1\n",                   # empty cell
    "1,2,3,4,5,6\n # indented comment\n",
    "1,2,3,4,5,6\n1,2,3,4,5,6\nabc\n",
]


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode())
    return str(p)


def test_csv_matches_reference(tmp_path, ref):
    path = _write(tmp_path, "good.csv", GOOD)
    ours = vx.read_segments_csv(path)
    theirs, err = ref.read_segments_csv(path)
    assert err is None
    assert ours.shape == theirs.shape == (5, 6)
    assert np.array_equal(ours.view(np.uint64), theirs.view(np.uint64))  # bit for bit (-0.0)


@pytest.mark.parametrize("text", BAD)
def test_csv_errors_match_reference(tmp_path, ref, text):
    path = _write(tmp_path, "bad.csv", text)
    _, err = ref.read_segments_csv(path)
    assert err is not None
    with pytest.raises(vx.InvalidArgument) as e:
        vx.read_segments_csv(path)
    assert str(e.value) == err  # same message, same (first) line number


def test_csv_large_parallel(tmp_path, ref, oracle):
    segs = oracle.gen_batch(20000, 0, 300, 1024, 9)
    lines = ["# big"] + [",".join(repr(float(v)) for v in s) for s in segs]
    lines.insert(7777, "")
    path = _write(tmp_path, "big.csv", "\n".join(lines) + "\n")
    ours = vx.read_segments_csv(path)
    theirs, _ = ref.read_segments_csv(path)
    assert np.array_equal(ours.view(np.uint64), theirs.view(np.uint64))
    assert np.array_equal(ours, segs)
    bad = lines.copy()
    bad[15000] = "1,2,3"
    path = _write(tmp_path, "bigbad.csv", "\n".join(bad))
    _, err = ref.read_segments_csv(path)
    with pytest.raises(vx.InvalidArgument) as e:
        vx.read_segments_csv(path)
    assert str(e.value) == err


def test_csv_missing_file():
    with pytest.raises(vx.IoError):
        vx.read_segments_csv("/nonexistent/segments.csv")


@pytest.mark.parametrize("fmt", ["vox3", "xyz"])
def test_writers_match_reference(tmp_path, ref, oracle, fmt):
    """write_chains over the oracle's chains == the reference's run_batch + writer, bytes."""
    segs = np.concatenate([oracle.gen_batch(300, 0, 200, 0, 5),
                           np.array([[0.5, 0.5, 0.5, -0.5, -0.5, -0.5],
                                     [3.2, 3.2, 3.2, 3.4, 3.1, 3.3]])])
    vox, off, _ = oracle.run_batch(segs)
    ours, theirs = tmp_path / f"ours.{fmt}", tmp_path / f"ref.{fmt}"
    vx.write_chains(str(ours), vox, off, fmt)
    ref.batch_write(segs, str(theirs), fmt)
    assert ours.read_bytes() == theirs.read_bytes()


def test_cli_usage_and_input_errors(tmp_path):
    assert os.path.exists(CLI), "paper_2009_09500_b200/bin/voxgpu not built"
    run = lambda *a: subprocess.run([CLI, *a], capture_output=True, text=True)  # noqa: E731
    assert run().returncode == 2
    assert run("bogus", "--out", "x").returncode == 2
    assert run("batch", "--out", "x").returncode == 2                     # no --input
    assert run("batch", "--input", "a", "--out", "b", "--workers", "0").returncode == 2
    r = run("batch", "--input", "/nonexistent.csv", "--out", str(tmp_path / "o"))
    assert r.returncode == 2 and "cannot read input file" in r.stderr
    bad = _write(tmp_path, "bad.csv", "1,2,3,4,5,6\n1,2\n")
    r = run("batch", "--input", bad, "--out", str(tmp_path / "o"))
    assert r.returncode == 2 and "line 2" in r.stderr
    empty = _write(tmp_path, "empty.csv", "# nothing\n\n")
    r = run("batch", "--input", empty, "--out", str(tmp_path / "o"))
    assert r.returncode == 2 and "no segments" in r.stderr


def test_cli_no_gpu_fails_loudly(tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    path = _write(tmp_path, "s.csv", "0,0,0,5,3,1\n")
    r = subprocess.run([CLI, "batch", "--input", path, "--out", str(tmp_path / "o")],
                       capture_output=True, text=True)
    assert r.returncode == 3 and "no CPU fallback" in r.stderr


# ------------------------------------------------------------------------------ on the GPU
@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["vox3", "xyz"])
def test_cli_batch_matches_reference(tmp_path, ref, oracle, fmt):
    """`voxgpu batch` == the reference CLI's batch output (tests/test_cli.cpp:153-175 pins it
    byte-identical across worker counts; here across implementations)."""
    segs = np.concatenate([oracle.gen_batch(2000, 0, 500, 1024, 11),
                           oracle.gen_batch(500, 0, 40, 0, 12)])
    lines = [",".join(repr(float(v)) for v in s) for s in segs]
    csv = _write(tmp_path, "in.csv", "\n".join(lines) + "\n")
    out = tmp_path / f"gpu.{fmt}"
    r = subprocess.run([CLI, "batch", "--input", csv, "--out", str(out), "--format", fmt,
                        "--workers", "8", "--group-size", "3"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert r.stderr.startswith(f"batch: {len(segs)} segments, ")
    theirs = tmp_path / f"ref.{fmt}"
    ref.batch_write(vx.read_segments_csv(csv), str(theirs), fmt)
    assert out.read_bytes() == theirs.read_bytes()
    # the Python entry point writes the same file
    again = tmp_path / f"py.{fmt}"
    vx.batch_to_file(vx.read_segments_csv(csv), str(again), fmt)
    assert again.read_bytes() == theirs.read_bytes()


@pytest.mark.gpu
def test_cli_voxelize(tmp_path, oracle):
    out = tmp_path / "one.vox3"
    r = subprocess.run([CLI, "voxelize", "--start", "0.1,0.3,0.7", "--end", "12.45,4.9,0.2",
                        "--out", str(out), "--format", "vox3"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    data = out.read_bytes()
    assert data[:8] == b"VOX3\x01\x00\x00\x00"
    n = int.from_bytes(data[8:16], "little")
    chain = np.frombuffer(data[16:], dtype=np.int32).reshape(n, 3)
    assert np.array_equal(chain, oracle.voxelize_parametric([0.1, 0.3, 0.7, 12.45, 4.9, 0.2]))
    assert n == 14 and tuple(chain[12]) == (11, 5, 0)
