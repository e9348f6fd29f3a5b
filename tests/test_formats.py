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
    # bench (tools/voxline_cli.cpp:143-156, tests/test_cli.cpp:227-233): bad scenario -> 2
    r = run("bench", "--scenario", "nope")
    assert r.returncode == 2 and "unknown scenario" in r.stderr
    assert run("bench").returncode == 2                                    # --scenario required
    assert run("bench", "--scenario", "single", "--reps", "0").returncode == 2
    assert run("bench", "--scenario", "single", "--scale", "-1").returncode == 2
    assert run("bench", "--scenario", "single", "--warmup", "-1").returncode == 2


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


def _expected_bench(oracle, kind, scale, seed):
    """Parameter points and total voxels of the reference's run_scenario (src/bench.cpp:148-203,
    288-313) from the oracle: same sub-seeds, same generators, chain lengths from the oracle."""
    sc = lambda v: max(1, int(np.floor(v * scale + 0.5)))  # noqa: E731  (llround, v*scale > 0)
    sub = oracle.splitmix(seed, 4)
    if kind == "single":
        pts = [sc(1000), sc(10000), sc(100000), sc(1000000)]
        sets = [oracle.gen_segment_of_length(p, sub[i])[None] for i, p in enumerate(pts)]
    elif kind == "fixed-batch":
        pts = [sc(20), sc(200), sc(2000), sc(20000)]
        sets = [np.stack([oracle.gen_segment_of_length(p, s2) for s2 in oracle.splitmix(sub[i], 1024)])
                for i, p in enumerate(pts)]
    else:
        pts = [max(1024, sc(10000000))]
        sets = [oracle.gen_arbitrary_batch(pts[0], 1024, sub[0])]
    return pts, [int(oracle.chain_lengths(s).sum()) for s in sets]


@pytest.mark.gpu
@pytest.mark.parametrize("kind,scale", [("single", 0.01), ("fixed-batch", 0.05), ("arbitrary", 0.01)])
def test_cli_bench_reports(tmp_path, oracle, kind, scale):
    """`voxgpu bench`: the reference harness's scenarios (tests/test_cli.cpp:201-225 pins the
    table, the CSV header and the JSON sections), same parameter points and workloads -- every
    method's total_voxels equals the oracle's chain-length sum on the same generated segments."""
    import json
    csv, js = tmp_path / "r.csv", tmp_path / "r.json"
    r = subprocess.run([CLI, "bench", "--scenario", kind, "--scale", str(scale), "--reps", "2",
                        "--warmup", "1", "--seed", "7", "--workers", "3", "--report", str(csv),
                        "--report-json", str(js)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert r.stdout.splitlines()[0].split() == ["scenario", "parameter", "method", "workers",
                                                "group", "median_ms", "total_voxels", "MVps"]
    rows = csv.read_text().splitlines()
    assert rows[0] == "scenario,parameter,method,workers,group_size,median_ms,total_voxels,mvps"
    recs = [x.split(",") for x in rows[1:]]
    pts, totals = _expected_bench(oracle, kind, scale, 7)
    assert len(recs) == 3 * len(pts)
    for i, (p, t) in enumerate(zip(pts, totals)):
        trio = recs[3 * i: 3 * i + 3]
        assert [x[2] for x in trio] == ["sequential", "batch", "batch-device"]
        for x in trio:
            assert x[0] == kind and int(x[1]) == p and int(x[6]) == t, (x, p, t)
            assert float(x[5]) > 0 and abs(float(x[7]) - t / float(x[5]) / 1e3) <= 1e-6 * float(x[7])
        assert trio[0][3] == "1" and trio[1][3] == "3" and trio[1][4] == "64"
    ref_bench = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    if os.path.exists(ref_bench):  # the reference's own harness (src/bench.cpp) on the host
        rr = tmp_path / "ref.csv"
        q = subprocess.run([ref_bench, kind, "--scale", str(scale), "--reps", "1", "--warmup", "0",
                            "--seed", "7", "--workers", "3", "--report", str(rr)],
                           capture_output=True, text=True, timeout=600)
        assert q.returncode == 0, q.stderr
        theirs = [x.split(",") for x in rr.read_text().splitlines()[1:]]
        assert [(x[0], x[1], x[6]) for x in theirs] == \
            [(x[0], x[1], x[6]) for x in recs if x[2] != "batch-device"]
    doc = json.loads(js.read_text())
    assert doc["metadata"]["scenario"] == kind and doc["metadata"]["seed"] == 7
    assert ("length_distribution" in doc["metadata"]) == (kind == "arbitrary")
    assert [d["total_voxels"] for d in doc["records"]] == [int(x[6]) for x in recs]


@pytest.mark.gpu
def test_cli_bench_bad_report_path():
    r = subprocess.run([CLI, "bench", "--scenario", "single", "--scale", "0.001", "--reps", "1",
                        "--warmup", "0", "--report", "/nonexistent-dir/r.csv"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 3 and "cannot open report file" in r.stderr
