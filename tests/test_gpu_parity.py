"""Parity of the B200 path (through the C ABI) with the oracle and the reference's golden vectors.

Bar: bit-exact voxel lists, chain offsets, plans (W compared as raw doubles), bitmaps and error
classes. Small/medium corpora are compared element for element; full BASELINE sizes through
size-independent properties and per-chain hashes (tests/gpu_checks.py).
"""
import threading

import numpy as np
import pytest

from tests.golden.make_golden import decimal_grid_corpus, digest, mixed_batch, seg_digest
from tests.test_oracle_golden import _corpus

pytestmark = pytest.mark.gpu


# ------------------------------------------------------------------ golden vectors
def test_golden_plans_chains_bounds(vx, golden):
    for name, case in golden["plans"].items():
        s = case["segment"]
        n, w = vx.make_plan(s[:3], s[3:])
        assert n == case["n"], name
        assert w == [float.fromhex(h) for h in case["w_hex"]], name
        assert [list(v) for v in vx.voxelize_parametric(s[:3], s[3:])] == case["chain"], name
        assert list(vx.chain_length_bounds(s[:3], s[3:])) == case["bounds"], name


def test_golden_rounding(vx, golden):
    for case in golden["round_ok"]:
        assert list(vx.round_point(case["p"])) == case["v"]
    for case in golden["round_bad"]:
        with pytest.raises(ValueError):
            vx.round_point([float(x) for x in case["p"]])
        with pytest.raises(vx.RangeError):
            vx.round_point([float(x) for x in case["p"]])


def test_fma_sensitive_vector(vx):
    # under FMA the k=12 sample rounds to (12,5,0) and the chain has 13 voxels
    chain = vx.voxelize_parametric((0.1, 0.3, 0.7), (12.45, 4.9, 0.2))
    assert len(chain) == 14 and chain[12] == (11, 5, 0)


def test_golden_batch(vx, golden):
    plan = vx.batch_preprocess([((0, 0, 0), (5, 0, 0)), ((0, 0, 0), (3, 3, 3))])
    g = golden["batch_two"]
    assert plan.step_counts == g["steps"] and plan.output_offsets == g["offsets"]
    assert plan.max_steps == g["max_steps"] and plan.total_voxel_capacity == g["capacity"] == 12
    segs = [((0, 0, 0), (5, 0, 0)), ((0, 0, 0), (2, 1, 0))]
    plan = vx.batch_preprocess(segs)
    g = golden["batch_short"]
    assert vx.kernel_work_item(plan, 1, 2) == tuple(g["item_1_2"]) == (2, 1, 0)
    assert vx.kernel_work_item(plan, 0, 0) == tuple(g["item_0_0"])
    assert vx.kernel_work_item(plan, 1, 5) is None
    assert vx.effective_item_count(plan) == (g["live"], g["redundant"]) == (9, 3)
    for i, k in [(2, 0), (-1, 0), (0, 6), (0, -1)]:
        with pytest.raises(IndexError):
            vx.kernel_work_item(plan, i, k)
    res = vx.batch_voxelize(plan, workers=1, group_size=64)
    assert [[list(v) for v in c] for c in res["chains"]] == g["chains"]
    assert res["total_voxels"] == g["total"]
    assert res["timing"]["preprocess_ns"] == 0


def test_golden_generators(vx, golden):
    for key, hexes in golden["gen_segment_of_length"].items():
        target, seed = map(int, key.split("_"))
        s, e = vx.gen_segment_of_length(target, seed)
        assert list(s) + list(e) == [float.fromhex(h) for h in hexes], key
    arb = np.asarray([list(s) + list(e) for s, e in vx.gen_arbitrary_batch(10000000, 1024, 7)])
    assert seg_digest(arb) == golden["gen_arbitrary_10M_1024_7"]["digest"]


def test_acceptance_c4_c5(vx, golden):
    c = golden["acceptance_c4c5"]
    segs = vx.gen_arbitrary_batch(500000, 1024, c["seed"])
    arr = np.asarray([list(s) + list(e) for s, e in segs])
    assert seg_digest(arr) == c["digest_segments"]
    plan = vx.batch_preprocess(segs)
    live, red = vx.effective_item_count(plan)
    assert (live, red) == (c["live"], c["redundant"])
    assert live + red == c["grid"]
    vox, off, total = vx.run_batch_flat(arr)
    assert total == c["total_voxels"] and digest(vox, off) == c["digest_chains"]
    # criterion 4: output independent of the (host) partitioning knobs
    seq = [vx.voxelize_parametric(s, e) for s, e in segs[:64]]
    for workers, group in [(1, 1), (8, 256)]:
        res = vx.batch_voxelize(plan, workers, group)
        assert res["chains"][:64] == seq


def test_golden_corpora(vx, oracle, golden):
    for name, spec in golden["corpora"].items():
        segs = _corpus(name, spec, oracle)
        vox, off, total = vx.run_batch_flat(segs)
        assert total == spec["total_voxels"], name
        assert digest(vox, off) == spec["digest"], name


def test_gpu_generator_matches_oracle(vx, oracle):
    for kw in [dict(n=5000, len_fixed=128, V=512, seed=3), dict(n=5000, len_fixed=64, V=1024, seed=4),
               dict(n=5000, len_max=2048, V=4096, seed=5), dict(n=3000, len_fixed=77, V=0, seed=6),
               dict(n=3000, len_max=300, V=0, seed=7)]:
        g = vx.gen_segments(kw["n"], kw.get("len_fixed", 0), kw.get("len_max", 0), kw["V"],
                            kw["seed"])
        o = oracle.gen_batch(kw["n"], kw.get("len_fixed", 0), kw.get("len_max", 0), kw["V"],
                             kw["seed"])
        assert np.array_equal(g.view(np.uint64), o.view(np.uint64)), kw


# ------------------------------------------------------------------ seeded corpora vs oracle
def _compare(vx, oracle, segs):
    vox, off, total = vx.run_batch_flat(segs)
    ovox, ooff, ototal = oracle.run_batch(segs)
    assert total == ototal
    assert np.array_equal(off, ooff)
    assert np.array_equal(vox, ovox)
    return total


@pytest.mark.parametrize("scale", [1.0, 37.5, 1e3, 1e6, 1e9])
def test_random_uniform(vx, oracle, scale):
    rng = np.random.default_rng(int(scale) % 1000 + 11)
    n = 20000 if scale < 1e3 else 200
    segs = rng.uniform(-scale, scale, size=(n, 6))
    if scale >= 1e3:  # keep the capacity modest: short segments far from the origin
        segs[:, 3:] = segs[:, :3] + rng.uniform(-300, 300, size=(n, 3))
    _compare(vx, oracle, segs)


def test_ties_and_grids(vx, oracle):
    rng = np.random.default_rng(3)
    for q in (2, 4, 10, 20):
        segs = np.round(rng.uniform(-60, 60, size=(20000, 6)) * q) / q
        _compare(vx, oracle, segs)
    segs = np.asarray(decimal_grid_corpus(30000, 1234))
    _compare(vx, oracle, segs)


def test_reference_corpora(vx, oracle):
    for count, seed, every, mx in [(300, 402, 3, 500.0), (1500, 203, 5, 1e4), (64, 404, 3, 500.0)]:
        _compare(vx, oracle, np.asarray(mixed_batch(count, seed, every, mx)))


def test_zero_and_one_sample_segments(vx, oracle):
    rng = np.random.default_rng(9)
    base = rng.uniform(10, 20, size=(50000, 3))
    segs = np.concatenate([base, base + rng.uniform(-0.3, 0.3, size=(50000, 3))], axis=1)
    # thousands of N = 0 segments per 4096-sample tile (m close to the tile size)
    _compare(vx, oracle, segs)
    segs[::7, 3:] += 1.0
    _compare(vx, oracle, segs)


def test_tile_boundaries(vx, oracle):
    # segment starts landing exactly on and around 2048/4096-sample tile boundaries
    for L in (4095, 4096, 4097, 2047, 2048, 1, 2, 31, 32, 33):
        segs = oracle.gen_batch(64, L, 0, 0 if L > 1000 else 0, 100 + L)
        _compare(vx, oracle, segs)


def test_single_long_segments(vx, oracle):
    # config 2: one segment swept 1 .. 10^6 voxels
    for L in (1, 10, 100, 1000, 10_000, 100_000, 1_000_000):
        s = oracle.gen_segment_of_length(L, 2024 + L)
        got = np.asarray(vx.voxelize_parametric(s[:3], s[3:]), dtype=np.int32)
        assert np.array_equal(got, oracle.voxelize_parametric(s)), L


def test_long_chain_kernel_device_api(vx, oracle, monkeypatch):
    """voxelize_parametric of chains longer than the one-CTA path (long_chain_kernel: 2048-sample
    CTAs joined by a decoupled look-back), through the device-output entry point and the host
    one, against the oracle: lengths straddling the CTA size, ties, negative and descending
    segments, the int32 edge (checked rounding), the cap contract and the range errors."""
    import torch
    cases = [oracle.gen_segment_of_length(L, 91 + L) for L in (1, 2047, 2048, 2049, 4097, 16385,
                                                               100_000, 1_000_000, 3_000_000)]
    cases += [np.array(c, dtype=np.float64) for c in (
        [0.5, 0.5, 0.5, 40000.5, 20000.5, -10000.5],           # ties on every axis
        [-70000.25, 300.5, -2.5, 10.5, -5000.5, 9000.75],        # negative, descending
        [2147000000.0, 5.0, -3.0, 2147483647.4, 9.0, 2.0],      # checked rounding at the edge
        [12.0, 12.0, 12.0, 12.0, 12.0, 50000.0])]               # axis-parallel
    for s in cases:
        want = oracle.voxelize_parametric(s)
        out = torch.zeros((len(want) + 7, 3), dtype=torch.int32, device="cuda")
        n = vx.voxelize_parametric_device(s, out.data_ptr(), out.shape[0])
        assert n == len(want), s
        assert np.array_equal(out[:n].cpu().numpy(), want), s
        got = np.asarray(vx.voxelize_parametric(s[:3], s[3:]), dtype=np.int32).reshape(-1, 3)
        assert np.array_equal(got, want), s
    s = cases[7]  # 10^6 voxels: a short buffer raises, nothing past cap is written
    out = torch.full((1000, 3), -1, dtype=torch.int32, device="cuda")
    with pytest.raises(vx.LogicError):
        vx.voxelize_parametric_device(s, out.data_ptr(), 999)
    assert (out[999] == -1).all()
    with pytest.raises(vx.RangeError):
        vx.voxelize_parametric_device([0.0, np.nan, 0.0, 1.0, 2.0, 3.0], out.data_ptr(), 1000)
    with pytest.raises(vx.RangeError):
        vx.voxelize_parametric_device([0.0, 0.0, 0.0, 3e9, 2.0, 3.0], out.data_ptr(), 1000)
    with pytest.raises(vx.RangeError):  # the samples leave the int32 lattice
        vx.voxelize_parametric_device([2147483000.0, 0.0, 0.0, 2147483647.6, 1.0, 0.0],
                                      out.data_ptr(), 1000)


def test_single_chain_kernel_matches_batch_path(vx, oracle, monkeypatch):
    """voxelize_parametric's one-launch path (single_chain_kernel: plan + samples + dedup in one
    CTA, chain into mapped pinned memory) == the batch path (VXG_NO_SINGLE) == the oracle, on the
    edge cases of both routes: lengths straddling the 2^14-sample dispatch bound, ties, negative
    coordinates, zero-length segments, the int32 edge (checked rounding), and the error / cap
    contract (range error for non-finite endpoints, LOGIC_ERROR + the true count when cap is
    short)."""
    import ctypes as C
    cases = [oracle.gen_segment_of_length(L, 77 + L) for L in (1, 2, 31, 32, 33, 1023, 1024, 1025,
                                                               16370, 16378, 16383, 16384, 16390)]
    cases += [np.array(c, dtype=np.float64) for c in (
        [0.5, 0.5, 0.5, -0.5, -0.5, -0.5], [0.1, 0.3, 0.7, 12.45, 4.9, 0.2],
        [3.2, 3.2, 3.2, 3.4, 3.1, 2.9], [-7.5, 2.5, -0.5, 9.5, -3.5, 0.5],
        [2147483640.0, 0.0, 0.0, 2147483647.4, 0.0, 0.0],
        [-2147483647.4, -5.0, 1.0, -2147483600.2, 6.0, -1.0])]
    rng = np.random.default_rng(5)
    cases += list(rng.uniform(-300, 300, size=(40, 6)))
    for s in cases:
        want = oracle.voxelize_parametric(s)
        monkeypatch.delenv("VXG_NO_SINGLE", raising=False)
        got = np.asarray(vx.voxelize_parametric(s[:3], s[3:]), dtype=np.int32).reshape(-1, 3)
        monkeypatch.setenv("VXG_NO_SINGLE", "1")
        got_b = np.asarray(vx.voxelize_parametric(s[:3], s[3:]), dtype=np.int32).reshape(-1, 3)
        assert np.array_equal(got, want), s
        assert np.array_equal(got_b, want), s
    monkeypatch.delenv("VXG_NO_SINGLE", raising=False)
    with pytest.raises(vx.RangeError):
        vx.voxelize_parametric((0.0, np.nan, 0.0), (1.0, 2.0, 3.0))
    with pytest.raises(vx.RangeError):
        vx.voxelize_parametric((0.0, 0.0, 0.0), (3e9, 2.0, 3.0))
    ctx = vx.default_context()
    seg = np.array([0.0, 0.0, 0.0, 100.0, 3.0, 1.0])
    out = np.zeros((10, 3), np.int32)
    cnt = C.c_int64()
    st = ctx.lib.vxg_voxelize_parametric(ctx.h, seg.ctypes.data, out.ctypes.data, 10, C.byref(cnt))
    assert st == vx._lib.VXG_LOGIC_ERROR and cnt.value == 101
    assert np.array_equal(out, oracle.voxelize_parametric(seg)[:10])


def test_config_scaled_lists(vx, oracle):
    for kw in [dict(n=65536, len_fixed=128, V=512, seed=0x5EED0101),
               dict(n=20000, len_max=2048, V=4096, seed=0x5EED0104)]:
        segs = vx.gen_segments(kw["n"], kw.get("len_fixed", 0), kw.get("len_max", 0), kw["V"],
                               kw["seed"])
        _compare(vx, oracle, segs)


# ------------------------------------------------------------------ errors
def test_error_semantics(vx):
    with pytest.raises(ValueError):
        vx.batch_preprocess([])
    with pytest.raises(vx.InvalidArgument):
        vx.run_batch([])
    # tests/test_batch.cpp:175-181: overflow surfaces as range_error (from preprocess)
    with pytest.raises(vx.RangeError):
        vx.run_batch([((0, 0, 0), (5, 0, 0)), ((0, 0, 0), (3e9, 0, 0))], workers=2, group_size=1)
    segs = [((0, 0, 0), (5, 0, 0)), ((0, float("nan"), 0), (1, 1, 1)), ((1, 1, 1), (2, 2, 2)),
            ((0, 0, 0), (float("inf"), 0, 0))]
    with pytest.raises(vx.RangeError) as e:
        vx.run_batch(segs)
    assert e.value.segment == 1  # lowest failing segment, as the reference's serial loop
    plan = vx.batch_preprocess([((0, 0, 0), (5, 0, 0))])
    with pytest.raises(ValueError):
        vx.batch_voxelize(plan, workers=0)
    with pytest.raises(ValueError):
        vx.batch_voxelize(plan, group_size=0)
    with pytest.raises(ValueError):
        vx.compute_mvps(10, 0.0)
    with pytest.raises(ValueError):
        vx.gen_arbitrary_batch(5, 10, 1)


def test_int32_edges(vx, oracle):
    segs = np.array([[2147483640.0, 0, 0, 2147483647.4, 0, 0],
                     [-2147483640.0, 5, 5, -2147483648.4, 9, -3],
                     [2147483000.5, -2147483000.5, 1, 2147483100.25, -2147483100.75, 7]])
    _compare(vx, oracle, segs)
    with pytest.raises(vx.RangeError):
        vx.run_batch_flat(np.array([[2147483640.0, 0, 0, 2147483647.5, 0, 0]]))


def test_concurrent_contexts(vx, oracle):
    segs = [oracle.gen_batch(3000, 0, 400, 1024, 50 + t) for t in range(4)]
    expect = [oracle.run_batch(s) for s in segs]
    errors = []

    def work(t):
        try:
            for _ in range(3):
                vox, off, total = vx.run_batch_flat(segs[t])  # per-thread default context
                assert total == expect[t][2] and np.array_equal(vox, expect[t][0])
        except Exception as e:  # pragma: no cover
            errors.append(e)

    ths = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    [t.start() for t in ths]
    [t.join() for t in ths]
    assert not errors, errors


# ------------------------------------------------------------------ bitmaps
def test_bitmap_vs_oracle(vx, oracle):
    segs = vx.gen_segments(20000, 64, 0, 256, 77)
    words, outside = vx.voxelize_bitmap(segs, 256, clip=False)
    ow, oo = oracle.bitmap(segs, 256)
    assert outside == oo == 0
    assert np.array_equal(words, ow)
    # z-slab partition (1, 2, 4, 8 slabs) with device clipping == the full bitmap
    for G in (1, 2, 4, 8):
        h = 256 // G
        parts = [vx.voxelize_bitmap(segs, 256, g * h, (g + 1) * h, clip=True)[0] for g in range(G)]
        assert np.array_equal(np.concatenate(parts), ow), G


def test_bitmap_outside_and_negative(vx, oracle):
    rng = np.random.default_rng(12)
    segs = rng.uniform(-40, 160, size=(5000, 6))
    for z0, z1, clip in [(0, 128, False), (17, 93, True), (0, 128, True)]:
        words, outside = vx.voxelize_bitmap(segs, 128, z0, z1, clip=clip)
        ow, oo = oracle.bitmap(segs, 128, z0, z1)
        assert np.array_equal(words, ow), (z0, z1, clip)
        if not clip:
            assert outside == oo


def test_bitmap_clip_adversarial(vx, oracle):
    # nearly-flat z, exact ties on slab boundaries, descending z
    rng = np.random.default_rng(4)
    segs = np.round(rng.uniform(0, 63, size=(20000, 6)) * 2) / 2
    segs[::3, 5] = segs[::3, 2] + 1e-13
    for z0, z1 in [(0, 32), (32, 64), (10, 11), (31, 33)]:
        words, _ = vx.voxelize_bitmap(segs, 64, z0, z1, clip=True)
        ow, _ = oracle.bitmap(segs, 64, z0, z1)
        assert np.array_equal(words, ow), (z0, z1)


def test_bitmap_tiles_adversarial(vx, oracle):
    """The tile-binned path (V % 128 == 0): half-integer endpoints (ties on every tile and slab
    boundary), nearly-flat axes, descending directions, segments leaving the volume, partial
    x/y/z tiles (V = 384, 640) and slabs that cut tiles; bit-exact against the oracle."""
    rng = np.random.default_rng(41)
    for V in (128, 384, 640):
        segs = np.round(rng.uniform(-20, V + 20, size=(8000, 6)) * 2) / 2
        segs[::4, 5] = segs[::4, 2] + 1e-13          # flat z
        segs[1::4, 3] = segs[1::4, 0] - 1e-12         # flat x, descending
        long_ = rng.uniform(0, V - 1, size=(500, 6))  # long segments across many tiles
        segs = np.concatenate([segs, long_])
        words, outside = vx.voxelize_bitmap(segs, V, clip=False)
        ow, oo = oracle.bitmap(segs, V)
        assert np.array_equal(words, ow), V
        assert outside == oo, V
        for z0, z1 in [(0, 70), (69, min(141, V)), (V // 3, V // 3 + 1), (V - 71, V)]:
            words, _ = vx.voxelize_bitmap(segs, V, z0, z1, clip=True)
            ow, _ = oracle.bitmap(segs, V, z0, z1)
            assert np.array_equal(words, ow), (V, z0, z1)


@pytest.mark.parametrize("order", ["copy", "index", "none"])
def test_bitmap_walk_orders(vx, oracle, monkeypatch, order):
    """The count/scatter walk orders of large batches with long segments (n >= 2^16, N >= 256):
    records copied into walk order (N carried in the copy's flag word), the index permutation,
    and no sort; on the whole volume, a thin selected slab (sorted on request) and a slab cut
    mid-tile -- bit-exact against the oracle every time."""
    if order == "index":
        monkeypatch.setenv("VXG_BITMAP_PERM_INDEX", "1")
    elif order == "none":
        monkeypatch.setenv("VXG_BITMAP_NO_PERM", "1")
    monkeypatch.setenv("VXG_BITMAP_PERM", "1")  # (thin slabs sorted too)
    segs = vx.gen_segments(70000, 0, 600, 1024, 23)
    for z0, z1 in [(0, 1024), (400, 460), (7, 131)]:
        words, outside = vx.voxelize_bitmap(segs, 1024, z0, z1, clip=True)
        ow, oo = oracle.bitmap(segs, 1024, z0, z1)
        assert np.array_equal(words, ow), (order, z0, z1)
        if (z0, z1) == (0, 1024):
            assert outside == oo, order


def test_bitmap_tiles_accumulate_and_match_atomic_path(vx, oracle, monkeypatch):
    """Words are OR-ed into (the caller's bits survive), and the tile path equals the generic
    global-atomic path on the same batch."""
    segs = vx.gen_segments(3000, 0, 300, 512, 17)
    b = vx.Batch(segs)
    prior = np.zeros(512 ** 3 // 64, np.uint64)
    prior[::97] = np.uint64(0x8000000000000001)
    w_tiles, _ = b.emit_bitmap(512, 0, 512, words=prior.copy())
    monkeypatch.setenv("VXG_BITMAP_ATOMIC", "1")
    w_atomic, _ = b.emit_bitmap(512, 0, 512, words=prior.copy())
    b.close()
    ow, _ = oracle.bitmap(segs, 512)
    assert np.array_equal(w_tiles, ow | prior)
    assert np.array_equal(w_atomic, w_tiles)


@pytest.mark.parametrize("V,slab", [(512, (0, 512)), (1024, (100, 700)), (1024, (900, 1000)),
                                     (384, (0, 384)), (384, (119, 241)), (640, (7, 8))])
def test_bitmap_streamed_readback(vx, oracle, monkeypatch, V, slab):
    """Host bitmaps (>= 64 MiB by default) through the tile path are read back layer by layer while the
    fill runs (mapped per-layer tile counters, copy stream): same words and outside count as the
    plain readback (VXG_BITMAP_NO_STREAM), overwriting or OR-ing into the caller's words, and an
    empty slab still returns the caller's words."""
    z0, z1 = slab
    monkeypatch.setenv("VXG_BITMAP_STREAM_MIN", "0")  # stream every size here
    segs = np.concatenate([vx.gen_segments(4000, 0, min(500, V // 2), V, 71),
                           oracle.gen_batch(300, 0, 200, 0, 72)])
    b = vx.Batch(segs)
    want, _ = oracle.bitmap(segs, V, z0, z1)
    monkeypatch.setenv("VXG_BITMAP_NO_STREAM", "1")
    plain, out_p = b.emit_bitmap(V, z0, z1)
    monkeypatch.delenv("VXG_BITMAP_NO_STREAM")
    streamed, out_s = b.emit_bitmap(V, z0, z1)
    assert np.array_equal(plain, want) and np.array_equal(streamed, want)
    assert out_s == out_p
    prior = np.zeros_like(want)
    prior[::11] = np.uint64(3)
    got, _ = b.emit_bitmap(V, z0, z1, words=prior.copy(), overwrite=False)
    assert np.array_equal(got, want | prior)
    b.close()
    far = vx.Batch(np.array([[5000.0, 5000, 5000, 5010, 5003, 5001]]))  # no sample in the volume
    got, outside = far.emit_bitmap(V, z0, z1, words=prior.copy(), overwrite=False)
    assert np.array_equal(got, prior) and outside == 11
    far.close()


def test_bitmap_fill_fixed_point_vs_exact(vx, oracle, monkeypatch):
    """The fill's 32.32 fixed-point stepping (REC_FX records) against its exact-FP64 form
    (VXG_FILL_PF bit 3) and the oracle: random long segments, tie lines (samples exactly on and
    a few ulp beside half-integers: the near-boundary redo), the quarter grid, and segments that
    start far outside the volume (|S| >= 2^24: no REC_FX, exact path) crossing it."""
    rng = np.random.default_rng(2024)
    V = 512
    far = np.empty((4, 6))
    far[:, 0] = -rng.uniform(2 ** 24, 2 ** 24 + 1000, 4)  # S.x far to the left
    far[:, 1:3] = rng.uniform(10, V - 10, (4, 2))
    far[:, 3:6] = rng.uniform(10, V - 10, (4, 3))
    ties = _tie_lines(6000, 5, [0, 1, -1, 2, -2], hi=100)
    segs = np.concatenate([vx.gen_segments(20000, 0, 400, V, 91), ties,
                           np.abs(_quarter_grid(20000, 3)) * 3, far])
    want, oo = oracle.bitmap(segs, V)
    b = vx.Batch(segs)
    got, out = b.emit_bitmap(V)
    monkeypatch.setenv("VXG_FILL_PF", "9")  # L1 prefetch + exact FP64 fill
    exact, out_e = b.emit_bitmap(V)
    b.close()
    assert np.array_equal(got, want)
    assert np.array_equal(exact, want)
    assert out == out_e == oo


@pytest.mark.parametrize("stream", [False, True])
def test_bitmap_splits_slab_when_pieces_overflow(vx, oracle, monkeypatch, stream):
    """More pieces than the bin cursors count (2^32; here a test bound of 2000) or than the device
    holds: the tile path does the slab as two thinner slabs, recursively, instead of failing --
    same words and outside count as the oracle, for the device readback and the streamed one."""
    if stream:
        monkeypatch.setenv("VXG_BITMAP_STREAM_MIN", "0")
    segs = np.concatenate([vx.gen_segments(2000, 0, 300, 512, 33),
                           oracle.gen_batch(200, 0, 100, 0, 34) * 4.0 - 30.0])
    b = vx.Batch(segs)
    for z0, z1 in [(0, 512), (37, 401)]:
        monkeypatch.delenv("VXG_BITMAP_MAX_PIECES", raising=False)
        _, out_whole = b.emit_bitmap(512, z0, z1)
        monkeypatch.setenv("VXG_BITMAP_MAX_PIECES", "2000")
        got, out = b.emit_bitmap(512, z0, z1)
        want, _ = oracle.bitmap(segs, 512, z0, z1)
        assert np.array_equal(got, want), (z0, z1)
        assert out == out_whole
    b.close()


def test_select_slab_segments(vx, oracle):
    """The z-slab partitioner's device filter (vxg_select_slab_segments): a rank's slab of the
    bitmap from its filtered segments equals that slab of the full batch's bitmap (and the slab's
    sample count); segments with non-finite endpoints are kept for the plan to report."""
    import torch
    from paper_2009_09500_b200.shard import select_slab_segments
    V = 1024
    segs = np.concatenate([vx.gen_segments(20000, 0, 400, V, 91),
                           oracle.gen_batch(2000, 0, 300, 0, 92) * 3.0 - 200.0])
    d = torch.from_numpy(segs).cuda()
    local = torch.empty_like(d)
    ctx = vx.default_context()
    full = vx.Batch(None, device_ptr=d.data_ptr(), n=d.shape[0])
    for z0, z1 in [(0, 100), (300, 700), (1000, 1024), (512, 513)]:
        k = select_slab_segments(ctx, d.data_ptr(), d.shape[0], z0, z1, local.data_ptr())
        assert 0 < k < d.shape[0]
        nw = V * V * (z1 - z0) // 64
        w_full = torch.zeros(nw, dtype=torch.int64, device="cuda")
        w_sel = torch.zeros(nw, dtype=torch.int64, device="cuda")
        full.emit_bitmap_device(w_full.data_ptr(), V, z0, z1, True)
        part = vx.Batch(None, device_ptr=local.data_ptr(), n=k)
        part.emit_bitmap_device(w_sel.data_ptr(), V, z0, z1, True)
        assert torch.equal(w_full, w_sel), (z0, z1)
        w_sel.zero_()  # stated as filtered (vxg_batch_set_slab): the tile path's filter skipped
        part.set_slab(z0, z1).emit_bitmap_device(w_sel.data_ptr(), V, z0, z1, True)
        assert torch.equal(w_full, w_sel), (z0, z1)
        assert part.slab_samples(z0, z1) == full.slab_samples(z0, z1)
        part.close()
    full.close()
    bad = torch.from_numpy(np.array([[0.0, 0.0, np.nan, 1, 1, 1], [0, 0, 0, 1, 1, 1.0]])).cuda()
    out = torch.empty_like(bad)
    assert select_slab_segments(ctx, bad.data_ptr(), 2, 500, 600, out.data_ptr()) == 1


def test_sample_balanced_slabs_on_device(vx):
    """The bench's z-slab partition from Batch.slab_samples: the slabs tile [0, V), their sample
    counts add up to the whole volume's, and each is within a few percent of the mean."""
    from paper_2009_09500_b200.shard import sample_balanced_slabs
    V = 1024
    b = vx.Batch(vx.gen_segments(200000, 0, 600, V, 93))
    total = b.slab_samples(0, V)
    for world in (2, 3, 8):
        slabs = sample_balanced_slabs(b.slab_samples, V, world)
        assert slabs[0][0] == 0 and slabs[-1][1] == V
        work = [b.slab_samples(z0, z1) for z0, z1 in slabs]
        assert sum(work) == total
        assert max(work) / (total / world) < 1.05, (world, work)
    b.close()


def test_bitmap_overwrite_discards_prior_words(vx, oracle):
    """VXG_BITMAP_OVERWRITE replaces the caller's words: garbage in the buffer (host or device)
    does not survive, on the tile path and on a slab."""
    import torch
    segs = vx.gen_segments(2000, 0, 300, 512, 23)
    b = vx.Batch(segs)
    junk = np.full(512 ** 3 // 64, np.uint64(0xFFFF0000FFFF0000), np.uint64)
    w_host, _ = b.emit_bitmap(512, 0, 512, words=junk, overwrite=True)
    ow, _ = oracle.bitmap(segs, 512)
    assert np.array_equal(w_host, ow)
    w_fresh, _ = b.emit_bitmap(512, 128, 384, clip=True)  # words=None: overwrite by default
    ow, _ = oracle.bitmap(segs, 512, 128, 384)
    assert np.array_equal(w_fresh, ow)
    d = torch.full((512 ** 3 // 64,), -1, dtype=torch.int64, device="cuda")
    b.emit_bitmap_device(d.data_ptr(), 512, 0, 512, clip=False, overwrite=True)
    torch.cuda.synchronize()
    ow, _ = oracle.bitmap(segs, 512)
    assert np.array_equal(d.cpu().numpy().view(np.uint64), ow)
    b.close()


@pytest.mark.parametrize("route", ["plain", "streamed", "split", "atomic"])
def test_bitmap_overwrite_store_only(vx, oracle, monkeypatch, route):
    """Overwrite mode on the tile path stores every word of the slab from the fill (empty tiles as
    zeros; no memset, no read of the old words): junk in host and device buffers never survives --
    partial tiles (V = 384, 640), slabs cutting tiles, the streamed host readback, the slab split
    on piece overflow, a batch with no sample in the slab, and the global-atomic path."""
    import torch
    if route == "streamed":
        monkeypatch.setenv("VXG_BITMAP_STREAM_MIN", "0")
    elif route == "split":  # (whole-volume slabs split; no layer alone holds that many)
        monkeypatch.setenv("VXG_BITMAP_MAX_PIECES", "4000")
    elif route == "atomic":
        monkeypatch.setenv("VXG_BITMAP_ATOMIC", "1")
    for V in (384, 640):
        segs = np.concatenate([vx.gen_segments(2000 if route == "split" else 3000, 0, 250, V,
                                               29 + V),
                               np.array([[5.0, 5.0, 5.0, 9.0, 7.0, 6.0]])])  # (all in one corner)
        b = vx.Batch(segs)
        for z0, z1 in [(0, V), (V // 3, V // 3 + 130), (V - 100, V)]:
            n = V * V * (z1 - z0) // 64
            junk = np.full(n, np.uint64(0xF0F0F0F0F0F0F0F0), np.uint64)
            w, _ = b.emit_bitmap(V, z0, z1, clip=True, words=junk, overwrite=True)
            ow, _ = oracle.bitmap(segs, V, z0, z1)
            assert np.array_equal(w, ow), (route, V, z0, z1)
            d = torch.full((n,), -1, dtype=torch.int64, device="cuda")
            b.emit_bitmap_device(d.data_ptr(), V, z0, z1, clip=True, overwrite=True)
            torch.cuda.synchronize()
            assert np.array_equal(d.cpu().numpy().view(np.uint64), ow), (route, V, z0, z1)
        b.close()
    # no sample in the slab at all: the slab comes back as zeros
    b = vx.Batch(np.array([[1.0, 1.0, 1.0, 20.0, 9.0, 4.0]] * 70000))
    d = torch.full((384 * 384 * 128 // 64,), -1, dtype=torch.int64, device="cuda")
    b.emit_bitmap_device(d.data_ptr(), 384, 200, 328, clip=True, overwrite=True)
    torch.cuda.synchronize()
    assert int(d.count_nonzero()) == 0
    b.close()


@pytest.mark.parametrize("mode", ["fused", "twopass"])
def test_list_modes_match_oracle(vx, oracle, monkeypatch, mode):
    """Both list implementations -- the fused count/emit-task kernel (default for large batches)
    and the count pass + scan + emit pass -- on the same corpora, bit-exact against the oracle:
    arbitrary lengths (ranges cut segments everywhere), 1-sample segments, negative coordinates."""
    monkeypatch.setenv("VXG_LIST_MODE", mode)
    rng = np.random.default_rng(99)
    corpora = [
        vx.gen_segments(30000, 0, 2048, 4096, 123),
        np.concatenate([rng.uniform(-30, 30, size=(20000, 6)),
                        np.repeat(rng.uniform(0, 9, size=(5000, 3)), 2, axis=1).reshape(-1, 6)]),
        vx.gen_segments(50000, 37, 0, 0, 5),
    ]
    for segs in corpora:
        vox, off, total = vx.run_batch_flat(segs)
        ovox, ooff, ototal = oracle.run_batch(segs)
        assert total == ototal
        assert np.array_equal(off, ooff)
        assert np.array_equal(vox, ovox)


@pytest.mark.parametrize("mode", ["fused", "twopass"])
def test_list_fixed_point_runs_vs_fp64(vx, oracle, monkeypatch, mode):
    """The list walker's fast runs step REC_FX samples in 32.32 fixed point (vxg_device.cuh) and
    re-evaluate samples near a rounding boundary in FP64: against the all-FP64 walker
    (VXG_LIST_FX=0) and the oracle, on long random segments, tie lines (samples exactly on and a
    few ulp beside half-integers) and coordinates up to just below 2^24 (REC_FX's bound)."""
    monkeypatch.setenv("VXG_LIST_MODE", mode)
    rng = np.random.default_rng(7)
    big = rng.uniform(2 ** 24 - 5000, 2 ** 24 - 1, size=(3000, 6))
    corpora = [vx.gen_segments(20000, 0, 2048, 4096, 321),
               _tie_lines(20000, 13, [0, 1, -1, 2, -2, 3, -3]), big]
    for segs in corpora:
        ovox, ooff, ototal = oracle.run_batch(segs)
        vox, off, total = vx.run_batch_flat(segs)
        monkeypatch.setenv("VXG_LIST_FX", "0")
        vox64, off64, total64 = vx.run_batch_flat(segs)
        monkeypatch.delenv("VXG_LIST_FX")
        assert total == total64 == ototal
        assert np.array_equal(off, ooff) and np.array_equal(off64, ooff)
        assert np.array_equal(vox, ovox) and np.array_equal(vox64, ovox)


# ------------------------------------------------------------------ device-resident (torch)
def test_torch_device_buffers(vx, oracle):
    import torch
    segs = oracle.gen_batch(10000, 0, 512, 1024, 31)
    d = torch.from_numpy(segs).cuda()
    b = vx.Batch(None, device_ptr=d.data_ptr(), n=segs.shape[0])
    out = torch.empty((b.capacity, 3), dtype=torch.int32, device="cuda")
    chain = torch.empty(b.n + 1, dtype=torch.int64, device="cuda")
    total = b.emit_list_device(out.data_ptr(), b.capacity, chain.data_ptr())
    vox, off, ototal = oracle.run_batch(segs)
    assert total == ototal
    assert np.array_equal(out[:total].cpu().numpy(), vox)
    assert np.array_equal(chain.cpu().numpy(), off)
    words = torch.zeros((1024 ** 3) // 64, dtype=torch.int64, device="cuda")
    b.emit_bitmap_device(words.data_ptr(), 1024, 0, 1024, False)
    ow, _ = oracle.bitmap(segs, 1024)
    assert np.array_equal(words.cpu().numpy().view(np.uint64), ow)


@pytest.mark.parametrize("n,lmax", [(1, 1000000), (1, 1), (3000, 2048), (65536, 128)])
def test_device_batch_deferred_plan(vx, oracle, n, lmax):
    """A device-resident batch below 2^18 segments emits before its plan is read back: the
    count / scan / emit kernels take the range geometry from off[n] on the device, and the plan's
    and the emit's control blocks come back in one readback. Bit-exact against the oracle,
    capacity/N_max resolved afterwards, too-small buffers and plan errors still reported."""
    import torch
    segs = oracle.gen_batch(n, 0, lmax, 0, 40 + n)
    d = torch.from_numpy(segs).cuda()
    vox, off, ototal = oracle.run_batch(segs)
    cap = int(sum(oracle.make_plan(s)[0] + 1 for s in segs)) if n <= 3000 else None
    out = torch.empty((ototal + 4096, 3), dtype=torch.int32, device="cuda")
    chain = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    b = vx.Batch(None, device_ptr=d.data_ptr(), n=n)
    assert b._info is None                      # nothing read back yet
    total = b.emit_list_device(out.data_ptr(), out.shape[0], chain.data_ptr())
    assert total == ototal
    assert np.array_equal(out[:total].cpu().numpy(), vox)
    assert np.array_equal(chain.cpu().numpy(), off)
    if cap is not None:
        assert b.capacity == cap
    b.close()
    b = vx.Batch(None, device_ptr=d.data_ptr(), n=n)
    with pytest.raises(vx.VoxGpuError):          # buffer smaller than the list: nothing written
        b.emit_list_device(out.data_ptr(), ototal - 1, chain.data_ptr())
    b.close()
    bad = segs.copy()
    bad[n // 2, 4] = np.inf
    db = torch.from_numpy(bad).cuda()
    b = vx.Batch(None, device_ptr=db.data_ptr(), n=n)   # enqueued: no error yet
    for _ in range(2):                                   # reported, and again on the next call
        with pytest.raises(vx.RangeError):
            b.emit_list_device(out.data_ptr(), out.shape[0], chain.data_ptr())
    with pytest.raises(vx.RangeError):
        b.capacity
    b.close()


# ------------------------------------------------------------------ bulk plans (batch_preprocess)
def _quarter_grid(n, seed):
    rng = np.random.default_rng(seed)
    return np.round(rng.uniform(-80, 80, size=(n, 6)) * 4) / 4


def _plan_parity(vx, oracle, segs, d=None):
    """Every plan field of a batch against the oracle's batch_preprocess (src/batch.cpp:57-73):
    N_i, W_i as raw uint64 bit patterns, output offsets, N_max and the capacity."""
    b = vx.Batch(None, device_ptr=d.data_ptr(), n=d.shape[0]) if d is not None else vx.Batch(segs)
    p = b.plans()
    o = oracle.batch_preprocess(segs)
    assert np.array_equal(p["step_count"], o["steps"])
    w = np.stack([p["wx"], p["wy"], p["wz"]], axis=1)
    assert np.array_equal(w.view(np.uint64), o["step_vectors"].view(np.uint64))
    assert np.array_equal(p["output_offset"], o["offsets"])
    assert b.max_steps == o["max_steps"] and b.capacity == o["capacity"]
    b.close()
    return o["capacity"]


def test_bulk_plans_tie_corpora(vx, oracle):
    """Plans of corpora built to expose rounding and FMA contraction: the decimal grid (317 of
    2.8M samples round differently under FMA), the quarter grid (ties in
    round(S) == round(E) and in N), the reference tests' mixed corpora, random doubles."""
    for segs in (np.asarray(decimal_grid_corpus(200000, 4321)), _quarter_grid(200000, 17),
                 np.asarray(mixed_batch(20000, 402, 3, 500.0)),
                 np.random.default_rng(5).uniform(-1e6, 1e6, size=(200000, 6))):
        _plan_parity(vx, oracle, segs)


@pytest.mark.parametrize("cfg", ["cfg1", "cfg4", "cfg3"])
def test_bulk_plans_full_configs(vx, oracle, cfg):
    """batch_preprocess at the bench's full sizes and seeds: cfg1 (65,536 x N=128), cfg4 (4M, N ~
    U{1..2048}), cfg3 (16M x N=64): every N_i, W_i bit pattern and offset equals the oracle's."""
    import torch
    n, lf, lm, V, seed = {"cfg1": (65536, 128, 0, 512, 0x5EED0101),
                          "cfg4": (4 << 20, 0, 2048, 4096, 0x5EED0104),
                          "cfg3": (16 << 20, 64, 0, 1024, 0x5EED0103)}[cfg]
    ctx = vx.default_context()
    d = torch.empty((n, 6), dtype=torch.float64, device="cuda")
    ctx.check(ctx.lib.vxg_gen_segments(ctx.h, n, None, None, lf, lm, V, seed, d.data_ptr(), 1))
    segs = d.cpu().numpy()
    assert np.array_equal(segs.view(np.uint64),
                          oracle.gen_batch(n, lf, lm, V, seed, nthreads=0).view(np.uint64))
    _plan_parity(vx, oracle, segs, d)


def test_count_voxels(vx, oracle):
    """vxg_batch_count_voxels (the count pass alone) equals BatchResult.total_voxels of the
    oracle and the list path's total, on short, long and tie-heavy corpora."""
    for segs in (vx.gen_segments(20000, 128, 0, 512, 3), vx.gen_segments(5000, 0, 2048, 4096, 4),
                 _quarter_grid(30000, 9), np.asarray(decimal_grid_corpus(30000, 77))):
        b = vx.Batch(segs)
        t = b.count_voxels()
        _, _, total = b.emit_list()
        assert t == total == oracle.run_batch(segs)[2]
        b.close()


@pytest.mark.parametrize("case", ["cfg1", "mixed", "ties", "long", "one", "errors", "cap"])
def test_run_batch_device_one_launch(vx, oracle, case):
    """vxg_run_batch_device (plan + count + look-back prefix + emit in one kernel) against the
    oracle: config-1 shape, arbitrary lengths with zero-step segments, ties, a batch holding a
    segment too long for it (re-routed to the multi-pass path), n = 1, a range error (lowest
    segment reported), an undersized output buffer; also the asynchronous form."""
    import torch
    segs = {"cfg1": lambda: vx.gen_segments(65536, 128, 0, 512, 0x5EED0101),
            "mixed": lambda: np.concatenate([vx.gen_segments(3000, 0, 700, 1024, 5),
                                             np.array([[3.2, 4.4, 5.1, 3.3, 4.2, 5.0]] * 70)]),
            "ties": lambda: _quarter_grid(50000, 31),
            "long": lambda: np.concatenate([vx.gen_segments(500, 0, 300, 1024, 6),
                                            [[0.0, 0.0, 0.0, 40000.0, 3.0, 1.0]]]),
            "one": lambda: np.array([[0.1, 0.3, 0.7, 12.45, 4.9, 0.2]]),
            "errors": lambda: np.array([[0, 0, 0, 5, 5, 5], [0, 0, 0, 1, 1, 1],
                                        [0, 0, 0, 3e9, 0, 0], [0, 0, 0, 1, 2, 3],
                                        [np.nan, 0, 0, 1, 1, 1]], dtype=np.float64),
            "cap": lambda: vx.gen_segments(2000, 64, 0, 256, 8)}[case]()
    d = torch.from_numpy(np.ascontiguousarray(segs, dtype=np.float64)).cuda()
    n = d.shape[0]
    if case == "errors":
        out = torch.empty((1000, 3), dtype=torch.int32, device="cuda")
        chain = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        with pytest.raises(vx.RangeError) as ei:
            vx.run_batch_device(d.data_ptr(), n, out.data_ptr(), 1000, chain.data_ptr())
        assert ei.value.segment == 2  # the lowest failing segment, as batch_preprocess reports
        return
    ovox, ooff, ototal = oracle.run_batch(segs)
    cap = ototal - 1 if case == "cap" else ototal
    out = torch.empty((max(cap, 1), 3), dtype=torch.int32, device="cuda")
    chain = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    if case == "cap":
        with pytest.raises(vx.LogicError):
            vx.run_batch_device(d.data_ptr(), n, out.data_ptr(), cap, chain.data_ptr())
        return
    total = vx.run_batch_device(d.data_ptr(), n, out.data_ptr(), cap, chain.data_ptr())
    assert total == ototal
    assert np.array_equal(chain.cpu().numpy(), ooff)
    assert np.array_equal(out.cpu().numpy()[:total], ovox)
    out.zero_()
    if case == "long":  # asynchronous: one call is re-routed by its result, a chain is refused
        vx.run_batch_device(d.data_ptr(), n, out.data_ptr(), cap, chain.data_ptr(), sync=False)
        t, mx, capa = vx.run_batch_device_result()
        o = oracle.batch_preprocess(segs)  # (N_max and capacity of the re-routed plan)
        assert t == ototal and capa == o["capacity"] and mx == o["max_steps"]
        assert np.array_equal(out.cpu().numpy()[:total], ovox)
        for _ in range(2):
            vx.run_batch_device(d.data_ptr(), n, out.data_ptr(), cap, chain.data_ptr(), sync=False)
        with pytest.raises(vx.InvalidArgument):
            vx.run_batch_device_result()
        return
    for _ in range(3):  # asynchronous form: enqueue several, read the last
        vx.run_batch_device(d.data_ptr(), n, out.data_ptr(), cap, chain.data_ptr(), sync=False)
    t, mx, capa = vx.run_batch_device_result()
    o = oracle.batch_preprocess(segs)
    assert t == ototal and capa == o["capacity"] and mx == o["max_steps"]
    assert np.array_equal(out.cpu().numpy()[:total], ovox)


def _tie_lines(n, seed, ulps, hi=3000):
    """Axis-parallel and diagonal segments whose samples S + W*k land exactly on (or a few ulp
    beside) half-integers: W is an exact small dyadic step and S.x sits on/next to a tie."""
    rng = np.random.default_rng(seed)
    segs = np.empty((n, 6))
    base = rng.integers(2, hi, size=(n, 3)).astype(np.float64) + 0.5
    for i in range(n):
        u = ulps[i % len(ulps)]
        s = base[i].copy()
        for _ in range(abs(u)):
            s[0] = np.nextafter(s[0], np.inf if u > 0 else 0.0)
        L = float(rng.integers(1, 400))
        dirs = [(L, 0.0, 0.0), (L, L, 0.0), (L, L / 2, L / 4), (L, 0.0, L)]
        d = dirs[i % len(dirs)]
        segs[i, :3] = s
        segs[i, 3:] = s + np.asarray(d)
    return segs


def test_round_pos_ties_in_situ(vx, oracle):
    """The one-DADD rounding (round_pos, records with every coordinate >= 1) on samples that sit
    exactly on ties and within +-3 ulp of them: voxel lists and bitmaps equal the oracle's
    (llround, ties away from zero). The host-side proof check is
    tests/test_oracle_golden.py::test_round_pos_identity_host."""
    segs = _tie_lines(40000, 11, [0, 1, -1, 2, -2, 3, -3])
    assert segs.min() >= 1.0  # REC_POS: the round_pos path
    _compare(vx, oracle, segs)
    V = 4096
    words, outside = vx.voxelize_bitmap(segs, V, 0, V, clip=False)
    ow, oo = oracle.bitmap(segs, V, nthreads=0, zpart=True)
    assert outside == oo
    assert np.array_equal(words, ow)


# ------------------------------------------------------------------ full BASELINE sizes
@pytest.mark.slow
def test_full_config4_list_hashes(vx, oracle):
    """Config 4 at full size and the bench's seed: 4M segments, N ~ U{1..2048}: every chain's
    length and order-sensitive hash equal the oracle's (4.3 G samples); first/last voxels
    pinned."""
    import torch
    from tests.gpu_checks import device_chain_hashes
    n = 4 * 1024 * 1024
    d = torch.empty((n, 6), dtype=torch.float64, device="cuda")
    ctx = vx.default_context()
    ctx.check(ctx.lib.vxg_gen_segments(ctx.h, n, None, None, 0, 2048, 4096, 0x5EED0104, d.data_ptr(), 1))
    b = vx.Batch(None, device_ptr=d.data_ptr(), n=n)
    out = torch.empty((b.capacity, 3), dtype=torch.int32, device="cuda")
    chain = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    total = b.emit_list_device(out.data_ptr(), b.capacity, chain.data_ptr())
    segs = d.cpu().numpy()
    h, ln = device_chain_hashes(out[:total], chain)
    oh, oln = oracle.chain_hashes(segs)
    assert int(oln.sum()) == total
    assert np.array_equal(ln, oln)
    assert np.array_equal(h, oh)
    # first voxel of every chain is round(S), last is round(E)
    first = out[chain[:-1]].cpu().numpy()
    last = out[chain[1:] - 1].cpu().numpy()
    assert np.array_equal(first, np.floor(segs[:, :3] + 0.5).astype(np.int32))
    assert np.array_equal(last, np.floor(segs[:, 3:] + 0.5).astype(np.int32))


@pytest.mark.slow
def test_full_config3_bitmap(vx, oracle):
    """Config 3 at full size (16M segments, N = 64, 1024^3, the bench's seed): the device
    bitmap, the streamed host bitmap and the oracle's bitmap over all 1.09 G samples agree bit
    for bit, and so do the outside counts."""
    import torch
    V, n = 1024, 16 * 1024 * 1024
    d = torch.empty((n, 6), dtype=torch.float64, device="cuda")
    ctx = vx.default_context()
    ctx.check(ctx.lib.vxg_gen_segments(ctx.h, n, None, None, 64, 0, V, 0x5EED0103, d.data_ptr(), 1))
    b = vx.Batch(None, device_ptr=d.data_ptr(), n=n)
    w = torch.zeros(V ** 3 // 64, dtype=torch.int64, device="cuda")
    out_d = b.emit_bitmap_device(w.data_ptr(), V, 0, V, False)
    host, out_h = b.emit_bitmap(V)  # 128 MiB: the streamed readback
    segs = d.cpu().numpy()
    ow, oo = oracle.bitmap(segs, V)
    assert np.array_equal(w.cpu().numpy().view(np.uint64), ow)
    assert np.array_equal(host, ow)
    assert out_d == out_h == oo


@pytest.mark.slow
def test_full_config5_slabs_consistent(vx, oracle):
    """Config 5 geometry (4096^3 bitmap, N ~ U{1..2048}) on 8M segments: the 8 device-clipped
    z-slabs reassemble the unclipped full bitmap bit for bit, and a 1/512 subsample of the
    segments matches the oracle's bitmap exactly."""
    import torch
    V, n = 4096, 8 * 1024 * 1024
    d = torch.empty((n, 6), dtype=torch.float64, device="cuda")
    ctx = vx.default_context()
    ctx.check(ctx.lib.vxg_gen_segments(ctx.h, n, None, None, 0, 2048, V, 0x5EED0005, d.data_ptr(), 1))
    b = vx.Batch(None, device_ptr=d.data_ptr(), n=n)
    nwords = V * V * V // 64
    full = torch.zeros(nwords, dtype=torch.int64, device="cuda")
    b.emit_bitmap_device(full.data_ptr(), V, 0, V, False)
    slabs = torch.zeros(nwords, dtype=torch.int64, device="cuda")
    h = V // 8
    per = nwords // 8
    for g in range(8):
        b.emit_bitmap_device(slabs.data_ptr() + 8 * g * per, V, g * h, (g + 1) * h, True)
    assert torch.equal(full, slabs)
    del slabs, full
    sub = d[::512].contiguous()
    bs = vx.Batch(None, device_ptr=sub.data_ptr(), n=sub.shape[0])
    w = torch.zeros(nwords, dtype=torch.int64, device="cuda")
    bs.emit_bitmap_device(w.data_ptr(), V, 0, V, True)
    ow, _ = oracle.bitmap(sub.cpu().numpy(), V)
    assert np.array_equal(w.cpu().numpy().view(np.uint64), ow)


@pytest.mark.slow
def test_full_config5_bitmap_oracle(vx, oracle):
    """Config 5 at full size and the bench's seed (64M segments, N ~ U{1..2048}, 4096^3, 68.8 G
    samples): the full-volume device bitmap and its outside count equal the oracle's bit for bit
    (oracle: z-partitioned over all host cores); then, for N = 2, 4, 8 ranks, the bench's own
    per-rank pipeline -- sample-balanced slabs (shard.sample_balanced_slabs over
    Batch.slab_samples) -> on-device slab filter (vxg_select_slab_segments) -> Batch -> clipped
    emit_bitmap -- reassembles that same bitmap."""
    import torch
    from paper_2009_09500_b200.shard import sample_balanced_slabs, select_slab_segments
    V, n = 4096, 64 << 20
    ctx = vx.default_context()
    d = torch.empty((n, 6), dtype=torch.float64, device="cuda")
    ctx.check(ctx.lib.vxg_gen_segments(ctx.h, n, None, None, 0, 2048, V, 0x5EED0105, d.data_ptr(), 1))
    nwords = V * V * V // 64
    full = torch.zeros(nwords, dtype=torch.int64, device="cuda")
    b = vx.Batch(None, device_ptr=d.data_ptr(), n=n)
    out_dev = b.emit_bitmap_device(full.data_ptr(), V, 0, V, False)
    segs = d.cpu().numpy()
    ow, oo = oracle.bitmap(segs, V, nthreads=0, zpart=True)
    assert out_dev == oo
    assert np.array_equal(full.cpu().numpy().view(np.uint64), ow)
    del ow, segs
    plane = V * V // 64
    local = torch.empty_like(d)
    for world in (2, 4, 8):
        slabs = sample_balanced_slabs(b.slab_samples, V, world)
        assert slabs[0][0] == 0 and slabs[-1][1] == V
        cat = torch.zeros(nwords, dtype=torch.int64, device="cuda")
        for z0, z1 in slabs:
            k = select_slab_segments(ctx, d.data_ptr(), n, z0, z1, local.data_ptr())
            part = vx.Batch(None, device_ptr=local.data_ptr(), n=k)
            part.emit_bitmap_device(cat.data_ptr() + 8 * z0 * plane, V, z0, z1, True)
            part.close()
        assert torch.equal(cat, full), world
        del cat
    b.close()


def test_host_buffer_validation(vx):
    """Caller-supplied host buffers are checked before the library writes through them."""
    b = vx.Batch(vx.gen_segments(100, 16, 0, 64, 3))
    cap = b.capacity
    with pytest.raises(vx.InvalidArgument):
        b.emit_list(out=np.empty((cap, 3), np.int64))
    with pytest.raises(vx.InvalidArgument):
        b.emit_list(out=np.empty((cap, 4), np.int32))
    with pytest.raises(vx.InvalidArgument):
        b.emit_list(chain_off=np.empty(50, np.int64))
    with pytest.raises(vx.InvalidArgument):
        b.emit_list(out=np.empty((cap, 6), np.int32)[:, ::2])
    with pytest.raises(vx.InvalidArgument):
        b.emit_bitmap(64, words=np.empty(10, np.uint64))
    with pytest.raises(vx.InvalidArgument):
        b.emit_bitmap(64, words=np.empty(64 ** 3 // 64, np.int32))
    words, _ = b.emit_bitmap(64, words=np.zeros(64 ** 3 // 64, np.uint64))
    assert words.any()
    b.close()
