"""Pin the CPU oracle (oracle/voxline_oracle.c) before trusting it (CPU only).

1. against the golden vectors generated from the reference itself (tests/golden/golden.json);
2. against the reference compiled unmodified (oracle/_ref), when it was built here.
"""
import numpy as np
import pytest

from tests.golden.make_golden import (decimal_grid_corpus, digest, mixed_batch, seg_digest)

pytestmark = pytest.mark.filterwarnings("ignore")


def test_splitmix_kat(oracle, golden):
    # tests/test_bench.cpp:226-239
    assert [hex(v) for v in oracle.splitmix(0, 3)] == golden["splitmix_seed0"]
    assert golden["splitmix_seed0"] == ["0xe220a8397b1dcdaf", "0x6e789e6aa1b965f4",
                                        "0x6c45d188009454f"]


def test_plans_and_chains(oracle, golden):
    for name, case in golden["plans"].items():
        n, w = oracle.make_plan(case["segment"])
        assert n == case["n"], name
        assert [float.fromhex(h) for h in case["w_hex"]] == list(w), name
        assert oracle.voxelize_parametric(case["segment"]).tolist() == case["chain"], name
        assert list(oracle.chain_length_bounds(case["segment"])) == case["bounds"], name


def test_reference_known_answers(golden):
    p = golden["plans"]
    # tests/test_parametric.cpp:37-73
    assert p["x5"]["n"] == 5 and p["diag3"]["n"] == 5 and p["same_voxel"]["n"] == 0
    assert p["clamp1"]["n"] == 1 and p["ceil_extent"]["n"] == 3
    assert p["ceil_extent"]["chain"] == [[0, 0, 0], [1, 0, 0], [2, 0, 0], [3, 0, 0]]
    # tests/test_parametric.cpp:115-125
    assert p["diag3"]["chain"] == [[0, 0, 0], [1, 1, 1], [2, 2, 2], [3, 3, 3]]
    assert p["degenerate"]["chain"] == [[2, -1, 7]]
    # SURVEY.md §8c adversarial vectors
    assert len(p["fma_sensitive"]["chain"]) == 14 and p["fma_sensitive"]["chain"][12] == [11, 5, 0]
    assert p["ties"]["chain"] == [[1, 1, 1], [-1, -1, -1]]
    assert p["int32_edge"]["chain"][-1] == [2147483647, 0, 0] and len(p["int32_edge"]["chain"]) == 8
    # tests/acceptance_main.cpp:314-339 (criterion 5)
    c = golden["acceptance_c4c5"]
    assert (c["live"], c["redundant"], c["grid"]) == (501024, 2986720, 3487744)


def test_rounding(oracle, golden):
    for case in golden["round_ok"]:
        assert list(oracle.round_point(case["p"])) == case["v"]
    from oracle.pyoracle import OracleError
    for case in golden["round_bad"]:
        p = [float(x) for x in case["p"]]
        with pytest.raises(OracleError) as e:
            oracle.round_point(p)
        assert e.value.code == case["code"]


def test_batch_known_answers(oracle, golden):
    b = oracle.batch_preprocess([[0, 0, 0, 5, 0, 0], [0, 0, 0, 3, 3, 3]])
    assert b["steps"].tolist() == golden["batch_two"]["steps"]
    assert b["offsets"].tolist() == golden["batch_two"]["offsets"] == [0, 6]
    assert b["capacity"] == golden["batch_two"]["capacity"] == 12
    vox, off, total = oracle.run_batch([[0, 0, 0, 5, 0, 0], [0, 0, 0, 2, 1, 0]])
    gs = golden["batch_short"]
    assert [vox[off[i]:off[i + 1]].tolist() for i in range(2)] == gs["chains"]
    assert gs["chains"][1] == [[0, 0, 0], [1, 1, 0], [2, 1, 0]]  # tests/test_batch.cpp:94-102
    assert total == gs["total"]


def test_generators(oracle, golden):
    for key, hexes in golden["gen_segment_of_length"].items():
        target, seed = map(int, key.split("_"))
        s = oracle.gen_segment_of_length(target, seed)
        assert [float.fromhex(h) for h in hexes] == s.tolist(), key
        assert oracle.make_plan(s)[0] == target
    arb = oracle.gen_arbitrary_batch(10000000, 1024, 7)
    assert seg_digest(arb) == golden["gen_arbitrary_10M_1024_7"]["digest"]
    assert int(oracle.batch_preprocess(arb)["steps"].sum()) == 10000000


def test_acceptance_c4_c5(oracle, golden):
    c = golden["acceptance_c4c5"]
    arb = oracle.gen_arbitrary_batch(500000, 1024, c["seed"])
    assert seg_digest(arb) == c["digest_segments"]
    b = oracle.batch_preprocess(arb)
    assert b["capacity"] == c["live"]
    assert 1024 * (b["max_steps"] + 1) - b["capacity"] == c["redundant"]
    vox, off, total = oracle.run_batch(arb)
    assert total == c["total_voxels"] and digest(vox, off) == c["digest_chains"]


def _corpus(name, spec, oracle):
    if spec["kind"] == "gen":
        return oracle.gen_batch(**spec["params"])
    if name.startswith("decimal_grid_fine"):
        return np.asarray(decimal_grid_corpus(20000, 78, step=0.1, span=60))
    if name.startswith("decimal_grid"):
        return np.asarray(decimal_grid_corpus(20000, 77))
    count, seed = int(name.split("_")[-2]), int(name.split("_")[-1])
    long_every, max_len = {"test_batch_mixed": (3, 500.0),
                           "test_parametric_invariants": (5, 1e4),
                           "test_parametric_plans": (4, 1e4)}["_".join(name.split("_")[:-2])]
    return np.asarray(mixed_batch(count, seed, long_every, max_len))


def test_corpora_digests(oracle, golden):
    for name, spec in golden["corpora"].items():
        segs = _corpus(name, spec, oracle)
        assert seg_digest(segs) == spec["digest_segments"], name
        vox, off, total = oracle.run_batch(segs)
        assert total == spec["total_voxels"], name
        assert digest(vox, off) == spec["digest"], name


def test_bitmap_matches_chains(oracle):
    segs = oracle.gen_batch(500, 64, 0, 128, 99)
    words, outside = oracle.bitmap(segs, 128)
    vox, off, total = oracle.run_batch(segs)
    expect = np.zeros_like(words)
    b = vox[:, 0].astype(np.uint64) + 128 * (vox[:, 1].astype(np.uint64) + 128 * vox[:, 2].astype(np.uint64))
    np.bitwise_or.at(expect, (b >> np.uint64(6)).astype(np.int64), np.uint64(1) << (b & np.uint64(63)))
    assert outside == 0 and np.array_equal(words, expect)
    # z-slabs tile the full bitmap
    parts = [oracle.bitmap(segs, 128, z0, z0 + 32)[0] for z0 in range(0, 128, 32)]
    assert np.array_equal(np.concatenate(parts), words)


def test_oracle_matches_reference_random(oracle, ref):
    rng = np.random.default_rng(5)
    for trial in range(5):
        segs = rng.uniform(-300, 300, size=(3000, 6))
        if trial == 4:
            segs = np.round(segs * 4) / 4  # quarter grid: exact ties
        vox_o, off_o, t_o = oracle.run_batch(segs)
        vox_r, off_r, t_r, _ = ref.run_batch(segs, workers=4)
        assert t_o == t_r and np.array_equal(off_o, off_r) and np.array_equal(vox_o, vox_r)


def test_volume_generator_plans_exact(oracle, ref):
    for V, L, Lm in [(512, 128, 0), (1024, 64, 0), (4096, 0, 2048)]:
        segs = oracle.gen_batch(2000, L, Lm, V, 123)
        steps = ref.batch_preprocess(segs)["steps"]
        if Lm == 0:
            assert (steps == L).all()
        else:
            assert steps.min() >= 1 and steps.max() <= Lm
        vox, _, _ = oracle.run_batch(segs)
        assert vox.min() >= 1 and vox.max() <= V - 2


def test_round_pos_identity_host(oracle):
    """The GPU hot loops' rounding (vxg_device.cuh round_pos: RM(c + 2^51 + 0.5), mantissa >> 1)
    equals llround (src/geometry.cpp:21) on every tie k + 0.5 (k < 2^24) and both its neighbours,
    on 2^22 random values in [0, 2^31 - 1) and 2^22 near-ties (+-8 ulp), and on edge values: 58.7M
    values, emulated on the host with the same IEEE-754 addition in round-toward-minus-infinity."""
    bad, n, first = oracle.check_round_pos(1 << 24, 1 << 22, seed=7)
    assert n > 5 * 10 ** 7
    assert bad == 0, f"round_pos differs from llround at {first!r}"
    # the check has teeth: the same addition in round-to-nearest (ties to even) must fail
    bad_rn, _, _ = oracle.check_round_pos(1 << 12, 1 << 10, seed=7, mode=1)
    assert bad_rn > 0


@pytest.mark.parametrize("V,z_lo,z_hi", [(256, 0, 256), (256, 17, 200), (100, 3, 97), (128, 0, 1),
                                         (96, 0, 96)])
def test_bitmap_zpart_matches_bitmap(oracle, V, z_lo, z_hi):
    """The z-partitioned oracle bitmap (used for the full config-5 parity run) equals the plain
    per-sample one, outside count included, on volume-crossing and out-of-volume segments."""
    rng = np.random.default_rng(V + z_lo)
    segs = rng.uniform(-60, V + 60, size=(4000, 6))
    segs[::7] = np.round(segs[::7] * 2) / 2  # ties
    a, oa = oracle.bitmap(segs, V, z_lo, z_hi, nthreads=4)
    b, ob = oracle.bitmap(segs, V, z_lo, z_hi, nthreads=4, zpart=True)
    assert oa == ob
    assert np.array_equal(a, b)


def test_bitmap_zpart_volume_generator(oracle):
    segs = oracle.gen_batch(20000, 0, 512, 1024, 0x5EED0105)
    a, oa = oracle.bitmap(segs, 1024, nthreads=4)
    b, ob = oracle.bitmap(segs, 1024, nthreads=4, zpart=True)
    assert oa == ob and np.array_equal(a, b)
