"""Generate tests/golden/*.json from the REFERENCE implementation itself.

Runs in the build container only (needs oracle/_ref/libref_voxline.so, compiled unmodified from
/root/reference by `make -C oracle ref`). The fixtures it writes are small and committed; the GPU
box (which has no /root/reference) checks against them.

    python tests/golden/make_golden.py

Contents:
  * the known-answer vectors of the reference's own tests (tests/test_parametric.cpp:37-125,
    tests/test_batch.cpp:35-102, tests/test_bench.cpp:21-30,226-239, tests/python/test_smoke.py,
    tests/acceptance_main.cpp:282-339) evaluated by the reference;
  * survey-found adversarial vectors (FMA-sensitive, ties, int32 edge);
  * hashes of reference run_batch outputs over seeded corpora: the reference's random_segment /
    random_long_segment corpora (tests/test_support.hpp:20-52), a decimal-grid corpus that
    exposes FMA contraction, and scaled-down BASELINE configs from the volume generator.
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Oracle, OracleError, RefOracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
MASK = (1 << 64) - 1


class SplitMix64:
    """include/voxline/bench.hpp:20-37 (pure Python, for building corpora)."""

    def __init__(self, seed: int):
        self.state = seed & MASK

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def uniform(self, lo=None, hi=None) -> float:
        u = float(self.next() >> 11) * 2.0 ** -53
        if lo is None:
            return u
        return lo + (hi - lo) * u


def random_segment(rng: SplitMix64, lo: float, hi: float):
    """tests/test_support.hpp:25-28"""
    return [rng.uniform(lo, hi) for _ in range(6)]


def random_long_segment(rng: SplitMix64, max_length: float):
    """tests/test_support.hpp:33-52 (Python floats are IEEE doubles; no FMA)."""
    s = [rng.uniform(-50.0, 50.0) for _ in range(3)]
    length = math.exp(rng.uniform(0.0, math.log(max_length)))
    while True:
        u = rng.uniform(-1.0, 1.0)
        v = rng.uniform(-1.0, 1.0)
        q = u * u + v * v
        if q >= 1.0 or q == 0.0:
            continue
        f = 2.0 * math.sqrt(1.0 - q)
        d = (u * f, v * f, 1.0 - 2.0 * q)
        break
    return s + [s[0] + d[0] * length, s[1] + d[1] * length, s[2] + d[2] * length]


def mixed_batch(count: int, seed: int, long_every: int, max_len: float):
    rng = SplitMix64(seed)
    return [random_long_segment(rng, max_len) if i % long_every == 0 else
            random_segment(rng, -50.0, 50.0) for i in range(count)]


def decimal_grid_corpus(count: int, seed: int, step: float = 0.05, span: int = 400):
    """Endpoints on a decimal grid (k * 0.05): rounding ties and FMA-sensitive samples."""
    rng = SplitMix64(seed)
    segs = []
    for _ in range(count):
        segs.append([(int(rng.next() % (2 * span)) - span) * step for _ in range(6)])
    return segs


def digest(vox: np.ndarray, off: np.ndarray) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(vox, dtype=np.int32).tobytes())
    h.update(np.ascontiguousarray(off, dtype=np.int64).tobytes())
    return h.hexdigest()


def seg_digest(segs: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(segs, dtype=np.float64).tobytes()).hexdigest()


def hexf(x: float) -> str:
    return float(x).hex()


def main():
    ref = RefOracle()
    orc = Oracle()
    g: dict = {"generator": "tests/golden/make_golden.py",
               "source": "oracle/_ref/libref_voxline.so (reference compiled unmodified)"}

    # --- SplitMix64 KAT (tests/test_bench.cpp:226-239)
    g["splitmix_seed0"] = [hex(v) for v in ref.splitmix(0, 3)]

    # --- plans (tests/test_parametric.cpp:37-73, tests/python/test_smoke.py:26-36)
    plan_cases = {
        "x5": [0, 0, 0, 5, 0, 0], "diag3": [0, 0, 0, 3, 3, 3], "same_voxel": [0, 0, 0, 0.2, 0.1, 0],
        "clamp1": [0.4, 0, 0, 0.6, 0, 0], "ceil_extent": [0, 0, 0, 2.999, 0, 0],
        "short": [0, 0, 0, 2, 1, 0], "negative": [-4, 2, 7, 13, -9, 4],
        "fma_sensitive": [0.1, 0.3, 0.7, 12.45, 4.9, 0.2],
        "ties": [0.5, 0.5, 0.5, -0.5, -0.5, -0.5],
        "int32_edge": [2147483640.0, 0, 0, 2147483647.4, 0, 0],
        "degenerate": [2, -1, 7, 2, -1, 7],
        "half_steps": [-2.5, 0.5, 1.5, 3.5, -0.5, -1.5],
    }
    g["plans"] = {}
    for name, s in plan_cases.items():
        n, w = ref.make_plan(s)
        chain = ref.voxelize_parametric(s)
        lo, hi = ref.chain_length_bounds(s)
        g["plans"][name] = {"segment": s, "n": n, "w_hex": [hexf(x) for x in w],
                            "chain": chain.tolist(), "bounds": [lo, hi]}

    # --- rounding (tests/python/test_smoke.py:13-23, src/geometry.cpp:15-34)
    pts = [[0.5, -0.5, 1.5], [2.5, -2.5, 0.49999999999999994], [-0.49999999999999994, 1e-300, -0.0],
           [2147483647.4, -2147483648.4, 0], [4503599627370495.5 - 4503599627370000, 0, 0]]
    g["round_ok"] = [{"p": p, "v": list(ref.round_point(p))} for p in pts]
    bad = [[3e9, 0, 0], [0, float("nan"), 0], [0, 0, float("inf")], [2147483647.5, 0, 0],
           [-2147483648.5, 0, 0], [1e300, 0, 0]]
    g["round_bad"] = []
    for p in bad:
        try:
            ref.round_point(p)
            raise SystemExit(f"reference accepted {p}")
        except OracleError as e:
            g["round_bad"].append({"p": [repr(x) for x in p], "code": e.code})

    # --- batch known answers (tests/test_batch.cpp, tests/python/test_smoke.py:69-96)
    b = ref.batch_preprocess([[0, 0, 0, 5, 0, 0], [0, 0, 0, 3, 3, 3]])
    g["batch_two"] = {"steps": b["steps"].tolist(), "offsets": b["offsets"].tolist(),
                      "max_steps": b["max_steps"], "capacity": b["capacity"]}
    b = ref.batch_preprocess([[0, 0, 0, 5, 0, 0], [0, 0, 0, 2, 1, 0]])
    g["batch_short"] = {"steps": b["steps"].tolist(), "offsets": b["offsets"].tolist(),
                        "max_steps": b["max_steps"], "capacity": b["capacity"],
                        "live": b["live"], "redundant": b["redundant"],
                        "item_1_2": list(ref.kernel_work_item([[0, 0, 0, 5, 0, 0], [0, 0, 0, 2, 1, 0]], 1, 2)),
                        "item_0_0": list(ref.kernel_work_item([[0, 0, 0, 5, 0, 0], [0, 0, 0, 2, 1, 0]], 0, 0))}
    vox, off, total, _ = ref.run_batch([[0, 0, 0, 5, 0, 0], [0, 0, 0, 2, 1, 0]])
    g["batch_short"]["chains"] = [vox[off[i]:off[i + 1]].tolist() for i in range(2)]
    g["batch_short"]["total"] = total

    # --- generators (tests/test_bench.cpp:21-57)
    gens = {}
    for target, seed in [(1000, 42), (1, 9), (2, 7), (17, 7), (333, 7), (5000, 7), (50, 42)]:
        s = ref.gen_segment_of_length(target, seed)
        gens[f"{target}_{seed}"] = [hexf(x) for x in s]
    g["gen_segment_of_length"] = gens
    arb = ref.gen_arbitrary_batch(10000000, 1024, 7)
    g["gen_arbitrary_10M_1024_7"] = {"digest": seg_digest(arb),
                                     "step_sum": int(ref.batch_preprocess(arb)["steps"].sum())}
    arb = ref.gen_arbitrary_batch(500000, 1024, 0x5EED0004)
    p = ref.batch_preprocess(arb)
    vox, off, total, _ = ref.run_batch(arb, workers=4, group_size=64)
    g["acceptance_c4c5"] = {"seed": 0x5EED0004, "digest_segments": seg_digest(arb),
                            "live": p["live"], "redundant": p["redundant"],
                            "grid": 1024 * (p["max_steps"] + 1), "total_voxels": total,
                            "digest_chains": digest(vox, off)}

    # --- corpora: reference run_batch digests
    corpora = {
        "test_batch_mixed_300_402": (mixed_batch(300, 402, 3, 500.0), None),
        "test_parametric_invariants_1500_203": (mixed_batch(1500, 203, 5, 1e4), None),
        "test_parametric_plans_1000_201": (mixed_batch(1000, 201, 4, 1e4), None),
        "decimal_grid_20000_77": (decimal_grid_corpus(20000, 77), None),
        "decimal_grid_fine_20000_78": (decimal_grid_corpus(20000, 78, step=0.1, span=60), None),
    }
    vol = {
        "cfg1_scaled_4096": dict(n=4096, len_fixed=128, len_max=0, V=512, seed=0x5EED0101),
        "cfg3_scaled_4096": dict(n=4096, len_fixed=64, len_max=0, V=1024, seed=0x5EED0103),
        "cfg4_scaled_2048": dict(n=2048, len_fixed=0, len_max=2048, V=4096, seed=0x5EED0104),
        "ref_fixed_2048_x100": dict(n=2048, len_fixed=100, len_max=0, V=0, seed=0x5EED0105),
    }
    g["corpora"] = {}
    for name, (segs, _) in corpora.items():
        a = np.asarray(segs, dtype=np.float64)
        vox, off, total, _ = ref.run_batch(a, workers=8)
        g["corpora"][name] = {"kind": "list", "digest_segments": seg_digest(a), "n": len(a),
                              "total_voxels": total, "digest": digest(vox, off),
                              "capacity": ref.batch_preprocess(a)["capacity"]}
    for name, kw in vol.items():
        a = orc.gen_batch(kw["n"], kw["len_fixed"], kw["len_max"], kw["V"], kw["seed"])
        # the volume generator is ours; pin it by re-deriving every plan with the reference
        steps = ref.batch_preprocess(a)["steps"]
        if kw["len_max"] == 0:
            assert (steps == kw["len_fixed"]).all(), name
        vox, off, total, _ = ref.run_batch(a, workers=8)
        g["corpora"][name] = {"kind": "gen", "params": kw, "digest_segments": seg_digest(a),
                              "n": kw["n"], "total_voxels": total, "digest": digest(vox, off),
                              "capacity": int((steps + 1).sum())}
    path = os.path.join(OUT, "golden.json")
    with open(path, "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
