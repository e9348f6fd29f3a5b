"""Lane-vector emulation of the emit kernels' warp-level control flow (debug aid, CPU only).

Mirrors RowWalker / warp_find_entry / walker_row and the bitmap kernel of
paper_2009_09500_b200/csrc/vxg_kernels.cu with numpy lane vectors, so index logic can be checked
against the oracle without a GPU. Arithmetic (sampling) uses the oracle's scalar functions.

    python tools/warp_emu.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Oracle  # noqa: E402

LANES = np.arange(32, dtype=np.int64)
NO_ENTRY = (1 << 63) - 1


def warp_find_entry(off, lo, hi, f):
    while hi - lo > 31:
        step = (hi - lo + 32) // 32
        p = lo + LANES * step
        ok = (p <= hi) & (off[np.minimum(p, len(off) - 1)] <= f)
        last = int(np.nonzero(ok)[0].max())
        lo = lo + last * step
        hi = min(hi, lo + step - 1)
    p = lo + LANES
    ok = (p <= hi) & (off[np.minimum(p, len(off) - 1)] <= f)
    return lo + int(np.nonzero(ok)[0].max())


class Walker:
    def __init__(self, off, lo, hi, f):
        self.c = warp_find_entry(off, lo, hi, f)
        self.so_c = int(off[self.c])
        self.so_next = int(off[self.c + 1])

    def row(self, off, n_entries, row_start):
        if self.so_next > row_start + 32:
            z = np.zeros(32, np.int64)
            return z + self.c, z + self.so_c, z + self.so_next
        idx = self.c + 1 + LANES
        B = np.where(idx <= n_entries, off[np.minimum(idx, n_entries)], NO_ENTRY)
        d = B - row_start
        pos = 0
        for dd in d:
            if dd < 32:
                pos |= 1 << int(dd)
        nb = np.array([bin(pos & ((2 << L) - 1)).count("1") for L in range(32)], np.int64)
        b_prev = B[np.where(nb == 0, 0, nb - 1)]
        b_next = B[nb]
        my_entry = self.c + nb
        my_start = np.where(nb == 0, self.so_c, b_prev)
        adv = int((d <= 32).sum())
        if adv > 0:
            nc, nn = B[adv - 1], B[adv & 31]
            self.c += adv
            self.so_c = int(nc)
            self.so_next = int(nn) if adv < 32 else int(off[self.c + 1])
        return my_entry, my_start, b_next


def tile_index(off, n_entries, ts):
    ntiles = (off[n_entries] + ts - 1) // ts
    tile_seg = np.zeros(ntiles, np.int64)
    for c in range(n_entries):
        o, e = off[c], off[c + 1]
        if e <= o:
            continue
        for t in range((o + ts - 1) // ts, (e - 1) // ts + 1):
            tile_seg[t] = c
    return tile_seg


def emulate_entries(off, nw=8, ipt=16):
    """-> per flat sample (entry, k) as assigned by the walker, for every tile/warp/row."""
    n = len(off) - 1
    total = int(off[n])
    ch = 32 * ipt
    ts = ch * nw
    tile_seg = tile_index(off, n, ts)
    ntiles = len(tile_seg)
    ent = np.full(total, -1, np.int64)
    kk = np.full(total, -1, np.int64)
    for tile in range(ntiles):
        t0 = tile * ts
        tend = min(t0 + ts, total)
        e_lo = tile_seg[tile]
        e_hi = tile_seg[tile + 1] if tile + 1 < ntiles else n - 1
        for warp in range(nw):
            wbase = t0 + warp * ch
            if wbase >= tend:
                continue
            w = Walker(off, e_lo, e_hi, wbase)
            for j in range(ipt):
                row_start = wbase + 32 * j
                if row_start >= tend:
                    break
                e, st, nx = w.row(off, n, row_start)
                f = row_start + LANES
                v = f < tend
                ent[f[v]] = e[v]
                kk[f[v]] = (f - st)[v]
    return ent, kk


def main():
    o = Oracle()
    rng = np.random.default_rng(1)
    for trial, segs in enumerate([o.gen_batch(2000, 64, 0, 256, 77), o.gen_batch(3000, 0, 40, 256, 5),
                                  o.gen_batch(500, 0, 3, 256, 9)]):
        p = o.batch_preprocess(segs)
        steps = p["steps"]
        off = np.concatenate([p["offsets"], [p["capacity"]]]).astype(np.int64)
        ent, kk = emulate_entries(off)
        exp_ent = np.repeat(np.arange(len(steps)), steps + 1)
        exp_k = np.concatenate([np.arange(s + 1) for s in steps])
        bad = np.nonzero((ent != exp_ent) | (kk != exp_k))[0]
        print(f"trial {trial}: samples {len(ent)}, mismatches {len(bad)}", bad[:10])


if __name__ == "__main__":
    main()
