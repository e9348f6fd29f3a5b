"""Multi-GPU host logic (paper_2009_09500_b200/shard.py) on CPU: world_size-2 gloo process groups
stand in for the 8xB200 NVSwitch box (this run's GPU boxes have one GPU).

The oracle computes each rank's shard (the kernels are covered by the -m gpu tests: the device
slab clip is checked against the unclipped bitmap there); here the partitioning and the
verification gathers must reassemble exactly the single-rank result.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2009_09500_b200 import shard


def test_slab_bounds_partition():
    for V in (64, 100, 128, 4096):
        for world in range(1, 9):
            b = [shard.slab_bounds(V, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == V
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.slab_bounds(64, 2, 2)


def test_sample_balanced_slabs():
    """Equal-sample z-slabs: contiguous, disjoint, covering [0, V), and balanced to within the
    interpolation error for a density peaked in the middle of the volume (as volume-fitted
    segments are)."""
    from paper_2009_09500_b200.shard import sample_balanced_slabs
    V = 4096
    z = np.arange(V)
    dens = np.exp(-((z - V / 2) / (V / 5)) ** 2) + 0.05
    cum = np.concatenate([[0.0], np.cumsum(dens)])
    samples_in = lambda a, b: cum[b] - cum[a]  # noqa: E731
    for world in (1, 2, 3, 4, 8):
        slabs = sample_balanced_slabs(samples_in, V, world)
        assert slabs[0][0] == 0 and slabs[-1][1] == V
        assert all(a < b for a, b in slabs)
        assert all(slabs[i][1] == slabs[i + 1][0] for i in range(world - 1))
        work = np.array([samples_in(a, b) for a, b in slabs])
        assert work.max() / work.mean() < 1.02, (world, work)
    eq = [(r * V // 8, (r + 1) * V // 8) for r in range(8)]
    ew = np.array([samples_in(a, b) for a, b in eq])
    assert ew.max() / ew.mean() > 1.5  # what equal depths would have given


def test_time_balanced_slabs():
    """Rebalancing from measured times: a rank that was slow for its samples (a per-rank fixed
    cost) gets fewer samples, the cuts stay contiguous and cover [0, V), equal speeds leave the
    sample-balanced cuts as they were."""
    from paper_2009_09500_b200.shard import sample_balanced_slabs, time_balanced_slabs
    V = 4096
    z = np.arange(V)
    dens = np.exp(-((z - V / 2) / (V / 5)) ** 2) + 0.05
    cum = np.concatenate([[0.0], np.cumsum(dens)])
    samples_in = lambda a, b: cum[b] - cum[a]  # noqa: E731
    slabs = sample_balanced_slabs(samples_in, V, 8)
    work = np.array([samples_in(a, b) for a, b in slabs])
    same = time_balanced_slabs(samples_in, V, slabs, work / 1e6)  # equal speeds
    assert all(abs(a[0] - b[0]) <= 2 for a, b in zip(same, slabs))
    times = work / 1e6
    times[0] *= 1.05  # rank 0 is 5% slower than its samples say
    new = time_balanced_slabs(samples_in, V, slabs, times)
    assert new[0][0] == 0 and new[-1][1] == V
    assert all(new[i][1] == new[i + 1][0] for i in range(7))
    nw = np.array([samples_in(a, b) for a, b in new])
    assert nw[0] < work[0] and nw[1:].sum() > work[1:].sum()
    pred = nw / (work / times)  # each rank at its measured speed
    assert pred.max() / pred.min() < 1.02


def test_sample_balanced_cuts(oracle):
    segs = oracle.gen_batch(5000, 0, 2048, 4096, 0x5EED0004)
    steps, _, off, nmax, cap = _plan(oracle, segs)
    for world in (1, 2, 3, 8):
        c = shard.sample_balanced_cuts(off, world)
        assert c[0] == 0 and c[-1] == len(segs) and np.all(np.diff(c) >= 0)
        work = np.diff(off[c])
        assert work.sum() == cap
        assert work.max() - cap / world <= nmax + 1  # within one segment of balanced


def _plan(oracle, segs):
    import ctypes as C
    n = segs.shape[0]
    steps = np.zeros(n, np.int64)
    w3 = np.zeros((n, 3))
    off = np.zeros(n + 1, np.int64)
    nmax, cap = C.c_int64(), C.c_int64()
    p = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
    assert oracle.lib.vo_batch_preprocess(p(np.ascontiguousarray(segs), C.c_double), n,
                                          p(steps, C.c_int64), p(w3, C.c_double),
                                          p(off, C.c_int64), C.byref(nmax), C.byref(cap)) == 0
    off[n] = cap.value
    return steps, w3, off, nmax.value, cap.value


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle.pyoracle import Oracle
        o = Oracle()
        V = 128
        segs = o.gen_batch(3000, 0, 96, V, 77 + 0)  # identical inputs on every rank
        # ---- bitmap: z-slab per rank, gathered == the full bitmap
        z_lo, z_hi = shard.slab_bounds(V, world, rank)
        words, _ = o.bitmap(segs, V, z_lo, z_hi)
        full = shard.gather_bitmap(torch.from_numpy(words.view(np.int64)), V)
        ref, _ = o.bitmap(segs, V)
        ok_bitmap = np.array_equal(full.numpy().view(np.uint64), ref)
        # ---- list: sample-balanced segment ranges, gathered == the single-rank list
        _, _, off, _, _ = _plan(o, segs)
        c = shard.sample_balanced_cuts(off, world)
        mine = segs[c[rank]:c[rank + 1]]
        vox, choff, total = o.run_batch(mine)
        gv, go = shard.gather_list(torch.from_numpy(vox), torch.from_numpy(choff))
        rv, ro, rt = o.run_batch(segs)
        ok_list = np.array_equal(gv.numpy(), rv) and np.array_equal(go.numpy(), ro)
        # ---- scalar reductions used by bench.py (max-over-ranks timing, summed work)
        mx = shard.max_over_ranks(float(rank + 1))
        sm = shard.sum_over_ranks(float(total))
        ok_reduce = mx == float(world) and sm == float(rt)
        # ---- bench --verify: every rank's digest equals the digest of the same slice of the
        # one-rank result (lists: chain range; bitmaps: z-slab words)
        dl = shard.list_digest(torch.from_numpy(vox), torch.from_numpy(choff))
        dw = shard.words_digest(torch.from_numpy(words.view(np.int64)))
        got = shard.gather_objects((int(c[rank]), int(c[rank + 1]), dl, z_lo, z_hi, dw))
        plane = V * V // 64
        refw = torch.from_numpy(ref.view(np.int64))
        ok_verify = all(
            tuple(shard.list_digest(torch.from_numpy(rv[ro[a]:ro[b]]),
                                    torch.from_numpy(ro[a:b + 1]))) == tuple(d1)
            and shard.words_digest(refw[za * plane:zb * plane]) == d2
            for a, b, d1, za, zb, d2 in got)
        # a digest notices a single flipped bit / voxel
        bad = words.copy()
        bad[len(bad) // 2] ^= np.uint64(1 << 17)
        ok_verify &= shard.words_digest(torch.from_numpy(bad.view(np.int64))) != dw
        vbad = vox.copy()
        if len(vbad):
            vbad[len(vbad) // 2, 1] += 1
            ok_verify &= tuple(shard.list_digest(torch.from_numpy(vbad), torch.from_numpy(choff))) != tuple(dl)
        # ---- bench's e2e input path: 1/world of the host segments per rank + all-gather
        out = torch.empty((segs.shape[0] - segs.shape[0] % world, 6), dtype=torch.float64)
        host = np.ascontiguousarray(segs[: out.shape[0]])
        shard.distribute_segments(host, out)
        ok_dist = np.array_equal(out.numpy(), host)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok_bitmap, ok_list, ok_reduce and ok_verify and ok_dist, None))
    except Exception as e:  # report instead of hanging the parent
        import traceback
        q.put((rank, False, False, False, traceback.format_exc()))


def test_gloo_world2_slabs_and_lists():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_b, ok_l, ok_r, err in sorted(results):
        assert err is None, f"rank {rank}: {err}"
        assert ok_b, f"rank {rank}: gathered slab bitmaps differ from the full bitmap"
        assert ok_l, f"rank {rank}: gathered list shards differ from the single-rank list"
        assert ok_r, f"rank {rank}: reductions, verify digests or distribute_segments wrong"
