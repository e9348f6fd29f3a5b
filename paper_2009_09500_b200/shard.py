"""Multi-GPU partitioning of the hot path: host-side logic only.

One process per GPU (torch.distributed; "nccl" on the B200 box, "gloo" in the CPU tests).
The path shards without a data-path collective:

* voxel lists (configs 1, 4): chains never interact (src/batch.cpp:139-142), so each rank owns a
  contiguous segment range; `sample_balanced_cuts` cuts the offsets scan at k * total / world so
  ranks get equal sample counts (the work), not equal segment counts;
* bitmaps (configs 3, 5): each rank owns one z-slab -- `sample_balanced_slabs` (equal sample
  counts), refined once by `time_balanced_slabs` from every rank's measured step (bench.py's
  default), or `slab_bounds(V, world, rank)` (equal depths); the device walk clips every segment
  to its slab (vxg_bitmap.cu), slabs are disjoint, no reduction.

The collectives here are input distribution, verification and reporting, never a reduction of
results: `distribute_segments` gives every rank the whole batch from one host->device slice per
rank plus an all-gather over NVLink (the z-slab ranks each need every segment that reaches their
slab); `gather_bitmap` / `gather_list` reassemble the full result on every rank and
`list_digest` / `words_digest` let ranks compare results without moving them;
`max_over_ranks` / `sum_over_ranks` reduce scalars (bench.py times each step as the max over
ranks).
"""
from __future__ import annotations

import numpy as np


def slab_bounds(V: int, world: int, rank: int) -> tuple[int, int]:
    """z-slab [z_lo, z_hi) of a V^3 volume owned by `rank` of `world` (contiguous, disjoint,
    covering [0, V); sizes differ by at most one plane)."""
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside world {world}")
    return rank * V // world, (rank + 1) * V // world


def sample_balanced_slabs(samples_in, V: int, world: int, bins: int = 64) -> list[tuple[int, int]]:
    """z-slabs [z_lo, z_hi) covering [0, V) with (nearly) equal sample counts -- the work of a
    rank's bitmap passes -- instead of equal depths: segments fitted into a volume are denser in
    its middle. `samples_in(z0, z1)` counts the samples whose rounded z lies in [z0, z1)
    (Batch.slab_samples); the cuts interpolate linearly inside `bins` equal-depth bins."""
    if world < 1:
        raise ValueError("world must be >= 1")
    edges = [i * V // bins for i in range(bins + 1)]
    counts = np.array([samples_in(edges[i], edges[i + 1]) for i in range(bins)], dtype=np.float64)
    cum = np.concatenate([[0.0], np.cumsum(counts)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        b = int(np.searchsorted(cum, target, side="right")) - 1
        b = min(max(b, 0), bins - 1)
        frac = (target - cum[b]) / counts[b] if counts[b] > 0 else 0.0
        z = int(round(edges[b] + frac * (edges[b + 1] - edges[b])))
        cuts.append(min(max(z, cuts[-1] + 1), V - (world - r)))
    cuts.append(V)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def time_balanced_slabs(samples_in, V: int, slabs, times, bins: int = 64) -> list[tuple[int, int]]:
    """One rebalancing step of z-slabs from measured per-rank step times (decided before the
    timed region): rank r's speed is its samples over its time, every rank is given the samples
    it would finish in the same time at its own speed, and the cuts are placed at those sample
    targets (interpolated in `bins` equal-depth bins, as sample_balanced_slabs). Samples alone
    miss per-rank fixed costs -- e.g. a slab that ends in a thin partial layer of tiles, or
    segments walked by two ranks -- that the times see."""
    world = len(slabs)
    if world < 2:
        return list(slabs)
    edges = [i * V // bins for i in range(bins + 1)]
    counts = np.array([samples_in(edges[i], edges[i + 1]) for i in range(bins)], dtype=np.float64)
    cum = np.concatenate([[0.0], np.cumsum(counts)])
    total = cum[-1]
    work = np.array([max(samples_in(a, b), 1) for a, b in slabs], dtype=np.float64)
    speed = work / np.maximum(np.asarray(times, dtype=np.float64), 1e-9)
    share = speed / speed.sum() * total
    cuts = [0]
    for r in range(1, world):
        target = share[:r].sum()
        b = int(np.searchsorted(cum, target, side="right")) - 1
        b = min(max(b, 0), bins - 1)
        frac = (target - cum[b]) / counts[b] if counts[b] > 0 else 0.0
        z = int(round(edges[b] + frac * (edges[b + 1] - edges[b])))
        cuts.append(min(max(z, cuts[-1] + 1), V - (world - r)))
    cuts.append(V)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def select_slab_segments(ctx, segs_ptr: int, n: int, z_lo: int, z_hi: int, out_ptr: int) -> int:
    """Device-side filter of the z-slab partitioner: copy to `out_ptr` (device, room for n) the
    segments of `segs_ptr` (device) that can reach planes [z_lo, z_hi); returns their count
    (vxg_select_slab_segments). A rank then plans and bins only its slab's segments."""
    import ctypes as C
    k = C.c_int64()
    ctx.check(ctx.lib.vxg_select_slab_segments(ctx.h, segs_ptr, n, z_lo, z_hi, out_ptr, C.byref(k)))
    return k.value


def sample_balanced_cuts(offsets: np.ndarray, world: int) -> np.ndarray:
    """Segment cut points c_0 = 0 <= c_1 <= ... <= c_world = n for a plan's sample offsets
    (n + 1 entries, offsets[n] = capacity): rank r owns segments [c_r, c_{r+1}), whose samples
    are within one segment of capacity / world."""
    off = np.asarray(offsets, dtype=np.int64)
    n = off.shape[0] - 1
    total = int(off[-1])
    targets = (np.arange(world + 1, dtype=np.int64) * total) // world
    cuts = np.searchsorted(off, targets, side="left").astype(np.int64)
    cuts[0], cuts[-1] = 0, n
    return np.minimum(np.maximum.accumulate(cuts), n)


def batch_sample_cuts(batch, world: int) -> np.ndarray:
    """Segment cut points of a planned Batch for `world` ranks, balanced by samples (the list
    configs' partition): rank r owns segments [c_r, c_{r+1})."""
    p = batch.plans()
    off = np.empty(batch.n + 1, np.int64)
    off[:-1] = p["output_offset"]
    off[-1] = batch.capacity
    return sample_balanced_cuts(off, world)


def row_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [a, b) of an n-row array that rank `rank` of `world` uploads (equal slices)."""
    return rank * n // world, (rank + 1) * n // world


def distribute_segments(host_segs: np.ndarray, out, group=None) -> None:
    """Fill the device tensor `out` ((n, 6) float64, on every rank) with all n segments of
    `host_segs` (pinned host memory, the same array content on every rank) moving only 1/world
    of them across each rank's PCIe link: rank r copies its equal slice host->device, then one
    all-gather over the process group (NCCL: NVLink) assembles the whole batch everywhere.
    (gloo, for functional tests: the gather runs through host memory.)"""
    import torch
    dist = _dist()
    n = out.shape[0]
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        out.copy_(torch.from_numpy(host_segs), non_blocking=True)
        return
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if n % world:
        raise ValueError("distribute_segments: the segment count must divide by the world size")
    a, b = row_range(n, world, rank)
    src = torch.from_numpy(host_segs[a:b])
    if dist.get_backend(group) == "nccl":
        mine = out[a:b]
        mine.copy_(src, non_blocking=True)
        dist.all_gather_into_tensor(out, mine.contiguous(), group=group)
    else:
        parts = [torch.empty((b - a, 6), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, src.clone(), group=group)
        out.copy_(torch.cat(parts), non_blocking=True)


_DIGEST_P = (0x9E3779B97F4A7C15, 0xC2B2AE3D27D4EB4F, 0x165667B19E3779F9, 0x27D4EB2F165667C5)


def _signed64(u: int) -> int:
    return u - (1 << 64) if u >= 1 << 63 else u


def list_digest(voxels, chain_off) -> tuple[int, int, int]:
    """Position-sensitive digest of a voxel list slice ((M, 3) int32 device tensor) and its chain
    offsets ((k + 1,) int64, rebased to 0 here): (voxels, sum_j (x P1 + y P2 + z P3) (j + 1),
    sum_i len_i (i + 1) P4), all mod 2^64 (torch int64 arithmetic wraps). Equal lists give equal
    digests; a rank's digest is compared with the same slice of the one-rank list."""
    import torch
    dev = voxels.device
    P = [_signed64(p) for p in _DIGEST_P]
    m = voxels.shape[0]
    h = torch.zeros((), dtype=torch.int64, device=dev)
    step = 1 << 27
    for a in range(0, m, step):
        v = voxels[a:a + step].to(torch.int64)
        j = torch.arange(a + 1, a + 1 + v.shape[0], dtype=torch.int64, device=dev)
        h += ((v[:, 0] * P[0] + v[:, 1] * P[1] + v[:, 2] * P[2]) * j).sum()
    c = chain_off.to(torch.int64)
    ln = c[1:] - c[:-1]
    i = torch.arange(1, ln.shape[0] + 1, dtype=torch.int64, device=dev)
    hc = (ln * i * P[3]).sum()
    return int(m), int(h.item()), int(hc.item())


def words_digest(words) -> int:
    """Position-sensitive digest of a bitmap slice (int64/uint64 words, device tensor):
    sum_i ((w_i xor (i + 1) P2) P1) mod 2^64, computed in chunks."""
    import torch
    P = [_signed64(p) for p in _DIGEST_P]
    w = words.reshape(-1).view(torch.int64)
    h = torch.zeros((), dtype=torch.int64, device=w.device)
    step = 1 << 28
    for a in range(0, w.shape[0], step):
        x = w[a:a + step]
        i = torch.arange(a + 1, a + 1 + x.shape[0], dtype=torch.int64, device=w.device)
        h += (torch.bitwise_xor(x, i * P[1]) * P[0]).sum()
    return int(h.item())


def gather_objects(obj, group=None) -> list:
    """all_gather_object: every rank's small Python object, in rank order."""
    dist = _dist()
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [obj]
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


def _dist():
    import torch.distributed as dist
    return dist


def _device(group=None):
    import torch
    dist = _dist()
    return torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")


def max_over_ranks(value: float, group=None) -> float:
    import torch
    dist = _dist()
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device(group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_floats(value: float, group=None) -> list[float]:
    """Every rank's `value`, in rank order, on every rank."""
    import torch
    dist = _dist()
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [float(value)]
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device(group))
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return [float(x.item()) for x in out]


def sum_over_ranks(value: float, group=None) -> float:
    import torch
    dist = _dist()
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device(group))
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())


def _all_gather_padded(t, group=None):
    """all_gather of 1-D tensors of different lengths -> list of the ranks' tensors."""
    import torch
    dist = _dist()
    world = dist.get_world_size(group)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes)
    pad = torch.zeros(m, dtype=t.dtype, device=t.device)
    pad[: t.numel()] = t
    parts = [torch.zeros(m, dtype=t.dtype, device=t.device) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return [p[:s] for p, s in zip(parts, sizes)]


def gather_bitmap(words, V: int, group=None):
    """Concatenate the ranks' z-slab bitmaps (uint64 words as an int64 tensor of V*V*depth/64
    words, rank order == z order) into the full V^3 bitmap on every rank (verification)."""
    import torch
    if (V * V) % 64:
        raise ValueError("slab gathering needs whole words per plane (V*V % 64 == 0)")
    parts = _all_gather_padded(words.reshape(-1), group)
    return torch.cat(parts)


def gather_list(voxels, chain_off, group=None):
    """Concatenate the ranks' voxel lists ((M_r, 3) int32) and chain offsets ((n_r + 1,) int64,
    each starting at 0) in rank order; offsets are rebased onto the concatenated list."""
    import torch
    vparts = _all_gather_padded(voxels.reshape(-1), group)
    oparts = _all_gather_padded(chain_off.reshape(-1), group)
    base = 0
    offs = []
    for i, o in enumerate(oparts):
        offs.append((o[:-1] if i + 1 < len(oparts) else o) + base)
        base += int(o[-1].item())
    return torch.cat(vparts).reshape(-1, 3), torch.cat(offs)
