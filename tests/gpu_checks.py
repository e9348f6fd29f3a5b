"""Device-side checking helpers for full-size outputs (test infrastructure).

Multi-GB GPU outputs are compared with the oracle through the order-sensitive per-chain hash of
oracle/voxline_oracle.c:vo_chain_hashes, computed here on the GPU with torch (wrapping int64
arithmetic == uint64 mod 2^64).
"""
import numpy as np

from oracle.pyoracle import HASH_P


def _signed(u: int) -> int:
    return int(np.array(u, dtype=np.uint64).astype(np.int64))


def device_chain_hashes(out, chain_off, chunk_voxels: int = 1 << 27):
    """out: int32 cuda tensor (M,3); chain_off: int64 cuda tensor (n+1,). -> (hashes, lengths)
    as uint64 / int64 numpy arrays."""
    import torch
    dev = out.device
    P = torch.tensor([_signed(p) for p in HASH_P], dtype=torch.int64, device=dev)
    n = chain_off.numel() - 1
    lengths = (chain_off[1:] - chain_off[:-1])
    hashes = torch.empty(n, dtype=torch.int64, device=dev)
    off_h = chain_off.cpu().numpy()
    i0 = 0
    while i0 < n:
        # grow the segment range until it holds ~chunk_voxels voxels
        i1 = int(np.searchsorted(off_h, off_h[i0] + chunk_voxels, side="right")) - 1
        i1 = max(min(i1, n), i0 + 1)
        a, b = int(off_h[i0]), int(off_h[i1])
        v = out[a:b].to(torch.int64)
        t = (v * P).sum(1)
        seg = torch.repeat_interleave(torch.arange(i0, i1, device=dev), lengths[i0:i1])
        j = torch.arange(a, b, device=dev, dtype=torch.int64) - chain_off[seg] + 1
        cs = torch.cumsum(t * j, 0)
        cs = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), cs])
        s = chain_off[i0:i1] - a
        e = chain_off[i0 + 1:i1 + 1] - a
        hashes[i0:i1] = cs[e] - cs[s]
        i0 = i1
    return hashes.cpu().numpy().view(np.uint64), lengths.cpu().numpy()
