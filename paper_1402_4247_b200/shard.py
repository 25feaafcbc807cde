"""Multi-GPU grid sharding: contiguous, cost-balanced block
ranges. Mirrors kb_api.cu:shard() exactly (same +1-per-block weights, same
lower-bound search), so host code and tests can predict each rank's range.
"""
from __future__ import annotations

import numpy as np


def partition(block_cost: np.ndarray, nranks: int) -> list[tuple[int, int]]:
    """Split blocks [0, nblock) into nranks contiguous ranges with balanced
    sum(cost + 1). Range r = [bound(r), bound(r+1)), bound(r) = first block b
    whose prefix weight * nranks >= total * r."""
    w = [int(c) + 1 for c in np.asarray(block_cost)]
    pre = [0]
    for x in w:
        pre.append(pre[-1] + x)
    nb = len(w)

    def bound(r):
        if r <= 0:
            return 0
        if r >= nranks:
            return nb
        lo, hi = 0, nb
        while lo < hi:  # first b with pre[b] * nranks >= total * r (exact integers)
            mid = (lo + hi) // 2
            if pre[mid] * nranks < pre[nb] * r:
                lo = mid + 1
            else:
                hi = mid
        return lo

    return [(bound(r), bound(r + 1)) for r in range(nranks)]


def block_costs(index: dict, norb_of_atom: np.ndarray) -> np.ndarray:
    """Per-block cost = sum over canonical cover pairs (ci <= cj) sharing points
    of ceil8(n_a) * ceil8(n_b) * 4 * (1x2x2 quads of mask_ci & mask_cj): the padded
    tile work of the DMMA kernels (the device's blk_cost, kb_index.cu:k_bp_count)."""
    bp, ca, cm = index["blk_ptr"], index["cov_atom"], index["cov_mask"].astype(np.uint64)
    out = np.zeros(index["nblock"], dtype=np.int64)
    for b in range(index["nblock"]):
        c0, c1 = bp[b], bp[b + 1]
        tot = 0
        for i in range(c0, c1):
            ni = int(norb_of_atom[ca[i]])
            for j in range(i, c1):
                both = int(cm[i]) & int(cm[j])
                if both:
                    nq = sum(1 for q in range(16) if (both >> (4 * q)) & 0xF)
                    nj = int(norb_of_atom[ca[j]])
                    tot += ((ni + 7) & ~7) * ((nj + 7) & ~7) * 4 * nq
        out[b] = tot
    return out
