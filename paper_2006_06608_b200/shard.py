"""Row sharding across ranks.

Each rank owns a contiguous, nnz-balanced range of (renumbered) rows and a
full replica of the input features.  After the rank's aggregation kernel has
written its rows, one all-gather of output rows per layer makes the full
output available on every rank.  Row counts differ per rank, so the
all-gather is over uneven row blocks, issued as one broadcast per owner.
"""
from __future__ import annotations

import numpy as np


def row_ranges(row_ptr_host, parts: int, community_starts=None, tol=0.01):
    """Contiguous row ranges with ~equal nnz: rank p starts at the first row
    whose CSR offset reaches nnz*p/parts (binary search on row_ptr).

    community_starts (sorted first rows of the renumbered communities, i.e.
    the exclusive scan of community sizes after build_mapping) snaps each cut
    to the nearest community boundary whose edge offset lies within
    tol*nnz of the balanced cut, so a community stays on one rank when that
    costs at most 1% of balance."""
    rp = np.asarray(row_ptr_host)
    n = len(rp) - 1
    nnz = int(rp[-1])
    starts = np.asarray(community_starts, dtype=np.int64) if community_starts is not None else None
    cuts = [0]
    for p in range(1, parts):
        target = nnz * p / parts
        c = int(np.searchsorted(rp, target, side="left"))
        if starts is not None and len(starts):
            k = int(np.searchsorted(starts, c))
            best = None
            for s in (starts[k - 1] if k > 0 else None, starts[k] if k < len(starts) else None):
                if s is None or not (0 <= s <= n):
                    continue
                dev = abs(float(rp[s]) - target)
                if dev <= tol * nnz and (best is None or dev < best[0]):
                    best = (dev, int(s))
            if best is not None:
                c = best[1]
        cuts.append(c)
    cuts.append(n)
    cuts = [min(max(c, 0), n) for c in cuts]
    for i in range(1, len(cuts)):
        cuts[i] = max(cuts[i], cuts[i - 1])
    return [(cuts[i], cuts[i + 1]) for i in range(parts)]


def allgather_rows(y, ranges, rank, group=None):
    """All-gather of uneven output row blocks into every rank's full `y`, in
    place: one broadcast per owner rank (each block is a contiguous row
    slice, so no staging copy; NCCL and gloo both accept it)."""
    import torch.distributed as dist
    for p, (a, b) in enumerate(ranges):
        if b > a:
            dist.broadcast(y[a:b], src=p, group=group)
    return y
