"""Row sharding across ranks.

Each rank owns a contiguous, nnz-balanced range of (renumbered) rows and a
full replica of the input features.  After the rank's aggregation kernel has
written its rows, one all-gather of output rows per layer makes the full
output available on every rank.  Row counts differ per rank, so the
all-gather is over uneven row blocks, issued as one broadcast per owner.
"""
from __future__ import annotations

import numpy as np


def row_ranges(row_ptr_host, parts: int):
    """Contiguous row ranges with ~equal nnz: rank p starts at the first row
    whose CSR offset reaches nnz*p/parts (binary search on row_ptr)."""
    rp = np.asarray(row_ptr_host)
    n = len(rp) - 1
    nnz = int(rp[-1])
    cuts = [0]
    for p in range(1, parts):
        cuts.append(int(np.searchsorted(rp, nnz * p / parts, side="left")))
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
