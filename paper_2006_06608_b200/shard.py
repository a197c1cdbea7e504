"""Row sharding across ranks.

Each rank owns a contiguous, nnz-balanced range of (renumbered) rows and a
full replica of the input features.  After the rank's aggregation kernel has
written its rows, one all-gather of output rows per layer makes the full
output available on every rank.  Row counts differ per rank, so the
all-gather is over uneven row blocks, issued as one broadcast per owner.
"""
from __future__ import annotations

import warnings

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


BARRIER_TIMEOUT_MS = 120_000  # a peer that never arrives fails the run instead of hanging it


class FusedRowGather:
    """The per-layer all-gather fused into the aggregation (SURVEY §8(e),
    "fused target").  The output y lives in torch symmetric memory, mapped
    into every rank.  Each rank's K3 writes the final values of its own rows
    straight into every replica (gnna_aggregate_fanout):

    * "multimem": with NVLS (NVSwitch multicast), one multimem.st per row
      vector to the multicast address writes all replicas, this rank's
      included;
    * "p2p": otherwise, P2P stores over NVLink into each peer's buffer beside
      the local store.

    Either way the transfer overlaps the gather, and no separate collective
    pass runs.  A stream-ordered symmetric-memory barrier then orders every
    rank's reads after all ranks' kernels.  `create` returns None when
    symmetric memory is unavailable (one rank, gloo/CPU, no P2P), and the
    caller keeps the NCCL `allgather_rows` path.  P2P is the default; the
    NVLS multicast store is opt-in (`multicast=True`)."""

    def __init__(self, y, handle, peers, mc, mode):
        self.y, self.handle, self.peers, self.mc, self.mode = y, handle, peers, mc, mode

    @staticmethod
    def peer_pointers(buffer_ptrs, rank, offset=0):
        """Device pointers of the other ranks' replicas (each rank's buffer
        base + the tensor's byte offset inside it), in rank order."""
        return [int(p) + offset for r, p in enumerate(buffer_ptrs) if r != rank]

    @classmethod
    def create(cls, shape, dtype, device, group=None, multicast=False):
        """(FusedRowGather, None), or (None, why) when the fused path cannot be
        set up here; the caller then keeps the NCCL path and reports `why`."""
        import torch.distributed as dist
        if not dist.is_initialized() or dist.get_world_size(group) < 2:
            return None, "needs an initialised process group of at least 2 ranks"
        if dist.get_world_size(group) - 1 > 7:  # GNNA_MAX_PEERS
            return None, "more than 8 ranks (GNNA_MAX_PEERS = 7 peer replicas)"
        try:
            import torch.distributed._symmetric_memory as symm
            y = symm.empty(*shape, dtype=dtype, device=device)
            h = symm.rendezvous(y, group if group is not None else dist.group.WORLD)
            ptrs = list(h.buffer_ptrs)
            offset = y.data_ptr() - int(ptrs[h.rank])
            if offset < 0:
                return None, "symmetric buffer offset is negative"
            peers = cls.peer_pointers(ptrs, h.rank, offset)
            mc = None
            if multicast:
                has = h.has_multicast_support
                has = has() if callable(has) else has
                if has and int(h.multicast_ptr):
                    mc = int(h.multicast_ptr) + offset
            y.zero_()
            h.barrier(channel=0, timeout_ms=BARRIER_TIMEOUT_MS)
            return cls(y, h, peers, mc, "multimem" if mc else "p2p"), None
        except Exception as exc:  # reported by the caller (config.allgather), never silent
            warnings.warn(f"FusedRowGather: symmetric memory unavailable, keeping NCCL: {exc!r}")
            return None, f"symmetric memory unavailable: {exc!r}"[:300]

    def aggregate(self, plan, x, **opts):
        """This rank's rows into every replica, then the cross-rank barrier.

        The barrier BEFORE the fan-out orders this step's remote stores after
        every rank finished reading the previous step's y (a rank that is
        ahead must not overwrite rows a slower peer still reads, e.g. when y
        feeds the next layer); the barrier AFTER orders every rank's reads
        after all ranks' stores."""
        self.handle.barrier(channel=0, timeout_ms=BARRIER_TIMEOUT_MS)
        if self.mc:
            plan.aggregate_fanout(x, self.y, mc=self.mc, **opts)
        else:
            plan.aggregate_fanout(x, self.y, peers=self.peers, **opts)
        self.handle.barrier(channel=0, timeout_ms=BARRIER_TIMEOUT_MS)
        return self.y

    def verify(self, plan, x, ranges, rank):
        """One fused step against the NCCL path on a separate buffer, on every
        rank; True only if all ranks agree bit for bit (the caller falls back
        to allgather_rows otherwise)."""
        import torch
        import torch.distributed as dist
        ref = torch.zeros_like(self.y)
        plan.aggregate(x, out=ref)
        allgather_rows(ref, ranges, rank)
        self.y.zero_()
        self.handle.barrier(channel=0, timeout_ms=BARRIER_TIMEOUT_MS)
        self.aggregate(plan, x)
        ok = torch.tensor([1 if torch.equal(self.y, ref) else 0], device=self.y.device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        return bool(ok.item())
