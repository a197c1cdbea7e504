"""Row-sharded 2-layer GCN training step across ranks.

Rank p owns the contiguous, nnz-balanced renumbered row range [r_p, r_p+1)
(`shard.row_ranges`).  Every layer aggregates only the owner's rows (a plan
over the row slice, `gnna_plan_create(row_begin, row_end)`); the tensors the
NEXT aggregation gathers from are made whole on every rank by one all-gather
of output rows per layer -- fused into the aggregation that produces them
when the communicator offers replicated buffers (gnna_aggregate_fanout: the
K3 flush also stores each finished row into the peers' replicas), else a
separate all-gather.  Weight gradients are row sums: each rank reduces its
own rows and the partials are all-reduced ("an all-gather of
dZ/dH, plus an all-reduce of dW/db").

The step is the C3 shape of `gcn.GCN2` (update-first layer 1 because it
shrinks the width, aggregate-first layer 2; gcn_layer's order rule,
engine.cpp:379-381), with the folded normalisation of GCN2:

  forward   t1  = norm * (x W1)                       all rows (x is replicated:
                                                      recomputing beats an all-gather)
            h1  = relu(norm^2 * (A t1 + ind*t1))      own rows -> all-gather (fused)
            z2  = norm * (A h1 + ind*h1)              own rows
            y   = z2 W2                               own rows
  backward  dz2 = norm * (dy W2^T),  dW2 = z2^T dy    own rows (one fused pass)
            all-gather dz2
            dp1 = norm^2 * (A dz2 + ind*dz2) [h1 > 0] own rows -> all-gather (fused)
            dt1 = norm * (A dp1 + ind*dp1)            own rows
            dW1 = x^T dt1                             own rows
            all-reduce dW1, dW2; SGD

The compute primitives come from an `ops` object and the exchanges from a
`comm` object, so the same orchestration runs on B200s (`GpuOps` over the
C-ABI, `TorchComm` over NCCL + symmetric memory) and, for the CPU tests, on
the oracle with gloo.
"""
from __future__ import annotations

import threading

import torch


class GpuOps:
    """The primitives on one GPU through libgnna (fp32)."""

    def __init__(self, ctx, row_ptr, col, rows, params=None, self_loops=False):
        from .capi import WARP_SHARED
        self.ctx = ctx
        self.n = row_ptr.numel() - 1
        self.rows = rows
        if params is None:
            params, _ = ctx.b200_params(row_ptr, 16)
        self.plan = ctx.plan(row_ptr, col, params, WARP_SHARED, rows=rows)
        norm, _, rs2, ind = ctx.gcn_fold_weights(row_ptr, col, self_loops)
        self.norm = norm                                   # f64: the GEMM row-scale epilogue
        self.rs = norm.float().contiguous()
        self.rs2 = rs2
        self.ind = ind if self_loops else None

    def gemm(self, a, w, scale=None):
        return self.ctx.gemm(a, w, None, 2, scale) if scale is not None else self.ctx.gemm(a, w)

    def agg(self, x, out, scale, relu=False, mask=None, peers=None):
        """Own rows of scale * (A x + ind * x) [relu] [mask] into out (and
        into every peer replica when `peers` is given)."""
        rs = self.rs2 if scale == "norm2" else self.rs
        if peers is not None:
            self.plan.aggregate_fanout(x, out, peers=peers, self_weight=self.ind, row_scale=rs, relu=relu,
                                       mask=mask)
        else:
            self.plan.aggregate_ex(x, out=out, self_weight=self.ind, row_scale=rs, relu=relu, mask=mask)
        return out

    def dense_backward(self, dy, w, z):
        r0, r1 = self.rows
        return self.ctx.dense_backward(dy, w, z, self.norm[r0:r1].contiguous())

    def gemm_tn(self, a, b):
        from .gcn import ctx_gemm_tn
        return ctx_gemm_tn(self.ctx, a, b)

    def empty(self, shape, like):
        return torch.empty(shape, dtype=like.dtype, device=like.device)


class ShardedGCN2:
    """One rank's share of the 2-layer GCN step (see the module docstring)."""

    def __init__(self, ops, comm, w1, w2, lr=0.01):
        self.ops, self.comm = ops, comm
        self.w1, self.w2, self.lr = w1, w2, lr
        self.n = ops.n
        self.r0, self.r1 = ops.rows
        hid, out_dim = w2.shape
        if not (hid < w1.shape[0] and out_dim >= hid):
            raise ValueError("ShardedGCN2 runs the C3 layer order: in > hidden <= out")
        # replicated activations (all-gathered every step) and a full-size scratch
        self.h1 = comm.replicated("h1", (self.n, hid), w1)
        self.dp1 = comm.replicated("dp1", (self.n, hid), w1)
        self.dz2 = comm.replicated("dz2", (self.n, hid), w1)
        self.z2 = ops.empty((self.n, hid), w1)
        self.dt1 = ops.empty((self.n, hid), w1)

    def step(self, x, dy_own):
        """x: all n rows (replicated input); dy_own: this rank's rows of the
        upstream gradient.  Returns (y_own, dW1, dW2) after the SGD update."""
        ops, comm, r0, r1 = self.ops, self.comm, self.r0, self.r1
        t1 = ops.gemm(x, self.w1, ops.norm)                             # norm * (x W1), all rows
        comm.fill(self.h1, lambda out, peers: ops.agg(t1, out, "norm2", relu=True, peers=peers))
        ops.agg(self.h1.local, self.z2, "norm")                         # own rows
        z2_own = self.z2[r0:r1]
        y_own = ops.gemm(z2_own, self.w2)
        dz2_own, dw2 = ops.dense_backward(dy_own, self.w2, z2_own)      # norm * (dY W2^T), z2^T dY
        self.dz2.local[r0:r1] = dz2_own
        comm.allgather(self.dz2)
        comm.fill(self.dp1, lambda out, peers: ops.agg(self.dz2.local, out, "norm2", mask=self.h1.local,
                                                       peers=peers))
        ops.agg(self.dp1.local, self.dt1, "norm")
        dw1 = ops.gemm_tn(x[r0:r1], self.dt1[r0:r1])
        comm.allreduce(dw1)
        comm.allreduce(dw2)
        self.w1 -= self.lr * dw1
        self.w2 -= self.lr * dw2
        return y_own, dw1, dw2


# ------------------------------------------------------------ communicators
class Replica:
    """A rank's copy of a replicated tensor (`local`), the other ranks'
    copies it may store into (`peers`: pointers or tensors, for the fused
    fan-out), and the owner's row range."""

    def __init__(self, local, peers=None, handle=None):
        self.local, self.peers, self.handle = local, peers, handle


class TorchComm:
    """torch.distributed: the all-gather fused into the aggregation through
    symmetric memory when `fused` (NCCL + FusedRowGather), else one broadcast
    per owner (NCCL or gloo); all-reduce of the weight gradients."""

    def __init__(self, ranges, rank, fused=True):
        self.ranges, self.rank, self.fused = ranges, rank, fused
        self.notes = {}

    def replicated(self, name, shape, like):
        if self.fused and like.is_cuda:
            from .shard import FusedRowGather
            g, why = FusedRowGather.create(shape, like.dtype, like.device)
            if g is not None:
                return Replica(g.y, g.peers, g)
            self.notes[name] = why
        return Replica(torch.zeros(shape, dtype=like.dtype, device=like.device))

    def fill(self, rep, produce):
        """Runs produce(out, peers) for this rank's rows, then makes the
        other ranks' rows present (fused: barriers around the fan-out)."""
        if rep.handle is not None:
            from .shard import BARRIER_TIMEOUT_MS
            rep.handle.handle.barrier(channel=0, timeout_ms=BARRIER_TIMEOUT_MS)  # peers done reading
            produce(rep.local, rep.peers)
            rep.handle.handle.barrier(channel=0, timeout_ms=BARRIER_TIMEOUT_MS)  # every row stored
        else:
            produce(rep.local, None)
            self.allgather(rep)

    def allgather(self, rep):
        from .shard import allgather_rows
        allgather_rows(rep.local, self.ranges, self.rank)

    def allreduce(self, t):
        import torch.distributed as dist
        dist.all_reduce(t)


class ThreadGroup:
    """N ranks as threads of ONE process on one GPU (tests): each rank has
    its own CUDA stream and context; replicated tensors are N local buffers
    and the fused fan-out stores into the other ranks' buffers exactly as
    it would over NVLink.  Collectives synchronise the ranks' streams and a
    thread barrier; the all-reduce sums the partials in rank order."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.bufs = {}
        self.lock = threading.Lock()
        self.slots = {}

    def comm(self, rank, ranges, stream):
        return _ThreadComm(self, rank, ranges, stream)


class _ThreadComm:
    def __init__(self, group, rank, ranges, stream):
        self.g, self.rank, self.ranges, self.stream = group, rank, ranges, stream

    def _sync(self):
        self.stream.synchronize()
        self.g.barrier.wait()

    def replicated(self, name, shape, like):
        with self.g.lock:
            if name not in self.g.bufs:
                self.g.bufs[name] = [torch.zeros(shape, dtype=like.dtype, device=like.device)
                                     for _ in range(self.g.world)]
        self._sync()
        bufs = self.g.bufs[name]
        return Replica(bufs[self.rank], [b for r, b in enumerate(bufs) if r != self.rank], handle=name)

    def fill(self, rep, produce):
        self._sync()                     # peers done reading the previous contents
        produce(rep.local, rep.peers)    # own rows into every replica (fused fan-out)
        self._sync()                     # every rank's rows stored

    def allgather(self, rep):
        a, b = self.ranges[self.rank]
        self._sync()
        with torch.cuda.stream(self.stream):
            for peer in rep.peers:
                peer[a:b].copy_(rep.local[a:b])
        self._sync()

    def allreduce(self, t):
        key = ("ar", id(self.g.barrier), t.shape)
        self._sync()
        with self.g.lock:
            self.g.slots.setdefault(key, [None] * self.g.world)[self.rank] = t.clone()
        self._sync()
        parts = self.g.slots[key]
        with torch.cuda.stream(self.stream):
            total = parts[0].clone()
            for p in parts[1:]:
                total += p                # rank order: every rank gets the same bits
            t.copy_(total)
        self._sync()
        with self.g.lock:
            self.g.slots.pop(key, None)
        self._sync()
