"""The row-sharded 2-layer GCN step (paper_2006_06608_b200/sharded.py) on
the GPU kernels, with two ranks as threads of one process on one B200
(sharded.ThreadGroup): each rank has its own stream and gnna context, a
plan over its row slice, and its aggregations store their rows into the
OTHER rank's replica through the fused fan-out (gnna_aggregate_fanout, node
weights included) exactly as over NVLink.  Two SGD steps must match the
unsharded GCN2 step (one plan over all rows) on the same inputs: output
rows, dW1, dW2 at the fp32 error-aware bar (they differ only by summation
order: per-rank partial row sums + the all-reduce)."""
import os
import sys
import threading

import numpy as np
import pytest
import torch

from conftest import ROOT, to_dev

if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu


def close(got, want, bound, rtol=2e-5):
    """Both sides are fp32 computations of the same value, each within the
    1e-5 error-aware bar of it: |got - want| <= 2e-5 (|want| + sum|terms|)."""
    got, want, bound = got.double().cpu(), want.double().cpu(), bound.double().cpu()
    lim = rtol * (want.abs() + bound)
    return bool(((got - want).abs() <= lim + 1e-30).all()), float(((got - want).abs() / (lim + 1e-30)).max())


def test_sharded_gcn2_two_ranks_one_gpu(ctx, orc):
    from paper_2006_06608_b200.capi import Context
    from paper_2006_06608_b200.gcn import GCN2
    from paper_2006_06608_b200.shard import row_ranges
    from paper_2006_06608_b200.sharded import GpuOps, ShardedGCN2, ThreadGroup
    rng = np.random.default_rng(8)
    n = 30000
    w = 1.0 / np.arange(1, n + 1) ** 0.9
    src = rng.choice(n, size=180000, p=w / w.sum())
    edges = np.stack([src, rng.integers(0, n, 180000)], 1).astype(np.uint32)
    rp, col = orc.to_csr(n, edges, True)
    drp, dcol = to_dev(rp, col)
    x = to_dev((rng.random((n, 96)) - 0.5).astype(np.float32))
    dy = to_dev((rng.random((n, 22)) - 0.5).astype(np.float32))
    import bench
    ref = GCN2(ctx, drp, dcol, 96, 16, 22, lr=0.05)
    w1, w2 = ref.w1.clone(), ref.w2.clone()
    want, bounds = [], []
    for _ in range(2):
        wa, wb = ref.w1.clone(), ref.w2.clone()
        y, dw1, dw2 = ref.step(x, dy)
        want.append((y.clone(), dw1.clone(), dw2.clone()))
        mask = (ref.saved["h1"] > 0).double()
        _, (by, bdw1, bdw2, _) = bench.gcn2_reference(drp, dcol, n, x, wa, wb, dy, mask)  # sum-of-|terms| bounds
        bounds.append((by, bdw1, bdw2))
    torch.cuda.synchronize()

    ranges = row_ranges(rp, 2)
    group = ThreadGroup(2)
    got, errors = [None, None], []

    def rank(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                c = Context(0, s)
                ops = GpuOps(c, drp, dcol, ranges[r], params=ref.params)
                model = ShardedGCN2(ops, group.comm(r, ranges, s), w1.clone(), w2.clone(), lr=0.05)
                a, b = ranges[r]
                out = []
                for _ in range(2):
                    y_own, g1, g2 = model.step(x, dy[a:b].contiguous())
                    out.append((y_own.clone(), g1.clone(), g2.clone()))
                s.synchronize()
                got[r] = out
        except BaseException as exc:  # surfaced below
            errors.append(repr(exc))
            group.barrier.abort()

    th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    for step in range(2):
        wy, wd1, wd2 = want[step]
        by, bd1, bd2 = bounds[step]
        for r in range(2):
            a, b = ranges[r]
            y_own, g1, g2 = got[r][step]
            for g, wv, bv, name in ((y_own, wy[a:b], by[a:b], "y"), (g1, wd1, bd1, "dW1"), (g2, wd2, bd2, "dW2")):
                ok, err = close(g, wv, bv)
                assert ok, (step, r, name, err)
        assert torch.equal(got[0][step][1], got[1][step][1])  # the all-reduce gives every rank the same bits
