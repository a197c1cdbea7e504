"""The row-sharded 2-layer GCN step (paper_2006_06608_b200/sharded.py) on
the GPU kernels, with two ranks as threads of one process on one B200
(sharded.ThreadGroup): each rank has its own stream and gnna context, a
plan over its row slice, and its aggregations store their rows into the
OTHER rank's replica through the fused fan-out (gnna_aggregate_fanout, node
weights included) exactly as over NVLink.  Two SGD steps must match the
unsharded GCN2 step (one plan over all rows) on the same inputs: output
rows, dW1, dW2 at the fp32 error-aware bar (they differ only by summation
order: per-rank partial row sums + the all-reduce)."""
import threading

import numpy as np
import pytest
import torch

from conftest import to_dev

pytestmark = pytest.mark.gpu


def close(got, want, rtol=1e-5):
    got, want = got.double().cpu(), want.double().cpu()
    scale = want.abs().max().item()
    return bool(((got - want).abs() <= rtol * (want.abs() + 1e-2 * scale)).all()), float((got - want).abs().max())


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
    ref = GCN2(ctx, drp, dcol, 96, 16, 22, lr=0.05)
    w1, w2 = ref.w1.clone(), ref.w2.clone()
    want = []
    for _ in range(2):
        y, dw1, dw2 = ref.step(x, dy)
        want.append((y.clone(), dw1.clone(), dw2.clone()))
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
        for r in range(2):
            a, b = ranges[r]
            y_own, g1, g2 = got[r][step]
            for g, wv, name in ((y_own, wy[a:b], "y"), (g1, wd1, "dW1"), (g2, wd2, "dW2")):
                ok, err = close(g, wv)
                assert ok, (step, r, name, err)
        assert torch.equal(got[0][step][1], got[1][step][1])  # the all-reduce gives every rank the same bits
