"""GPU: the all-gather fused into the aggregation (gnna_aggregate_fanout,
SURVEY §8(e) "fused target").  On one GPU the "peer replicas" are local
buffers, which exercises the kernel side exactly: every final row value of
the rank's row-slice plan lands in y and in each replica at the same offset,
rows outside the slice are never written, epilogues apply to every copy, and
the fan-out instantiations give the same bits as the plain K3.
"""
import numpy as np
import pytest
import torch

from conftest import random_graph, to_dev

pytestmark = pytest.mark.gpu


def powerlaw(orc, rng, n, e, a=0.9):
    w = 1.0 / np.arange(1, n + 1) ** a
    src = rng.choice(n, size=e, p=w / w.sum())
    edges = np.stack([src, rng.integers(0, n, size=e)], 1).astype(np.uint32)
    return orc.to_csr(n, edges, True)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_fanout_writes_slice_rows_to_every_replica(ctx, orc, dtype):
    from paper_2006_06608_b200.capi import Params
    rng = np.random.default_rng(31)
    for trial in range(6):
        n = int(rng.integers(50, 5000))
        rp, col = powerlaw(orc, rng, n, 8 * n) if trial % 2 else random_graph(rng, n, 5 * n, orc=orc)[:2]
        drp, dcol = to_dev(rp, col)
        dim = int(rng.choice([4, 16, 22, 64, 128]))
        r0 = int(rng.integers(0, n // 2))
        r1 = int(rng.integers(r0, n + 1))
        p = Params.make(ngs=int(rng.choice([4, 16, 64])), dw=32, tpb=int(rng.choice([128, 256, 512])), dim=dim)
        plan = ctx.plan(drp, dcol, p, rows=(r0, r1))
        x = torch.tensor(rng.random((n, dim)) - 0.4, dtype=dtype, device="cuda")
        want = torch.full((n, dim), 7.0, dtype=dtype, device="cuda")
        plan.aggregate(x, out=want)
        sentinel = -3.25
        y = torch.full((n, dim), sentinel, dtype=dtype, device="cuda")
        peers = [torch.full((n, dim), sentinel, dtype=dtype, device="cuda") for _ in range(int(rng.integers(1, 8)))]
        plan.aggregate_fanout(x, y, peers=peers)
        torch.cuda.synchronize()
        for buf in [y] + peers:
            assert torch.equal(buf[r0:r1], want[r0:r1]), (trial, dim, r0, r1)  # same bits as the plain K3
            assert bool((buf[:r0] == sentinel).all()) and bool((buf[r1:] == sentinel).all())


def test_fanout_epilogues_and_limits(ctx, orc):
    from paper_2006_06608_b200.capi import DomainError, Params
    rng = np.random.default_rng(5)
    n = 3000
    rp, col = powerlaw(orc, rng, n, 10 * n)
    drp, dcol = to_dev(rp, col)
    p = Params.make(ngs=16, dw=32, tpb=256, dim=32)
    plan = ctx.plan(drp, dcol, p, rows=(100, 2500))
    x = torch.tensor(rng.random((n, 32)) - 0.5, dtype=torch.float32, device="cuda")
    rs = torch.tensor(rng.random(n), dtype=torch.float32, device="cuda")
    want = torch.zeros((n, 32), device="cuda")
    plan.aggregate_ex(x, out=want, alpha=1.1, row_scale=rs, relu=True)
    y = torch.zeros((n, 32), device="cuda")
    peers = [torch.zeros((n, 32), device="cuda") for _ in range(3)]
    plan.aggregate_fanout(x, y, peers=peers, alpha=1.1, row_scale=rs, relu=True)
    for buf in [y] + peers:
        assert torch.equal(buf, want)
    with pytest.raises(ValueError):
        plan.aggregate_fanout(x, y, peers=[torch.zeros_like(y) for _ in range(8)])
    with pytest.raises(DomainError):
        plan.aggregate_fanout(x, y, peers=[0])  # null replica


def test_fanout_with_node_weights(ctx, orc):
    """The GCN gather (per-source norm[u], self weight, row scale) fused with
    the all-gather: every replica gets the plain weighted K3's bits."""
    from paper_2006_06608_b200.capi import Params
    rng = np.random.default_rng(12)
    n = 4000
    rp, col = powerlaw(orc, rng, n, 12 * n)
    drp, dcol = to_dev(rp, col)
    for dim, r0, r1 in ((16, 0, 2100), (64, 700, 4000), (128, 1, 3999)):
        plan = ctx.plan(drp, dcol, Params.make(ngs=16, dw=32, tpb=256, dim=dim), rows=(r0, r1))
        x = torch.tensor(rng.random((n, dim)), dtype=torch.float32, device="cuda")
        rs, sw, _ = ctx.gcn_weights(drp, dcol, True, edge_weights=False)
        want = torch.zeros((n, dim), device="cuda")
        plan.aggregate_ex(x, out=want, node_weight=rs, self_weight=sw, row_scale=rs)
        y = torch.zeros((n, dim), device="cuda")
        peers = [torch.zeros((n, dim), device="cuda") for _ in range(2)]
        plan.aggregate_fanout(x, y, peers=peers, node_weight=rs, self_weight=sw, row_scale=rs)
        for buf in [y] + peers:
            assert torch.equal(buf[r0:r1], want[r0:r1]), dim
    # rows wider than one chunk per lane (tpb 512 caps teams at 16 lanes: d 128 is two chunks): the
    # per-edge weighted fan-out does not exist there, the pre-scaled gather (>= 4 edges per row) does
    import os
    from paper_2006_06608_b200.capi import DomainError
    plan = ctx.plan(drp, dcol, Params.make(ngs=16, dw=32, tpb=512, dim=128))
    x = torch.rand((n, 128), device="cuda")
    want = plan.aggregate_ex(x, node_weight=rs)
    if os.environ.get("GNNA_PRESCALE") == "0":
        with pytest.raises(DomainError):
            plan.aggregate_fanout(x, torch.zeros_like(x), peers=[torch.zeros_like(x)], node_weight=rs)
    else:
        y, peer = torch.zeros_like(x), torch.zeros_like(x)
        plan.aggregate_fanout(x, y, peers=[peer], node_weight=rs)
        assert torch.equal(y, want) and torch.equal(peer, want)
