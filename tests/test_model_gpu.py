"""GPU: the fused aggregation options (gnna_aggregate_ex) and the 2-layer GCN
training step (paper_2006_06608_b200/gcn.py) built on them.

* aggregate_ex: per-edge weights, self weights, row scale, ReLU and the
  ReLU-backward mask, at widths other than the plan's, on power-law graphs
  whose hubs span many schedule blocks (carry path), vs an fp64 numpy
  restatement; fp32 bar 1e-5 relative to sum|terms|.
* GCN2: forward vs two REFERENCE-semantics gcn_layer calls (oracle, fp64) with
  a ReLU between; full step gradients vs torch float64 autograd.
"""
import numpy as np
import pytest
import torch

from conftest import random_graph, to_dev

pytestmark = pytest.mark.gpu


def powerlaw_graph(orc, rng, n, e, a=0.8):
    w = 1.0 / np.arange(1, n + 1) ** a
    src = rng.choice(n, size=e, p=w / w.sum())
    edges = np.stack([src, rng.integers(0, n, size=e)], 1).astype(np.uint32)
    return orc.to_csr(n, edges, True)


def ref_agg(rp, col, x, ew=None, sw=None, alpha=0.0, rs=None, relu=False, mask=None):
    n = len(rp) - 1
    y = np.zeros_like(x, dtype=np.float64)
    bound = np.zeros_like(y)
    for v in range(n):
        nb = col[rp[v]:rp[v + 1]]
        w = ew[nb].astype(np.float64) if ew is not None else np.ones(len(nb))  # per source node
        y[v] = (w[:, None] * x[nb]).sum(0)
        bound[v] = (np.abs(w)[:, None] * np.abs(x[nb])).sum(0)
        c = sw[v] if sw is not None else alpha
        y[v] += c * x[v]
        bound[v] += abs(c) * np.abs(x[v])
        if rs is not None:
            y[v] *= rs[v]
            bound[v] *= abs(rs[v])
    if relu:
        y = np.maximum(y, 0)
    if mask is not None:
        y = np.where(mask > 0, y, 0)
    return y, bound


def test_aggregate_ex_options(ctx, orc):
    from paper_2006_06608_b200.capi import Params
    rng = np.random.default_rng(40)
    for t in range(8):
        n = int(rng.integers(50, 6000))
        rp, col = powerlaw_graph(orc, rng, n, 6 * n)
        drp, dcol = to_dev(rp, col)
        plan_dim = int(rng.choice([16, 64]))
        p = Params.make(ngs=int(rng.choice([4, 16, 64])), dw=32, tpb=int(rng.choice([64, 128, 256])), dim=plan_dim)
        plan = ctx.plan(drp, dcol, p, 2)
        for dim in (16, 22, 64, 3):
            x = rng.random((n, dim)) - 0.3
            ew = rng.random(n).astype(np.float32)  # node weights
            sw = (rng.random(n) * (rng.random(n) < 0.5)).astype(np.float32)
            rs = rng.random(n).astype(np.float32)
            mask = rng.random((n, dim)) - 0.5
            dx = to_dev(x.astype(np.float32))
            opts = [dict(), dict(ew=ew), dict(ew=ew, sw=sw, rs=rs), dict(alpha=1.5), dict(ew=ew, rs=rs, relu=True),
                    dict(sw=sw, mask=mask)]
            for o in opts:
                want, bound = ref_agg(rp, col, x.astype(np.float32).astype(np.float64), o.get("ew"), o.get("sw"),
                                      o.get("alpha", 0.0), o.get("rs"), o.get("relu", False), o.get("mask"))
                got = plan.aggregate_ex(dx, node_weight=to_dev(o["ew"]) if "ew" in o else None,
                                        self_weight=to_dev(o["sw"]) if "sw" in o else None,
                                        alpha=o.get("alpha", 0.0), row_scale=to_dev(o["rs"]) if "rs" in o else None,
                                        relu=o.get("relu", False),
                                        mask=to_dev(o["mask"].astype(np.float32)) if "mask" in o else None)
                got = got.cpu().numpy().astype(np.float64)
                err = np.abs(got - want)
                assert (err <= 1e-5 * (bound + np.abs(want)) + 1e-30).all(), (t, dim, list(o), float(err.max()))


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_torch_autograd_layers(ctx, orc, dtype):
    """GCNConv / GINConv (torch.autograd over the C-ABI layer entry points)
    vs the same model written with dense torch ops, float64 autograd."""
    from paper_2006_06608_b200.torch_ops import GCNConv, GINConv
    rng = np.random.default_rng(12)
    n = 400
    rp, col = powerlaw_graph(orc, rng, n, 1500)
    drp, dcol = to_dev(rp, col)
    torch.manual_seed(0)
    l1 = GCNConv(ctx, 24, 16, self_loops=True, dtype=dtype)
    l2 = GINConv(ctx, 16, 8, eps=0.2, dtype=dtype)
    with torch.no_grad():
        l2.bias.uniform_(-0.2, 0.2)
    x = torch.tensor(rng.random((n, 24)) - 0.5, dtype=dtype, device="cuda", requires_grad=True)
    y = l2(drp, dcol, torch.relu(l1(drp, dcol, x)))
    g = torch.tensor(rng.random((n, 8)) - 0.5, dtype=dtype, device="cuda")
    y.backward(g)
    # dense float64 twin
    An = torch.tensor(dense_norm_adj(rp, col, True), dtype=torch.float64)
    A = torch.zeros((n, n), dtype=torch.float64)
    for v in range(n):
        A[v, torch.from_numpy(col[rp[v]:rp[v + 1]].astype(np.int64))] = 1.0
    X = x.detach().double().cpu().requires_grad_(True)
    W1 = l1.weight.detach().double().cpu().requires_grad_(True)
    W2 = l2.weight.detach().double().cpu().requires_grad_(True)
    B2 = l2.bias.detach().double().cpu().requires_grad_(True)
    H = torch.relu(An @ X @ W1)
    Y = torch.relu((A @ H + 1.2 * H) @ W2 + B2)
    Y.backward(g.double().cpu())
    if dtype == torch.float64:
        tol = dict(rtol=1e-9, atol=1e-11)
        np.testing.assert_allclose(y.detach().double().cpu().numpy(), Y.detach().numpy(), **tol)
        for got, ref in ((x.grad, X.grad), (l1.weight.grad, W1.grad), (l2.weight.grad, W2.grad),
                         (l2.bias.grad, B2.grad)):
            r = ref.numpy()
            np.testing.assert_allclose(got.double().cpu().numpy(), r, rtol=tol["rtol"],
                                       atol=tol["atol"] * max(1, np.abs(r).max()))
        return
    # fp32: error-aware 1e-5 bar; the bound is the same network on |inputs| with
    # every ReLU open (sum of |terms|), its gradients by float64 autograd as well
    Xb = X.detach().abs().requires_grad_(True)
    W1b, W2b, B2b = (t.detach().abs().requires_grad_(True) for t in (W1, W2, B2))
    Hb = An.abs() @ Xb @ W1b
    Yb = (A @ Hb + 1.2 * Hb) @ W2b + B2b
    Yb.backward(g.double().cpu().abs())
    assert_close_bound(y.detach(), Y.detach(), Yb.detach(), "y")
    for got, ref, bnd, nm in ((x.grad, X.grad, Xb.grad, "dx"), (l1.weight.grad, W1.grad, W1b.grad, "dW1"),
                              (l2.weight.grad, W2.grad, W2b.grad, "dW2"), (l2.bias.grad, B2.grad, B2b.grad, "db2")):
        assert_close_bound(got, ref, bnd, nm)


def assert_close_bound(got, want, bound, what, rtol=1e-5):
    """|got - want| <= rtol * (|want| + bound), bound = sum of |terms|."""
    got = got.double().cpu().numpy() if torch.is_tensor(got) else np.asarray(got, np.float64)
    want = want.double().cpu().numpy() if torch.is_tensor(want) else np.asarray(want, np.float64)
    bound = bound.double().cpu().numpy() if torch.is_tensor(bound) else np.asarray(bound, np.float64)
    err = np.abs(got - want)
    lim = rtol * (np.abs(want) + bound) + 1e-30
    assert (err <= lim).all(), (what, float((err / lim).max()))


def dense_norm_adj(rp, col, self_loops):
    n = len(rp) - 1
    A = np.zeros((n, n))
    for v in range(n):
        A[v, col[rp[v]:rp[v + 1]]] = 1.0
    if self_loops:
        for v in range(n):
            if A[v, v] == 0:
                A[v, v] = 1.0
    deg = np.maximum(A.sum(1), 1)
    d = 1 / np.sqrt(deg)
    return d[:, None] * A * d[None, :]


@pytest.mark.parametrize("dims,sl", [((96, 16, 22), False), ((12, 32, 8), True), ((20, 16, 16), False),
                                     ((24, 16, 16), True), ((40, 16, 8), True), ((24, 16, 8), False)])
def test_gcn2_step_vs_autograd_and_reference(ctx, orc, dims, sl):
    from paper_2006_06608_b200.gcn import GCN2
    rng = np.random.default_rng(sum(dims))
    n = 700
    rp, col = powerlaw_graph(orc, rng, n, 3000)
    drp, dcol = to_dev(rp, col)
    din, hid, dout = dims
    model = GCN2(ctx, drp, dcol, din, hid, dout, self_loops=sl, lr=0.0)
    x = (rng.random((n, din)) - 0.5).astype(np.float32)
    dy = (rng.random((n, dout)) - 0.5).astype(np.float32)
    w1, w2 = model.w1.double().cpu().numpy(), model.w2.double().cpu().numpy()
    y, dw1, dw2 = model.step(to_dev(x), to_dev(dy))
    # reference semantics: gcn_layer (oracle, fp64) twice with a ReLU between
    x64 = x.astype(np.float64)
    h1 = np.maximum(orc.gcn_layer(rp, col, x64, w1, sl), 0)
    want = orc.gcn_layer(rp, col, h1, w2, sl)
    bh1 = orc.gcn_layer(rp, col, np.abs(x64), np.abs(w1), sl)
    assert_close_bound(y, want, orc.gcn_layer(rp, col, bh1, np.abs(w2), sl), "y")
    # gradients: torch float64 autograd; bound: the same on |inputs|, ReLU open
    An = torch.tensor(dense_norm_adj(rp, col, sl))
    W1 = torch.tensor(w1, requires_grad=True)
    W2 = torch.tensor(w2, requires_grad=True)
    X = torch.tensor(x, dtype=torch.float64)
    Y = An @ torch.relu(An @ X @ W1) @ W2
    Y.backward(torch.tensor(dy, dtype=torch.float64))
    W1b = W1.detach().abs().requires_grad_(True)
    W2b = W2.detach().abs().requires_grad_(True)
    Yb = An @ (An @ X.abs() @ W1b) @ W2b
    Yb.backward(torch.tensor(np.abs(dy), dtype=torch.float64))
    for got, ref, bnd, nm in ((dw1, W1.grad, W1b.grad, "dW1"), (dw2, W2.grad, W2b.grad, "dW2")):
        assert_close_bound(got, ref, bnd, nm)


def test_gcn2_step_cuda_graph_replay(ctx, orc):
    """The whole training step (libgnna launches through the C-ABI, their
    stream-ordered scratch, the SGD update) captures into a CUDA graph, and
    replays are bit-identical to eager steps (deterministic kernels)."""
    from paper_2006_06608_b200.gcn import GCN2
    rng = np.random.default_rng(3)
    n = 900
    rp, col = powerlaw_graph(orc, rng, n, 4000)
    drp, dcol = to_dev(rp, col)
    x = to_dev((rng.random((n, 48)) - 0.5).astype(np.float32))
    dy = to_dev((rng.random((n, 10)) - 0.5).astype(np.float32))
    eager = GCN2(ctx, drp, dcol, 48, 16, 10, lr=0.05)
    graphed = GCN2(ctx, drp, dcol, 48, 16, 10, lr=0.05)
    assert torch.equal(eager.w1, graphed.w1) and torch.equal(eager.w2, graphed.w2)
    graphed.step(x, dy)  # warm-up (plans, attributes), then undo its update
    graphed.w1.copy_(eager.w1)
    graphed.w2.copy_(eager.w2)
    torch.cuda.synchronize()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    ctx.set_stream(cap)
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=cap):
            graphed.step(x, dy)
    finally:
        ctx.set_stream(torch.cuda.current_stream())
    graphed.w1.copy_(eager.w1)  # capture does not execute; keep both at the same start
    graphed.w2.copy_(eager.w2)
    for _ in range(3):
        g.replay()
        eager.step(x, dy)
    torch.cuda.synchronize()
    assert torch.equal(graphed.w1, eager.w1) and torch.equal(graphed.w2, eager.w2)
