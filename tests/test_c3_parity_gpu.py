"""GPU parity of the north-star target config at FULL size: BASELINE C3, the
amazon0505-shape graph (410,236 nodes, ~4.9M nnz), every aggregation form the
bench times and the 2-layer GCN training step, against the fp64 oracle
(oracle/gnnsim_oracle.c, pinned to the reference by tests/test_oracle.py).

Bar: |got - want| <= 1e-5 * (|want| + bound), where
`bound` is the same computation on |inputs| (the sum of |terms|), so signed
cancellation does not void the check.  With U[0,1) features and positive
weights bound == want and the bar is the plain 1e-5 relative one.

Forms (bench.py extra_workloads):
* GCN layer form: xs = norm * x (the update GEMM's row-scale epilogue), K3 =
  plain sum with the destination scale in the flush -- engine.cpp:338-369.
* GCN standalone gather: node_weight norm[u] gathered per edge, self weight,
  row scale, with and without implicit self loops (engine.cpp:344-353).
* GIN input: sum + (1 + eps) x, eps 0.1 (engine.cpp:384-408).
* The F32 layer entry points gcn_forward / gin_forward with signed weights.
* The C3 training step (GCN2 96 -> 16 -> 22, forward + backward): output and
  dW1 / dW2 vs the oracle's fp64 gcn_layer / gcn_backward chain.
"""
import numpy as np
import pytest
import torch

from conftest import to_dev

pytestmark = pytest.mark.gpu

TOL = 1e-5


def check(got, want, bound, what):
    got = np.asarray(got, np.float64)
    err = np.abs(got - want)
    lim = TOL * (np.abs(want) + bound)
    bad = err > lim + 1e-30
    worst = float((err / (np.abs(want) + bound + 1e-300)).max()) if err.size else 0.0
    assert not bad.any(), f"{what}: {int(bad.sum())} elements out of tolerance, worst {worst:.3g}"
    return worst


@pytest.fixture(scope="module")
def c3(ctx):
    from paper_2006_06608_b200 import synth
    from paper_2006_06608_b200.capi import WARP_SHARED
    cfg = synth.CONFIGS["c3"]
    _, rp, col = synth.build_graph(cfg, lambda n, e: ctx.to_csr(n, e, True), torch.device("cuda", 0))
    p, _ = ctx.b200_params(rp, cfg.dim)
    plan = ctx.plan(rp, col, p, WARP_SHARED)
    rph, colh = rp.cpu().numpy().view(np.uint64), col.cpu().numpy().view(np.uint32)
    x = np.random.default_rng(31).random((cfg.n, cfg.dim)).astype(np.float32)
    return dict(cfg=cfg, rp=rp, col=col, rph=rph, colh=colh, plan=plan, x=x, dx=to_dev(x))


def test_c3_graph_is_the_config(c3):
    n, nnz = c3["cfg"].n, int(c3["colh"].size)
    assert n == 410_236 and abs(nnz - 4_878_874) <= 0.002 * 4_878_874
    assert c3["plan"].info()["split_nodes"] > 0  # hubs span schedule blocks: the carry path runs


def test_c3_gcn_layer_form(ctx, orc, c3):
    """K3 as in the GCN layer: input pre-scaled by norm (GEMM epilogue),
    destination scale in the flush; no implicit self loops."""
    x64 = c3["x"].astype(np.float64)
    rs, _, _ = ctx.gcn_weights(c3["rp"], c3["col"], False, edge_weights=False)
    xs = c3["dx"] * rs[:, None]
    got = c3["plan"].aggregate_ex(xs, row_scale=rs).cpu().numpy()
    want = orc.gcn_layer(c3["rph"], c3["colh"], x64, np.eye(16), False)  # = normalized_aggregate (W = I)
    check(got, want, want, "gcn layer form")


@pytest.mark.parametrize("self_loops", [False, True])
def test_c3_gcn_standalone_gather(ctx, orc, c3, self_loops):
    x64 = c3["x"].astype(np.float64)
    rs, sw, _ = ctx.gcn_weights(c3["rp"], c3["col"], self_loops, edge_weights=False)
    got = c3["plan"].aggregate_ex(c3["dx"], node_weight=rs, self_weight=sw, row_scale=rs).cpu().numpy()
    want = orc.gcn_layer(c3["rph"], c3["colh"], x64, np.eye(16), self_loops)
    check(got, want, want, f"gcn gather self_loops={self_loops}")


def test_c3_gin_sum(orc, c3):
    x64 = c3["x"].astype(np.float64)
    got = c3["plan"].aggregate_ex(c3["dx"], alpha=1.1).cpu().numpy()
    want = orc.aggregate_oracle(c3["rph"], c3["colh"], x64) + 1.1 * x64  # gin_layer's z (engine.cpp:390-395)
    check(got, want, want, "gin sum")


def test_c3_plain_sum_fp32_and_determinism(orc, c3):
    x64 = c3["x"].astype(np.float64)
    y1 = c3["plan"].aggregate(c3["dx"])
    y2 = c3["plan"].aggregate(c3["dx"])
    assert torch.equal(y1, y2)
    want = orc.aggregate_oracle(c3["rph"], c3["colh"], x64)
    check(y1.cpu().numpy(), want, want, "sum")


def test_c3_layer_entry_points_signed(ctx, orc, c3):
    """gnna_gcn_forward / gnna_gin_forward F32 (plan, fused normalisation,
    tcgen05 update) on the full graph with signed weights and features."""
    rng = np.random.default_rng(32)
    n = c3["cfg"].n
    x = (rng.random((n, 96)) - 0.5).astype(np.float32)
    w = ((rng.random((96, 16)) * 2 - 1) / np.sqrt(96)).astype(np.float32)
    x64, w64 = x.astype(np.float64), w.astype(np.float64)
    got = ctx.gcn_forward(c3["rp"], c3["col"], to_dev(x), to_dev(w), False).cpu().numpy()
    want = orc.gcn_layer(c3["rph"], c3["colh"], x64, w64, False)
    bound = orc.gcn_layer(c3["rph"], c3["colh"], np.abs(x64), np.abs(w64), False)
    check(got, want, bound, "gcn_forward 96->16")
    x2 = (rng.random((n, 16)) - 0.5).astype(np.float32)
    w2 = (rng.random((16, 16)) - 0.5).astype(np.float32)
    b2 = (rng.random(16) - 0.5).astype(np.float32)
    eps = 0.1
    got = ctx.gin_forward(c3["rp"], c3["col"], to_dev(x2), eps, to_dev(w2), to_dev(b2)).cpu().numpy()
    x2d, w2d, b2d = x2.astype(np.float64), w2.astype(np.float64), b2.astype(np.float64)
    want = orc.gin_layer(c3["rph"], c3["colh"], x2d, eps, w2d, b2d)
    bound = orc.gin_layer(c3["rph"], c3["colh"], np.abs(x2d), eps, np.abs(w2d), np.abs(b2d))
    check(got, want, bound, "gin_forward 16->16")


def test_c3_train_step_full_size(ctx, orc, c3):
    """The timed C3 step (bench.py --workload c3train): 2-layer GCN 96 -> 16
    -> 22, forward + backward, at full size.  Reference: the oracle's fp64
    gcn_layer twice with a ReLU between, and gcn_backward through both layers.
    The ReLU mask of the backward is the GPU's own forward mask; the test
    first checks that every entry where it differs from the fp64 mask is a
    pre-activation within the error bar of zero (a legitimate tie)."""
    from paper_2006_06608_b200 import synth
    from paper_2006_06608_b200.gcn import GCN2
    rp, col, rph, colh = c3["rp"], c3["col"], c3["rph"], c3["colh"]
    n = c3["cfg"].n
    model = GCN2(ctx, rp, col, 96, 16, 22, self_loops=False, lr=0.0)
    x = synth.features(n, 96, 3, rp.device)
    dy = (synth.features(n, 22, 6 - 1000, rp.device) - 0.5).contiguous()
    y, dw1, dw2 = model.step(x, dy)
    h1_gpu = model.saved["h1"].cpu().numpy()  # norm * h1 (pre-scaled): same sign as h1
    x64, dy64 = x.double().cpu().numpy(), dy.double().cpu().numpy()
    w1, w2 = model.w1.double().cpu().numpy(), model.w2.double().cpu().numpy()
    ax, aw1, aw2, ady = np.abs(x64), np.abs(w1), np.abs(w2), np.abs(dy64)

    pre1 = orc.gcn_layer(rph, colh, x64, w1, False)
    b_pre1 = orc.gcn_layer(rph, colh, ax, aw1, False)
    h1 = np.maximum(pre1, 0.0)
    want_y = orc.gcn_layer(rph, colh, h1, w2, False)
    b_y = orc.gcn_layer(rph, colh, b_pre1, aw2, False)
    check(y.cpu().numpy(), want_y, b_y, "train step output")

    mask_gpu = h1_gpu > 0
    flips = mask_gpu != (pre1 > 0)
    assert (np.abs(pre1[flips]) <= TOL * b_pre1[flips]).all(), "ReLU mask differs away from a tie"

    dh1, want_dw2 = orc.gcn_backward(rph, colh, h1, w2, dy64, False)
    b_dh1, b_dw2 = orc.gcn_backward(rph, colh, b_pre1, aw2, ady, False)
    check(dw2.cpu().numpy(), want_dw2, b_dw2, "dW2")
    _, want_dw1 = orc.gcn_backward(rph, colh, x64, w1, dh1 * mask_gpu, False)
    _, b_dw1 = orc.gcn_backward(rph, colh, ax, aw1, b_dh1, False)
    check(dw1.cpu().numpy(), want_dw1, b_dw1, "dW1")
