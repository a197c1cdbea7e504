"""GPU parity: the layer entry points (gcn_layer / gin_layer forward, F64
bitwise vs the reference; F32 within an error-aware 1e-5 tolerance) and the
new backward entry points (vs the oracle's analytic gradients, which
tests/test_oracle.py pins by finite differences of the reference forward,
and vs torch float64 autograd)."""
import numpy as np
import pytest
import torch

from conftest import golden_cases, random_graph, to_dev

pytestmark = pytest.mark.gpu


def close32(got, want, bound, rtol=1e-5):
    """|got - want| <= rtol * (|want| + bound): bound = the same op on |inputs|
    (sum of |terms|), so signed cancellation does not void the check."""
    err = np.abs(got - want)
    return (err <= rtol * (np.abs(want) + bound) + 1e-30).all(), float((err / (np.abs(want) + bound + 1e-30)).max())


def test_forward_f64_golden(ctx):
    g = golden_cases()
    for i in g.ids("gcn"):
        rp, col, x, w = g[f"gcn/{i}/rp"], g[f"gcn/{i}/col"], g[f"gcn/{i}/x"], g[f"gcn/{i}/w"]
        sl = bool(g[f"gcn/{i}/self_loops"][0])
        drp, dcol, dx, dw = to_dev(rp, col, x, w)
        assert np.array_equal(ctx.gcn_forward(drp, dcol, dx, dw, sl).cpu().numpy(), g[f"gcn/{i}/y"]), i
        eps = float(g[f"gin/{i}/eps"][0])
        got = ctx.gin_forward(drp, dcol, dx, eps, dw, to_dev(g[f"gin/{i}/b"])).cpu().numpy()
        assert np.array_equal(got, g[f"gin/{i}/y"]), i


def test_forward_random_f64_bitwise_f32_tolerance(ctx, orc):
    rng = np.random.default_rng(8)
    for t in range(24):
        n = int(rng.integers(1, 600))
        rp, col, _ = random_graph(rng, n, int(rng.integers(0, 8 * n + 1)), orc=orc)
        din, dout = int(rng.integers(1, 70)), int(rng.integers(1, 70))
        x = rng.random((n, din)) - 0.4
        x[rng.random((n, din)) < 0.1] = 0.0  # exercise matmul's a == 0 skip
        w = rng.random((din, dout)) * 2 - 1
        b = rng.random(dout) - 0.5
        sl = bool(t % 2)
        eps = float(rng.choice([0.0, 0.3, -0.5]))
        drp, dcol, dx, dw, db = to_dev(rp, col, x, w, b)
        want = orc.gcn_layer(rp, col, x, w, sl)
        assert np.array_equal(ctx.gcn_forward(drp, dcol, dx, dw, sl).cpu().numpy(), want), t
        bound = orc.gcn_layer(rp, col, np.abs(x), np.abs(w), sl)
        ok, r = close32(ctx.gcn_forward(drp, dcol, dx.float(), dw.float(), sl).cpu().numpy(), want, bound)
        assert ok, (t, r)
        want = orc.gin_layer(rp, col, x, eps, w, b)
        assert np.array_equal(ctx.gin_forward(drp, dcol, dx, eps, dw, db).cpu().numpy(), want), t
        bound = orc.gin_layer(rp, col, np.abs(x), abs(1 + eps) - 1, np.abs(w), np.abs(b))
        ok, r = close32(ctx.gin_forward(drp, dcol, dx.float(), eps, dw.float(), db.float()).cpu().numpy(), want,
                        bound)
        assert ok, (t, r)


def test_gemm_epilogues(ctx):
    rng = np.random.default_rng(2)
    for m, k, n in ((1, 1, 1), (300, 96, 16), (257, 33, 70), (1000, 64, 64), (5, 0, 3)):
        a = rng.random((m, k)) - 0.5
        w = rng.random((k, n)) - 0.5
        b = rng.random(n) - 0.5
        s = rng.random(m)
        da, dw, db, ds = to_dev(a, w, b, s)
        # exact f64: sequential k with separately rounded products
        want = np.zeros((m, n))
        for kk in range(k):
            want = want + a[:, kk:kk + 1] * w[kk:kk + 1, :]
        got = ctx.gemm(da, dw).cpu().numpy()
        assert np.array_equal(got, want)
        assert np.array_equal(ctx.gemm(da, dw, db, 1).cpu().numpy(), np.maximum(0.0, want + b))
        assert np.array_equal(ctx.gemm(da, dw, None, 2, ds).cpu().numpy(), s[:, None] * want)
        got32 = ctx.gemm(da.float(), dw.float()).cpu().numpy()
        bound = np.abs(a) @ np.abs(w)
        assert close32(got32, want, bound)[0]


@pytest.mark.parametrize("sl", [False, True])
def test_gcn_backward(ctx, orc, sl):
    rng = np.random.default_rng(21 + sl)
    for t in range(10):
        n = int(rng.integers(2, 400))
        rp, col, _ = random_graph(rng, n, int(rng.integers(1, 6 * n)), orc=orc)
        din, dout = (int(rng.integers(2, 40)), int(rng.integers(1, 40)))
        if t % 2:
            din, dout = dout, din  # both update orders
        x = rng.random((n, din)) - 0.5
        w = rng.random((din, dout)) - 0.5
        dy = rng.random((n, dout)) - 0.5
        wdx, wdw = orc.gcn_backward(rp, col, x, w, dy, sl)
        drp, dcol, dx_, dw_, ddy = to_dev(rp, col, x, w, dy)
        gdx, gdw = ctx.gcn_backward(drp, dcol, dx_, dw_, ddy, sl)
        np.testing.assert_allclose(gdx.cpu().numpy(), wdx, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(gdw.cpu().numpy(), wdw, rtol=1e-10, atol=1e-12)
        # fp32 inputs rounded first, so the bar measures the kernels' error only
        x32, w32, dy32 = (a.astype(np.float32).astype(np.float64) for a in (x, w, dy))
        wdx, wdw = orc.gcn_backward(rp, col, x32, w32, dy32, sl)
        bdx, bdw = orc.gcn_backward(rp, col, np.abs(x32), np.abs(w32), np.abs(dy32), sl)
        fdx, fdw = ctx.gcn_backward(drp, dcol, dx_.float(), dw_.float(), ddy.float(), sl)
        ok, r = close32(fdx.cpu().numpy(), wdx, bdx)
        assert ok, (t, "dx", r)
        ok, r = close32(fdw.cpu().numpy(), wdw, bdw)
        assert ok, (t, "dw", r)


def test_gin_backward_vs_oracle_and_autograd(ctx, orc):
    rng = np.random.default_rng(33)
    for t in range(10):
        n = int(rng.integers(2, 300))
        rp, col, _ = random_graph(rng, n, int(rng.integers(1, 6 * n)), orc=orc)
        din, dout = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        x = rng.random((n, din)) - 0.5
        w = rng.random((din, dout)) - 0.5
        b = rng.random(dout) - 0.5
        dy = rng.random((n, dout)) - 0.5
        eps = float(rng.choice([0.0, 0.2]))
        wdx, wdw, wdb, wde = orc.gin_backward(rp, col, x, eps, w, b, dy)
        drp, dcol, dxx, dww, dbb, ddy = to_dev(rp, col, x, w, b, dy)
        gdx, gdw, gdb, gde = ctx.gin_backward(drp, dcol, dxx, eps, dww, dbb, ddy)
        np.testing.assert_allclose(gdx.cpu().numpy(), wdx, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(gdw.cpu().numpy(), wdw, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(gdb.cpu().numpy(), wdb, rtol=1e-10, atol=1e-12)
        assert gde == pytest.approx(wde, rel=1e-10, abs=1e-12)
        # fp32 within the error-aware 1e-5 bar (bound: the same backward on |inputs|, every ReLU open)
        x32, w32, b32, dy32 = (a.astype(np.float32).astype(np.float64) for a in (x, w, b, dy))
        wdx, wdw, wdb, _ = orc.gin_backward(rp, col, x32, eps, w32, b32, dy32)
        bdx, bdw, bdb, _ = orc.gin_backward(rp, col, np.abs(x32), eps, np.abs(w32), np.abs(b32) + 1.0,
                                            np.abs(dy32))
        fdx, fdw, fdb, _ = ctx.gin_backward(drp, dcol, dxx.float(), eps, dww.float(), dbb.float(), ddy.float())
        for got, want, bnd, nm in ((fdx, wdx, bdx, "dx"), (fdw, wdw, bdw, "dw"), (fdb, wdb, bdb, "db")):
            ok, r = close32(got.cpu().numpy(), want, bnd)
            assert ok, (t, nm, r)
        # independent: torch float64 autograd over a dense adjacency
        A = torch.zeros((n, n), dtype=torch.float64)
        for v in range(n):
            A[v, torch.from_numpy(col[rp[v]:rp[v + 1]].astype(np.int64))] = 1.0
        X = torch.tensor(x, requires_grad=True)
        W = torch.tensor(w, requires_grad=True)
        B = torch.tensor(b, requires_grad=True)
        E = torch.tensor(eps, dtype=torch.float64, requires_grad=True)
        Y = torch.relu((A @ X + (1 + E) * X) @ W + B)
        Y.backward(torch.tensor(dy))
        np.testing.assert_allclose(gdx.cpu().numpy(), X.grad.numpy(), rtol=1e-9, atol=1e-11)
        np.testing.assert_allclose(gdw.cpu().numpy(), W.grad.numpy(), rtol=1e-9, atol=1e-11)
        assert gde == pytest.approx(float(E.grad), rel=1e-9, abs=1e-11)


def test_features_close_matches_reference_rule(ctx):
    """engine.cpp:162-172: |a-b| <= tol*max(|a|,|b|) elementwise; NaN compares false (counts as close)."""
    rng = np.random.default_rng(4)
    a = rng.random(10000) - 0.5
    b = a * (1 + 1e-13)
    assert ctx.features_close(to_dev(a), to_dev(b), 1e-12)
    b2 = b.copy()
    b2[1234] *= 1 + 1e-9
    assert not ctx.features_close(to_dev(a), to_dev(b2), 1e-12)
    z = np.zeros(5)
    assert ctx.features_close(to_dev(z), to_dev(z), 0.0)
    n1 = np.array([np.nan, 1.0])
    assert ctx.features_close(to_dev(n1), to_dev(np.array([5.0, 1.0])), 1e-12)
    assert not ctx.features_close(to_dev(np.zeros(3)), to_dev(np.zeros(4)), 1.0)


def test_backward_nonsymmetric_uses_transpose(ctx, orc):
    rng = np.random.default_rng(5)
    n = 200
    edges = rng.integers(0, n, size=(900, 2)).astype(np.uint32)
    rp, col = orc.to_csr(n, edges, False)
    x = rng.random((n, 12)) - 0.5
    w = rng.random((12, 5)) - 0.5
    dy = rng.random((n, 5)) - 0.5
    drp, dcol = to_dev(rp, col)
    rt = ctx.csr_transpose(drp, dcol)
    gdx, gdw = ctx.gcn_backward(drp, dcol, *to_dev(x, w, dy), False, rt=rt)
    wdx, wdw = orc.gcn_backward(rp, col, x, w, dy, False)
    np.testing.assert_allclose(gdx.cpu().numpy(), wdx, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(gdw.cpu().numpy(), wdw, rtol=1e-10, atol=1e-12)


def test_dense_backward_fused(ctx):
    """gnna_dense_backward (backward of y = z W): dz = s * (dy W^T), dW = z^T dy.
    fp32 (one fused pass for p, q <= 32) at the error-aware 1e-5 bar, ragged
    row counts and widths incl. the C3 output layer (16 x 22); fp64 equals
    the separate exact products (gnna_gemm / gnna_gemm_tn orders)."""
    from paper_2006_06608_b200.gcn import ctx_gemm_tn
    rng = np.random.default_rng(9)
    for m, p, q in ((1, 1, 1), (63, 16, 22), (64, 16, 22), (1000, 16, 22), (4097, 7, 13), (3000, 32, 32),
                    (2500, 40, 22), (410236, 16, 22)):
        dy = rng.random((m, q)) - 0.5
        w = rng.random((p, q)) - 0.5
        z = rng.random((m, p)) - 0.5
        s = rng.random(m) + 0.5
        ddy, dw, dz, ds = to_dev(dy.astype(np.float32), w.astype(np.float32), z.astype(np.float32), s)
        gz, gw = ctx.dense_backward(ddy, dw, dz, ds)
        y32, w32, z32 = (a.astype(np.float32).astype(np.float64) for a in (dy, w, z))
        want_dz = s[:, None] * (y32 @ w32.T)
        bound_dz = s[:, None] * (np.abs(y32) @ np.abs(w32).T)
        ok, r = close32(gz.cpu().numpy(), want_dz, bound_dz)
        assert ok, (m, p, q, "dz", r)
        ok, r = close32(gw.cpu().numpy(), z32.T @ y32, np.abs(z32).T @ np.abs(y32))
        assert ok, (m, p, q, "dW", r)
        # fp64: the separate exact products
        d64 = to_dev(dy, w, z)
        gz64, gw64 = ctx.dense_backward(d64[0], d64[1], d64[2], ds)
        assert torch.equal(gw64, ctx_gemm_tn(ctx, d64[2], d64[0]))
        assert torch.equal(gz64, ctx.gemm(d64[0], d64[1].t().contiguous(), None, 2, ds))
    # no row scale
    dy, w, z = (torch.rand(s, device="cuda") - 0.5 for s in ((777, 22), (16, 22), (777, 16)))
    gz, _ = ctx.dense_backward(dy, w, z)
    want = dy.double() @ w.double().t()
    ok, r = close32(gz.cpu().numpy(), want.cpu().numpy(), (dy.double().abs() @ w.double().abs().t()).cpu().numpy())
    assert ok, r
