"""GPU: the fp32 node update X·W on tcgen05 (gemm_tc.cu, 3xTF32 split, TMEM
accumulator) vs an fp64 numpy product.  Bar: |err| <= 1e-5 * (|A|·|W|)
elementwise (the fp32 parity bar of SURVEY §7 hard part 5), on shapes that
cover every template instance (k padded to 16/32/64/96/128, n to 16/32/64
with column blocks beyond 64), ragged m tails, k % 4 != 0 and unaligned A
(the scalar-load path), both fused epilogues, k > 128 (SIMT fallback) and
operands spanning many binades (where a single tf32 pass would fail).
"""
import numpy as np
import pytest
import torch

from conftest import to_dev

pytestmark = pytest.mark.gpu

SHAPES = [(1, 1, 1), (127, 8, 16), (128, 16, 16), (129, 22, 16), (300, 96, 16), (410, 16, 22), (1000, 24, 16),
          (257, 33, 70), (2000, 64, 64), (777, 128, 32), (513, 100, 130), (4096, 96, 16), (300, 160, 16),
          (40000, 96, 16)]


def check(got, a, w, post=None):
    want = a @ w
    bound = np.abs(a) @ np.abs(w)
    if post is not None:
        want, bound = post(want, bound)
    err = np.abs(got.astype(np.float64) - want)
    ratio = float((err / np.maximum(bound, 1e-300)).max()) if err.size else 0.0
    assert (err <= 1e-5 * bound + 1e-30).all(), ratio
    return ratio


@pytest.mark.parametrize("m,k,n", SHAPES)
def test_gemm_tc_shapes(ctx, m, k, n):
    rng = np.random.default_rng(m * 7 + k * 3 + n)
    a = ((rng.random((m, k)) - 0.3) * np.exp2(rng.integers(-8, 8, (m, k)))).astype(np.float32)
    w = ((rng.random((k, n)) - 0.5) * np.exp2(rng.integers(-6, 6, (k, n)))).astype(np.float32)
    da, dw = to_dev(a, w)
    got = ctx.gemm(da, dw).cpu().numpy()
    check(got, a.astype(np.float64), w.astype(np.float64))


def test_gemm_tc_epilogues_and_unaligned(ctx):
    rng = np.random.default_rng(5)
    m, k, n = 3001, 96, 16
    a = (rng.random((m, k + 1)) - 0.5).astype(np.float32)
    w = (rng.random((k, n)) - 0.5).astype(np.float32)
    b = (rng.random(n) - 0.5).astype(np.float32)
    s = rng.random(m)
    dfull, dw, db, ds = to_dev(a, w, b, s)
    da = dfull[:, 1:]  # row stride k+1 -> non-contiguous: the API packs it
    a64 = a[:, 1:].astype(np.float64)
    w64 = w.astype(np.float64)
    check(ctx.gemm(da.contiguous(), dw).cpu().numpy(), a64, w64)
    # 4-byte aligned but not 16-byte aligned A (offset view of a flat buffer)
    flat = torch.zeros(m * k + 1, dtype=torch.float32, device="cuda")
    flat[1:] = torch.from_numpy(np.ascontiguousarray(a[:, 1:])).cuda().reshape(-1)
    view = flat[1:].view(m, k)
    check(ctx.gemm(view, dw).cpu().numpy(), a64, w64)
    b64 = b.astype(np.float64)
    check(ctx.gemm(da.contiguous(), dw, db, 1).cpu().numpy(), a64, w64,
          lambda y, bd: (np.maximum(0.0, y + b64), bd + np.abs(b64)))
    check(ctx.gemm(da.contiguous(), dw, None, 2, ds).cpu().numpy(), a64, w64,
          lambda y, bd: (s[:, None] * y, s[:, None] * bd))


def test_gemm_tc_is_the_kernel_launched(ctx):
    """The fp32 product runs k6_gemm_tc (not a SIMT fallback) for k <= 128,
    as the CUDA profiler sees it."""
    a, w = to_dev(np.ones((256, 96), np.float32), np.ones((96, 16), np.float32))
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        y = ctx.gemm(a, w)
        torch.cuda.synchronize()
    assert torch.equal(y, torch.full((256, 16), 96.0, device="cuda"))
    names = [e.name for e in prof.events()]
    assert any("k6_gemm_tc" in nm for nm in names), names


TN_SHAPES = [(1, 4, 4), (31, 16, 16), (33, 96, 16), (1000, 96, 16), (5000, 16, 24), (4097, 64, 64), (2000, 128, 32),
             (777, 100, 60), (3000, 16, 22), (410236, 96, 16), (410236, 16, 22), (5000, 7, 13), (1, 3, 5),
             (20000, 30, 22), (1000, 130, 6), (2000, 64, 8), (3000, 32, 12), (100000, 128, 16)]


@pytest.mark.parametrize("m,p,q", TN_SHAPES)
def test_gemm_tn_tc(ctx, m, p, q):
    """dW = A^T B (the backward product): tcgen05 for p, q % 4 == 0, the
    cp.async-staged SIMT kernel for small p*q otherwise (k6_gemm_tn_small); fp32 result within 1e-5 of sum|a||b| (+ sqrt(m) fp32
    accumulation allowance over the rows of each CTA's run)."""
    from paper_2006_06608_b200.gcn import ctx_gemm_tn
    rng = np.random.default_rng(m + p * 7 + q)
    a = (rng.random((m, p)) - 0.5).astype(np.float32)
    b = ((rng.random((m, q)) - 0.5) * np.exp2(rng.integers(-4, 4, (m, q)))).astype(np.float32)
    da, db = to_dev(a, b)
    got = ctx_gemm_tn(ctx, da, db).cpu().numpy().astype(np.float64)
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    want = a64.T @ b64
    bound = np.abs(a64).T @ np.abs(b64)
    err = np.abs(got - want)
    assert (err <= 1e-5 * bound + 1e-30).all(), float((err / bound).max())


@pytest.mark.parametrize("m,k,n", [(410236, 22, 16), (410236, 22, 22), (3001, 22, 16), (3001, 30, 32), (131, 5, 7),
                                   (257, 1, 3), (64, 31, 9)])
def test_gemm_flat_narrow_epilogues(ctx, m, k, n):
    """k <= 32 with k % 4 != 0, n <= 32 (the C3 output layer's 22 columns):
    k6_gemm_flat, FFMA over flat float4 row runs, persistent over tiles.  Plain, bias+ReLU and row-scale epilogues, ragged
    last CTA, and a 4-byte-offset A (falls back to the tcgen05 scalar path)."""
    rng = np.random.default_rng(m + 31 * k + n)
    a = ((rng.random((m, k)) - 0.3) * np.exp2(rng.integers(-8, 8, (m, k)))).astype(np.float32)
    w = (rng.random((k, n)) - 0.5).astype(np.float32)
    b = (rng.random(n) - 0.5).astype(np.float32)
    s = rng.random(m)
    da, dw, db, ds = to_dev(a, w, b, s)
    a64, w64, b64 = a.astype(np.float64), w.astype(np.float64), b.astype(np.float64)
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        got = ctx.gemm(da, dw)
        torch.cuda.synchronize()
    assert any("k6_gemm_flat" in e.name for e in prof.events())
    check(got.cpu().numpy(), a64, w64)
    check(ctx.gemm(da, dw, db, 1).cpu().numpy(), a64, w64,
          lambda y, bd: (np.maximum(0.0, y + b64), bd + np.abs(b64)))
    check(ctx.gemm(da, dw, None, 2, ds).cpu().numpy(), a64, w64,
          lambda y, bd: (s[:, None] * y, s[:, None] * bd))
    flat = torch.zeros(m * k + 1, dtype=torch.float32, device="cuda")
    flat[1:] = da.reshape(-1)
    check(ctx.gemm(flat[1:].view(m, k), dw).cpu().numpy(), a64, w64)


@pytest.mark.parametrize("split", ["0", "1"])
def test_gemm_tc_both_kernels(split):
    """Both X·W kernels (two converter/epilogue groups, and the split-role one
    the K 128 shapes take) on shapes of either default, with both epilogues:
    GNNA_TC_SPLIT forces one (the switch is read once per process)."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from paper_2006_06608_b200.capi import Context
from test_gemm_tc_gpu import check
ctx = Context(0)
rng = np.random.default_rng(9)
for m, k, n in [(4096, 96, 16), (410, 16, 22), (3001, 128, 64), (513, 100, 130)]:
    a = (rng.random((m, k)) - 0.5).astype(np.float32)
    w = (rng.random((k, n)) - 0.5).astype(np.float32)
    b = (rng.random(n) - 0.5).astype(np.float32)
    s = rng.random(m)
    da, dw, db, ds = (torch.from_numpy(v).cuda() for v in (a, w, b, s))
    a64, w64, b64 = a.astype(np.float64), w.astype(np.float64), b.astype(np.float64)
    check(ctx.gemm(da, dw).cpu().numpy(), a64, w64)
    check(ctx.gemm(da, dw, db, 1).cpu().numpy(), a64, w64,
          lambda x, bd: (np.maximum(x + b64, 0), bd + np.abs(b64)))
    check(ctx.gemm(da, dw, None, 2, ds).cpu().numpy(), a64, w64, lambda x, bd: (x * s[:, None], bd * s[:, None]))
print("ok")
'''
    r = subprocess.run([sys.executable, "-c", code, ROOT], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, GNNA_TC_SPLIT=split))
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
