"""Small GPU workload exercising every kernel family once, for compute-sanitizer
(memcheck / racecheck / synccheck).  Exits non-zero on any parity error."""
import os

os.environ.setdefault("GNNA_FLAT_CTAS", "1")  # k6_gemm_flat persistent loop with few CTAs
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle.cpu import Oracle  # noqa: E402
from paper_2006_06608_b200.capi import Context, Params  # noqa: E402
from paper_2006_06608_b200.gcn import GCN2  # noqa: E402


def dev(a):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if t.dtype == torch.uint64:
        t = t.view(torch.int64)
    elif t.dtype == torch.uint32:
        t = t.view(torch.int32)
    return t.cuda()


def main():
    orc = Oracle("orc")
    ctx = Context(0)
    rng = np.random.default_rng(1)
    n = 3000
    w = 1.0 / np.arange(1, n + 1) ** 0.8
    src = rng.choice(n, size=20000, p=w / w.sum())
    edges = np.stack([src, rng.integers(0, n, 20000)], 1).astype(np.uint32)
    rp, col = orc.to_csr(n, edges, True)
    drp, dcol = dev(rp), dev(col)
    rp2, col2 = ctx.to_csr(n, dev(edges), True)
    assert np.array_equal(rp2.cpu().numpy().view(np.uint64), rp)
    for dim in (16, 64, 130):
        x = rng.random((n, dim))
        for s in (0, 1, 2):
            p = Params.make(ngs=5, dw=8, tpb=128, dim=dim)
            plan = ctx.plan(drp, dcol, p, s)
            want, cost = orc.aggregate_scheduled(rp, col, x, p.tolist(), s, 1, cache=(4096, 128))
            got = plan.aggregate(dev(x)).cpu().numpy()
            assert np.array_equal(got, want)
            c = plan.cost(line=128, cache=(4096, 128))
            assert c.tolist() == cost.tolist()
            plan.aggregate(dev(x).float())
    x = rng.random((n, 24))
    wt = rng.random((24, 8)) - 0.5
    assert np.array_equal(ctx.gcn_forward(drp, dcol, dev(x), dev(wt), True).cpu().numpy(),
                          orc.gcn_layer(rp, col, x, wt, True))
    ctx.gcn_backward(drp, dcol, dev(x).float(), dev(wt).float(), dev(rng.random((n, 8))).float(), True)
    b = rng.random(8)
    ctx.gin_backward(drp, dcol, dev(x), 0.1, dev(wt), dev(b), dev(rng.random((n, 8))))
    com, k = ctx.detect_communities(drp, dcol)
    c2, k2 = orc.detect_communities(rp, col)
    assert k == k2 and np.array_equal(com.cpu().numpy().view(np.uint32), c2)
    o2n, n2o = ctx.build_mapping(com, k)
    ctx.apply_mapping_csr(drp, dcol, o2n, n2o)
    m = GCN2(ctx, drp, dcol, 24, 16, 8)
    m.step(dev(x).float(), dev(rng.random((n, 8))).float())
    # tcgen05 GEMMs: TMA-fed (k % 4 == 0), both dW kernels, fused epilogues;
    # k = 22 runs k6_gemm_flat (persistent loop: GNNA_FLAT_CTAS=1 below, 157 tiles on 148 CTAs)
    from paper_2006_06608_b200.gcn import ctx_gemm_tn
    for k, q in ((96, 16), (22, 16), (16, 22), (64, 64)):
        a = dev(rng.random((n, k)) - 0.5).float()
        wq = dev(rng.random((k, q)) - 0.5).float()
        g = dev(rng.random((n, q)) - 0.5).float()
        want = a.double() @ wq.double()
        assert torch.allclose(ctx.gemm(a, wq).double(), want, rtol=1e-4, atol=1e-4)
        ctx.gemm(a, wq, dev(rng.random(q)).float(), 1)
        ctx.gemm(a, wq, None, 2, dev(rng.random(n)))
        assert torch.allclose(ctx_gemm_tn(ctx, a, g).double(), a.double().t() @ g.double(), rtol=1e-4, atol=1e-3)
    a = dev(rng.random((20000, 22)) - 0.5).float()
    wq = dev(rng.random((22, 16)) - 0.5).float()
    assert torch.allclose(ctx.gemm(a, wq).double(), a.double() @ wq.double(), rtol=1e-4, atol=1e-4)
    # fused all-gather: K3 fan-out into local replicas
    p = Params.make(ngs=16, dw=16, tpb=256, dim=32)
    plan = ctx.plan(drp, dcol, p, 2, rows=(100, 2500))
    xf = dev(rng.random((n, 32))).float()
    y = torch.zeros((n, 32), device="cuda")
    reps = [torch.zeros((n, 32), device="cuda") for _ in range(3)]
    plan.aggregate_fanout(xf, y, peers=reps)
    assert all(torch.equal(r, y) for r in reps)
    # round 2: node-weight fan-out, the fused dense backward (C3 output-layer
    # widths), the hub remap / row gather of the drop-in, the device-aware
    # evaluator, empty rows + split nodes through the one-launch K3
    rs, sw, _ = ctx.gcn_weights(drp, dcol, True, edge_weights=False)
    plan.aggregate_fanout(xf, y, peers=reps, node_weight=rs, self_weight=sw, row_scale=rs)
    m2 = GCN2(ctx, drp, dcol, 96, 16, 22)
    m2.step(dev(rng.random((n, 96))).float(), dev(rng.random((n, 22)) - 0.5).float())
    dz, dwd = ctx.dense_backward(dev(rng.random((777, 22))).float(), dev(rng.random((16, 22))).float(),
                                 dev(rng.random((777, 16))).float(), dev(rng.random(777)))
    hubs = torch.empty(64, dtype=torch.int32, device="cuda")
    col_h = torch.empty_like(dcol)
    import ctypes as C
    he = C.c_uint64()
    assert ctx.L.gnna_hub_remap(ctx.h, C.c_void_p(drp.data_ptr()), C.c_void_p(dcol.data_ptr()), C.c_uint32(n),
                                C.c_uint32(64), C.c_void_p(hubs.data_ptr()), C.c_void_p(col_h.data_ptr()),
                                C.byref(he)) == 0
    xe = torch.empty((n + 64, 16), dtype=torch.float64, device="cuda")
    xe[:n] = dev(rng.random((n, 16)))
    assert ctx.L.gnna_gather_rows(ctx.h, C.c_int(1), C.c_void_p(xe.data_ptr()), C.c_uint32(16),
                                  C.c_void_p(hubs.data_ptr()), C.c_uint64(64),
                                  C.c_void_p(xe[n:].data_ptr())) == 0
    ph = ctx.plan(drp, col_h, Params.make(ngs=5, dw=8, tpb=128, dim=16), 2)
    pn = ctx.plan(drp, dcol, Params.make(ngs=5, dw=8, tpb=128, dim=16), 2)
    yh = torch.empty((n, 16), dtype=torch.float64, device="cuda")
    assert ctx.L.gnna_aggregate(ctx.h, ph.h, C.c_int(1), C.c_int(1), C.c_void_p(xe.data_ptr()),
                                C.c_void_p(yh.data_ptr())) == 0  # hub rows read from the tail
    assert torch.equal(yh, pn.aggregate(xe[:n].contiguous()))    # bit-identical to the plain layout
    ctx.b200_params(drp, 16, window=True)
    ctx.b200_params(drp, 64, dtype=torch.float64)
    # isolated nodes (empty rows) in a plan with split hubs: trailing blocks + last-writer combine
    e2 = edges[edges[:, 0] < n - 50]
    e2 = e2[e2[:, 1] < n - 50]
    rpe, cole = orc.to_csr(n, e2, True)
    pe = ctx.plan(dev(rpe), dev(cole), Params.make(ngs=4, dw=8, tpb=128, dim=16), 2)
    for dt in (torch.float32, torch.float64):
        xs = dev(rng.random((n, 16))).to(dt)
        got = pe.aggregate_ex(xs, alpha=0.5)
        want = orc.aggregate_oracle(rpe, cole, xs.double().cpu().numpy()) + 0.5 * xs.double().cpu().numpy()
        assert np.allclose(got.double().cpu().numpy(), want, rtol=1e-5)
    # round 2, late: the split-role X.W kernel (K 128), the packed / 128-row dW
    # kernel, the pre-scaled weighted gather (node weights, >= 4 edges per row)
    # and the staged pageable copies (pinned bounce ring)
    for k, q in ((128, 32), (96, 16)):
        a = dev(rng.random((5000, k)) - 0.5).float()
        wq = dev(rng.random((k, q)) - 0.5).float()
        assert torch.allclose(ctx.gemm(a, wq).double(), a.double() @ wq.double(), rtol=1e-4, atol=1e-4)
        g = dev(rng.random((5000, q)) - 0.5).float()
        assert torch.allclose(ctx_gemm_tn(ctx, a, g).double(), a.double().t() @ g.double(), rtol=1e-4, atol=1e-3)
    pw = ctx.plan(drp, dcol, Params.make(ngs=16, dw=16, tpb=256, dim=32), 2)
    yw = pw.aggregate_ex(xf, node_weight=rs, self_weight=sw, row_scale=rs)
    deg = np.diff(rp).astype(np.float64)
    x64 = xf.double().cpu().numpy()
    nrm = rs.double().cpu().numpy()
    swn = sw.double().cpu().numpy()
    want = orc.aggregate_oracle(rp, col, x64 * nrm[:, None]) + swn[:, None] * x64
    assert np.allclose(yw.double().cpu().numpy(), nrm[:, None] * want, rtol=1e-5, atol=1e-6), deg.mean()
    big = np.frombuffer(rng.bytes((9 << 20) + 20), dtype=np.uint8).copy()
    dbig = torch.empty(big.size, dtype=torch.uint8, device="cuda")
    assert ctx.L.gnna_copy_to_device(ctx.h, C.c_void_p(dbig.data_ptr()), C.c_void_p(big.ctypes.data),
                                     C.c_size_t(big.size)) == 0
    back = np.empty_like(big)
    assert ctx.L.gnna_copy_to_host(ctx.h, C.c_void_p(back.ctypes.data), C.c_void_p(dbig.data_ptr()),
                                   C.c_size_t(big.size)) == 0
    assert np.array_equal(back, big)
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
