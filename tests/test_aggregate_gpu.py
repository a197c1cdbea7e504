"""GPU parity: K1/K2 preprocessing, K3 aggregation, K8 counters through the
C-ABI (libgnna.so) against the CPU oracle (oracle/gnnsim_oracle.c), which
tests/test_oracle.py pins to the reference itself.

Bars: integer/index outputs bit-exact; fp64 aggregation bitwise equal to the
reference's summation tree; fp32 within 1e-5 relative of the fp64 reference
(inputs are non-negative U[0,1), so no cancellation: SURVEY Appendix A)."""
import numpy as np
import pytest
import torch

from conftest import random_graph, to_dev

pytestmark = pytest.mark.gpu

STRATS = (0, 1, 2)
MODES = (0, 1)


def corpus(seed, count, max_n=300):
    rng = np.random.default_rng(seed)
    dims = [1, 16, 64, 128, 3, 33, 8, 2]
    for i in range(count):
        n = int(np.exp(rng.random() * np.log(max_n / 4.0)) * 4)
        deg = 1 + int(rng.integers(0, 32))
        rp, col, _ = random_graph(rng, n, max(1, n * deg // 2))
        dim = dims[i % len(dims)]
        x = rng.random((n, dim))
        params = []
        for _ in range(3):
            params.append(dict(ngs=1 + int(rng.integers(0, 64)), dw=1 + int(rng.integers(0, 32)),
                               tpb=32 * (1 + int(rng.integers(0, 32))), dim=dim))
        yield i, rp, col, x, params


def P(**kw):
    from paper_2006_06608_b200.capi import Params
    return Params.make(**kw)


def test_partition_neighbors_bit_exact(ctx, orc):
    import torch
    rng = np.random.default_rng(5)
    for t in range(40):
        n = int(rng.integers(1, 500))
        rp, col, _ = random_graph(rng, n, int(rng.integers(0, 8 * n + 1)), symmetrize=bool(t % 2))
        ngs = int(rng.choice([1, 2, 3, 7, 16, 64, 1000]))
        ids, tg, bg, en = orc.partition_neighbors(rp, col, ngs)
        pp, p2n = ctx.partition_neighbors(to_dev(rp), ngs)
        pp, p2n = pp.cpu().numpy().view(np.uint64), p2n.cpu().numpy().view(np.uint32)
        assert len(p2n) == len(tg)
        assert (p2n == tg).all()
        assert (pp[:-1] == bg).all() and (pp[1:] == en).all()
        if len(tg) == 0:
            assert pp[0] == rp[-1]


def test_build_mem_plan_bit_exact(ctx, orc):
    rng = np.random.default_rng(2002)
    # hand-traced fixture (test_memplan.cpp:58-74)
    slot, lead, sb = ctx.build_mem_plan(to_dev(np.array([0, 0, 1, 2, 2, 2], np.uint32)), P(tpb=64, dim=16))
    assert slot.cpu().tolist() == [0, 0, 0, 1, 0, 0]
    assert lead.cpu().tolist() == [1, 0, 1, 1, 1, 0]
    assert sb == 2 * 16 * 4
    for _ in range(300):
        targets = []
        for v in range(1 + int(rng.integers(0, 40))):
            targets += [v] * int(rng.integers(0, 5))
        if not targets:
            targets = [0]
        t = np.array(targets, np.uint32)
        p = P(tpb=32 * (1 + int(rng.integers(0, 32))), dim=1 + int(rng.integers(0, 64)))
        s1, _, l1, b1 = orc.build_mem_plan(t, p.tolist())
        s2, l2, b2 = ctx.build_mem_plan(to_dev(t), p)
        assert (s2.cpu().numpy() == s1).all()
        assert (l2.cpu().numpy() == l1).all()
        assert b1 == b2


def test_build_mem_plan_rejects_non_consecutive(ctx, orc):
    from paper_2006_06608_b200.capi import DomainError
    from oracle.cpu import OracleError
    t = np.array([0, 0, 1, 0, 2], np.uint32)
    with pytest.raises(DomainError) as e:
        ctx.build_mem_plan(to_dev(t), P(tpb=64))
    with pytest.raises(OracleError) as e2:
        orc.build_mem_plan(t, P(tpb=64).tolist())
    assert e.value.msg == e2.value.msg


def test_aggregate_f64_bitwise_and_counters(ctx, orc):
    import torch
    for i, rp, col, x, params in corpus(1001, 60):
        drp, dcol, dx = to_dev(rp, col, x)
        for kw in params:
            p = P(**kw)
            for s in STRATS:
                plan = ctx.plan(drp, dcol, p, s)
                for m in MODES:
                    want, cost = orc.aggregate_scheduled(rp, col, x, p.tolist(), s, m, line=128, cache=None)
                    got = plan.aggregate(dx, dim_mode=m).cpu().numpy()
                    assert np.array_equal(got, want), (i, kw, s, m)
                    c = plan.cost(dim_mode=m, line=128)
                    assert c.tolist()[:5] == cost.tolist()[:5], (i, kw, s, m)


def test_aggregate_f32_tolerance(ctx, orc):
    import torch
    for i, rp, col, x, params in corpus(77, 30):
        drp, dcol = to_dev(rp, col)
        dx = to_dev(x.astype(np.float32))
        want = orc.aggregate_oracle(rp, col, x)
        for kw in params:
            plan = ctx.plan(drp, dcol, P(**kw), 2)
            got = plan.aggregate(dx).cpu().numpy().astype(np.float64)
            rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
            assert (np.abs(got - want) <= 1e-5 * np.abs(want)).all(), rel.max()


def test_cost_report_lines_and_cache(ctx, orc):
    rng = np.random.default_rng(29)
    for t in range(25):
        n = int(rng.integers(2, 120))
        rp, col, _ = random_graph(rng, n, 6 * n)
        dim = int(rng.choice([1, 3, 16, 32, 33, 64]))
        kw = dict(ngs=int(rng.integers(1, 9)), dw=int(rng.integers(1, 33)), tpb=32 * int(rng.integers(1, 9)),
                  dim=dim)
        x = rng.random((n, dim))
        drp, dcol = to_dev(rp, col)
        for s in STRATS:
            plan = ctx.plan(drp, dcol, P(**kw), s)
            for m in MODES:
                line = int(rng.choice([32, 100, 128, 4096]))
                cache = (int(rng.choice([1, 2, 8, 512])) * 128, 128) if t % 3 else (1 << 24, 128)
                _, want = orc.aggregate_scheduled(rp, col, x, P(**kw).tolist(), s, m, line=line, cache=cache)
                got = plan.cost(dim_mode=m, line=line, cache=cache)
                assert got.tolist() == want.tolist(), (t, kw, s, m, line, cache)


def test_aggregate_rows_is_oracle_order(ctx, orc):
    rng = np.random.default_rng(3)
    for t in range(20):
        n = int(rng.integers(1, 400))
        rp, col, _ = random_graph(rng, n, int(rng.integers(0, 10 * n)))
        dim = int(rng.choice([1, 2, 5, 16, 64, 128, 130]))
        x = rng.random((n, dim)) - 0.5
        want = orc.aggregate_oracle(rp, col, x)
        got = ctx.aggregate_rows(*to_dev(rp, col, x)).cpu().numpy()
        assert np.array_equal(got, want)


def test_aggregate_host_entry(ctx, orc):
    rng = np.random.default_rng(9)
    rp, col, _ = random_graph(rng, 500, 3000)
    x = rng.random((500, 16))
    for s in STRATS:
        p = P(ngs=4, dw=8, tpb=64, dim=16)
        y, cost = ctx.aggregate_host(rp, col, x, p, s, 1, cache=(64 * 1024, 128))
        want, wc = orc.aggregate_scheduled(rp, col, x, p.tolist(), s, 1, cache=(64 * 1024, 128))
        assert np.array_equal(y, want)
        assert cost.tolist() == wc.tolist()


def test_power_law_hubs_f32(ctx, orc):
    """Hubs spanning many schedule blocks exercise the carry + ordered fold."""
    rng = np.random.default_rng(11)
    n = 20000
    w = 1.0 / np.arange(1, n + 1) ** 0.8
    w /= w.sum()
    src = rng.choice(n, size=120000, p=w)
    dst = rng.integers(0, n, size=120000)
    edges = np.stack([src, dst], 1).astype(np.uint32)
    rp, col = orc.to_csr(n, edges, True)
    assert np.diff(rp).max() > 2000
    x = rng.random((n, 64))
    drp, dcol, dx = to_dev(rp, col, x)
    for kw in (dict(ngs=16, dw=32, tpb=128, dim=64), dict(ngs=3, dw=8, tpb=1024, dim=64),
               dict(ngs=256, dw=16, tpb=32, dim=64)):
        for s in STRATS:
            want, _ = orc.aggregate_scheduled(rp, col, x, P(**kw).tolist(), s, 1)
            plan = ctx.plan(drp, dcol, P(**kw), s)
            assert plan.info()["split_nodes"] > 0 or kw["ngs"] == 256
            got = plan.aggregate(dx).cpu().numpy()
            assert np.array_equal(got, want), (kw, s)
            got32 = plan.aggregate(dx.float()).cpu().numpy()
            assert (np.abs(got32 - want) <= 1e-5 * np.abs(want)).all()


def test_host_stream_matches_per_batch(ctx, orc):
    """gnna_aggregate_host_stream: pipelined batches (different graphs, row
    ranges and sizes) give exactly the per-batch results."""
    import torch
    rng = np.random.default_rng(31)
    p = P(ngs=8, dw=32, tpb=128, dim=16)
    batches, wants = [], []
    for t in range(5):
        n = int(rng.integers(50, 3000))
        rp, col, _ = random_graph(rng, n, 5 * n)
        r0 = int(rng.integers(0, n // 2))
        r1 = int(rng.integers(r0, n + 1))
        x = rng.random((n, 16))
        # a shard's schedule starts at its first row: the reference result is
        # aggregate_scheduled on the row-slice graph (rows x n CSR, full x)
        sub_rp = (rp[r0:r1 + 1] - rp[r0]).astype(np.uint64)
        sub_col = col[rp[r0]:rp[r1]].copy()
        want, _ = orc.aggregate_scheduled(sub_rp, sub_col, x, p.tolist(), 2, 1)
        want = np.concatenate([np.zeros((r0, 16)), want])
        out = torch.empty((r1 - r0, 16), dtype=torch.float64).pin_memory()
        batches.append((torch.from_numpy(rp.view(np.int64)).pin_memory(),
                        torch.from_numpy(col.view(np.int32)).pin_memory(),
                        torch.from_numpy(x).pin_memory(), r0, r1, out))
        wants.append(want[r0:r1])
    ctx.aggregate_host_stream(p, batches)
    for (_, _, _, _, _, out), want in zip(batches, wants):
        assert np.array_equal(out.numpy(), want)


def test_plan_info_runs_and_units(ctx, orc):
    """plan_info: units = partition_neighbors count, runs = Algorithm-1 leaders."""
    rng = np.random.default_rng(8)
    for t in range(10):
        n = int(rng.integers(1, 2000))
        rp, col, _ = random_graph(rng, n, int(rng.integers(0, 8 * n + 1)))
        kw = dict(ngs=int(rng.integers(1, 40)), dw=32, tpb=32 * int(rng.integers(1, 33)), dim=16)
        _, tg, _, _ = orc.partition_neighbors(rp, col, kw["ngs"])
        _, _, lead, _ = orc.build_mem_plan(tg, P(**kw).tolist()) if len(tg) else (None, None, np.zeros(0), 0)
        info = ctx.plan(*to_dev(rp, col), P(**kw), 2).info()
        assert info["groups"] == len(tg) and info["runs"] == int(np.sum(lead)), (t, info)


def test_l2_window_keeps_results(ctx, orc):
    """gnna_set_l2_window is a residency hint only: the pinned run is bit-identical."""
    import torch
    from paper_2006_06608_b200.capi import Params
    rng = np.random.default_rng(8)
    n = 4000
    rp, col, _ = random_graph(rng, n, 30000, orc=orc)
    drp, dcol = to_dev(rp, col)
    x = to_dev(rng.random((n, 64)))
    plan = ctx.plan(drp, dcol, Params.make(ngs=16, dw=16, tpb=256, dim=64), 2)
    want = plan.aggregate(x).clone()
    applied = ctx.set_l2_window(x, 1 << 20, 1.0)
    assert 0 < applied <= 1 << 20
    assert torch.equal(plan.aggregate(x), want)
    assert ctx.set_l2_window(None, 0) == 0
    assert torch.equal(plan.aggregate(x), want)
    # x smaller than L2: the data-driven pin leaves L2 alone
    assert ctx.pin_hot_rows(rp, x)["pinned"] is False


def test_capi_argument_checks(ctx, orc):
    """The ctypes layer refuses what the raw-pointer C-ABI cannot see: views,
    width mismatches against the plan, wrong dtypes."""
    from paper_2006_06608_b200.capi import Params
    rng = np.random.default_rng(1)
    rp, col, _ = random_graph(rng, 300, 1200, orc=orc)
    drp, dcol = to_dev(rp, col)
    plan = ctx.plan(drp, dcol, Params.make(ngs=8, dw=16, tpb=128, dim=16), 2)
    x = torch.rand((300, 32), device="cuda")
    with pytest.raises(ValueError):
        plan.aggregate(x)  # plan dim 16, x width 32
    with pytest.raises(ValueError):
        plan.aggregate(x[:, :16])  # a strided view
    with pytest.raises(TypeError):
        plan.aggregate(torch.zeros((300, 16), dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        plan.aggregate_ex(x, row_scale=torch.ones(299, device="cuda"))
    y = plan.aggregate_ex(x)  # aggregate_ex takes any width
    assert y.shape == x.shape


@pytest.mark.parametrize("nbytes", [1000, (4 << 20) - 4, 4 << 20, (21 << 20) + 12, 64 << 20])
def test_pageable_copies_staged(ctx, nbytes):
    """gnna_copy_to_device / gnna_copy_to_host with PAGEABLE host buffers:
    below 4 MiB the driver's own staging, from 4 MiB the context's pinned
    bounce ring (8 MiB chunks, threaded host copies, partial last chunk).
    Byte-exact round trip, through a device buffer the test also fills and
    reads with torch; the source may be overwritten as soon as the upload
    returns."""
    import ctypes as C
    rng = np.random.default_rng(nbytes)
    src = rng.integers(0, 256, nbytes, dtype=np.uint8)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    L = ctx.L
    ctx._check(L.gnna_copy_to_device(ctx.h, C.c_void_p(d.data_ptr()), C.c_void_p(src.ctypes.data), C.c_size_t(nbytes)))
    keep = src.copy()
    src[:] = 7  # the upload must not read the source after returning
    ctx.synchronize()
    assert np.array_equal(d.cpu().numpy(), keep)
    d2 = torch.from_numpy(rng.integers(0, 256, nbytes, dtype=np.uint8)).cuda()
    out = np.empty(nbytes, np.uint8)
    ctx._check(L.gnna_copy_to_host(ctx.h, C.c_void_p(out.ctypes.data), C.c_void_p(d2.data_ptr()), C.c_size_t(nbytes)))
    assert np.array_equal(out, d2.cpu().numpy())
