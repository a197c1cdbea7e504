"""GPU parity: graph utilities (to_csr, transpose, aes, degree stats) and
renumbering (detect_communities, modularity, build_mapping,
mapping_from_vector, apply_mapping) through the C-ABI, bit-exact against the
reference-produced vectors (tests/golden/) and the CPU oracle."""
import numpy as np
import pytest
import torch

from conftest import golden_cases, random_graph, to_dev

pytestmark = pytest.mark.gpu


def host(t, dtype):
    return t.cpu().numpy().view(dtype)


def test_to_csr_golden(ctx):
    g = golden_cases()
    for i in g.ids("csr"):
        n = int(g[f"csr/{i}/n"][0])
        edges = g[f"csr/{i}/edges"]
        rp, col = ctx.to_csr(n, to_dev(edges.reshape(-1, 2)) if len(edges) else torch.zeros((0, 2), dtype=torch.int32,
                                                                                              device="cuda"),
                             bool(g[f"csr/{i}/sym"][0]))
        assert np.array_equal(host(rp, np.uint64), g[f"csr/{i}/rp"])
        assert np.array_equal(host(col, np.uint32), g[f"csr/{i}/col"])


def test_to_csr_random_and_edge_cases(ctx, orc):
    rng = np.random.default_rng(12)
    for t in range(30):
        n = int(rng.integers(1, 3000))
        e = int(rng.integers(1, 20 * n))
        edges = rng.integers(0, n, size=(e, 2)).astype(np.uint32)
        sym = bool(t % 2)
        want_rp, want_col = orc.to_csr(n, edges, sym)
        rp, col = ctx.to_csr(n, to_dev(edges), sym)
        assert np.array_equal(host(rp, np.uint64), want_rp)
        assert np.array_equal(host(col, np.uint32), want_col)
    from paper_2006_06608_b200.capi import DomainError
    with pytest.raises(DomainError):
        ctx.to_csr(3, to_dev(np.array([[0, 5]], np.uint32)), True)


def test_transpose_aes_degree_stats(ctx, orc):
    rng = np.random.default_rng(4)
    for t in range(10):
        n = int(rng.integers(2, 2000))
        edges = rng.integers(0, n, size=(int(rng.integers(1, 10 * n)), 2)).astype(np.uint32)
        rp, col = orc.to_csr(n, edges, False)
        tp, tc = ctx.csr_transpose(*to_dev(rp, col))
        rt, ct = orc.to_csr(n, edges[:, ::-1].copy(), False)
        assert np.array_equal(host(tp, np.uint64), rt) and np.array_equal(host(tc, np.uint32), ct)
        assert ctx.aes(to_dev(edges)) == orc.aes(n, edges)
        a, m, s = ctx.degree_stats(to_dev(rp))
        a2, m2, s2 = orc.degree_stats(rp, col)
        assert a == a2 and m == m2 and abs(s - s2) <= 1e-12 * max(1.0, s2)


def test_renumber_golden(ctx):
    g = golden_cases()
    for i in g.ids("com"):
        rp, col, edges = g[f"com/{i}/rp"], g[f"com/{i}/col"], g[f"com/{i}/edges"]
        n = len(rp) - 1
        drp, dcol = to_dev(rp, col)
        com, k = ctx.detect_communities(drp, dcol)
        assert k == int(g[f"com/{i}/k"][0]) and np.array_equal(host(com, np.uint32), g[f"com/{i}/com"]), i
        assert ctx.modularity(drp, dcol, com, k) == float(g[f"com/{i}/q"][0])
        o2n, n2o = ctx.build_mapping(com, k)
        assert np.array_equal(host(o2n, np.uint32), g[f"com/{i}/o2n"])
        assert np.array_equal(host(n2o, np.uint32), g[f"com/{i}/n2o"])
        orp, ocol = ctx.apply_mapping_csr(drp, dcol, o2n, n2o)
        assert np.array_equal(host(orp, np.uint64), g[f"com/{i}/orp"])
        assert np.array_equal(host(ocol, np.uint32), g[f"com/{i}/ocol"])
        oe = ctx.apply_mapping_edges(to_dev(edges), n, o2n)
        assert np.array_equal(host(oe, np.uint32), g[f"com/{i}/oedges"])


def test_detect_communities_corpus(ctx, orc):
    """Random graphs (duplicates, self loops, isolated nodes) and planted
    partitions: the merge sequence must reproduce com_idx exactly."""
    rng = np.random.default_rng(300)
    for t in range(120):
        n = int(rng.integers(1, 400))
        rp, col, _ = random_graph(rng, n, int(rng.integers(0, 6 * n + 1)), orc=orc)
        want, k = orc.detect_communities(rp, col)
        got, k2 = ctx.detect_communities(*to_dev(rp, col))
        assert k == k2 and np.array_equal(host(got, np.uint32), want), t
    for seed in range(6):
        nn, edges = orc.planted_partition(6, 40, 0.3, 0.02, True, seed)
        rp, col = orc.to_csr(nn, edges, True)
        want, k = orc.detect_communities(rp, col)
        got, k2 = ctx.detect_communities(*to_dev(rp, col))
        assert k == k2 and np.array_equal(host(got, np.uint32), want)


def test_detect_communities_pubmed_shape(ctx):
    """C2 shape (19,717 nodes, 88.6k nnz, shuffled ids) against the
    reference's own output (tests/golden/c2_communities.npz, ~30 s of
    reference CPU time when generated), then the full renumbering chain."""
    import os
    from conftest import ROOT
    z = np.load(os.path.join(ROOT, "tests", "golden", "c2_communities.npz"))
    drp, dcol = to_dev(z["rp"], z["col"])
    got, k = ctx.detect_communities(drp, dcol)
    assert k == int(z["k"][0]) and np.array_equal(host(got, np.uint32), z["com"])
    assert ctx.modularity(drp, dcol, got, k) == float(z["q"][0])


def test_mapping_errors(ctx):
    from paper_2006_06608_b200.capi import DomainError
    with pytest.raises(DomainError) as e:
        ctx.mapping_from_vector(to_dev(np.array([0, 0, 1], np.uint32)))
    assert e.value.msg == "mapping is not a permutation of its index range"
    o2n, n2o = ctx.mapping_from_vector(to_dev(np.array([2, 1, 0], np.uint32)))
    assert host(n2o, np.uint32).tolist() == [2, 1, 0]
    rp, col = to_dev(np.array([0, 1, 2, 2], np.uint64), np.array([1, 0], np.uint32))
    bad = to_dev(np.array([0, 0, 1], np.uint32))
    with pytest.raises(DomainError):
        ctx.apply_mapping_csr(rp, col, bad, bad)


def test_degree_order_and_aggregation_equivalence(ctx, orc):
    """gnna_degree_order: descending degree, ties by old id (bit-exact vs a
    numpy stable sort); aggregating the renumbered graph on renumbered rows is
    the original aggregation permuted (fp64: identical bits per row, since each
    row's CSR order maps to the same neighbor sequence only up to the sort, so
    compare against the oracle on the renumbered CSR)."""
    import torch
    from conftest import random_graph, to_dev
    from paper_2006_06608_b200.capi import Params
    rng = np.random.default_rng(9)
    for n, e in ((1, 0), (50, 300), (3000, 20000)):
        rp, col, _ = random_graph(rng, n, e, orc=orc)
        drp, dcol = to_dev(rp, col)
        o2n, n2o = ctx.degree_order(drp)
        deg = np.diff(rp.astype(np.int64))
        want_n2o = np.lexsort((np.arange(n), -deg)).astype(np.uint32)
        assert np.array_equal(n2o.cpu().numpy().view(np.uint32), want_n2o)
        want_o2n = np.empty(n, np.uint32)
        want_o2n[want_n2o] = np.arange(n, dtype=np.uint32)
        assert np.array_equal(o2n.cpu().numpy().view(np.uint32), want_o2n)
        if e == 0:
            continue
        rp2, col2 = ctx.apply_mapping_csr(drp, dcol, o2n, n2o)
        x = rng.random((n, 16))
        x2 = x[want_n2o]
        p = Params.make(ngs=8, dw=16, tpb=128, dim=16)
        got = ctx.plan(rp2, col2, p, 2).aggregate(to_dev(x2)).cpu().numpy()
        want, _ = orc.aggregate_scheduled(rp2.cpu().numpy().view(np.uint64), col2.cpu().numpy().view(np.uint32), x2,
                                          p.tolist(), 2, 1)
        assert np.array_equal(got, want)
        # same sums as the original graph, row for row (to fp64 rounding of reordered adds)
        orig, _ = orc.aggregate_scheduled(rp, col, x, p.tolist(), 2, 1)
        np.testing.assert_allclose(got, orig[want_n2o], rtol=1e-12, atol=1e-12)
