"""CPU: pin the oracle (oracle/gnnsim_oracle.c) to the reference.

1. Hand golden vectors transcribed from the reference's own unit tests
   (file:line cited per case).
2. Reference-produced vectors committed in tests/golden/ref_golden.npz
   (tests/golden/make_golden.py ran the unmodified reference, oracle/_ref).
3. Live differential runs against oracle/_ref on seeded corpora (skipped when
   /root/reference was absent at build time).
No GPU is used here."""
import numpy as np
import pytest

from oracle.cpu import Oracle, OracleError, available, model_inputs, params_arr

from conftest import golden_cases


# ------------------------------------------------------------ 1. hand goldens
def test_to_csr_goldens(orc):
    # test_graph.cpp:91-95 symmetrized path
    rp, col = orc.to_csr(3, [[0, 1], [1, 2]], True)
    assert rp.tolist() == [0, 1, 3, 4] and col.tolist() == [1, 0, 2, 1]
    # test_graph.cpp:97-101 dedup
    rp, col = orc.to_csr(2, [[0, 1], [0, 1]], False)
    assert rp.tolist() == [0, 1, 1] and col.tolist() == [1]


def test_partition_goldens(orc):
    # test_schedule.cpp:42-54: group (2, 1, (4, 6))
    rp, col = orc.to_csr(5, [[0, 1], [0, 2], [0, 3], [0, 4], [1, 2], [1, 4]], False)
    ids, tg, bg, en = orc.partition_neighbors(rp, col, 2)
    assert (ids[2], tg[2], bg[2], en[2]) == (2, 1, 4, 6)
    # test_schedule.cpp:56-69: degree 5, ngs 2 -> [2, 2, 1]
    rp, col = orc.to_csr(6, [[0, 1], [0, 2], [0, 3], [0, 4], [0, 5]], False)
    ids, tg, bg, en = orc.partition_neighbors(rp, col, 2)
    assert (en - bg).tolist() == [2, 2, 1] and ids.tolist() == [0, 1, 2] and tg.tolist() == [0, 0, 0]


def test_params_validation_goldens(orc):
    # test_schedule.cpp:29-40 / schedule.cpp:7-14
    orc.validate_params(params_arr())
    for bad in (params_arr(ngs=0), params_arr(tpw=16), params_arr(dw=0), params_arr(dw=33),
                params_arr(tpb=48), params_arr(tpb=2048), params_arr(dim=0)):
        with pytest.raises(OracleError) as e:
            orc.validate_params(bad)
        assert e.value.code == 1


def test_memplan_fixture(orc):
    # test_memplan.cpp:58-74 / acceptance.cpp:127-136 hand-traced Algorithm 1
    s, nodes, lead, smem = orc.build_mem_plan(np.array([0, 0, 1, 2, 2, 2], np.uint32),
                                              params_arr(tpb=64, dim=16))
    assert s.tolist() == [0, 0, 0, 1, 0, 0]
    assert lead.tolist() == [1, 0, 1, 1, 1, 0]
    assert smem == 2 * 16 * 4
    with pytest.raises(OracleError) as e:
        orc.build_mem_plan(np.array([0, 0, 1, 0], np.uint32), params_arr(tpb=64))
    assert e.value.code == 1


def test_oracle_values_golden(orc):
    # test_engine.cpp:98-104
    rp, col = orc.to_csr(3, [[0, 1], [1, 2]], True)
    x = np.array([[1.0, 2.0], [10.0, 20.0], [100.0, 200.0]])
    assert orc.aggregate_oracle(rp, col, x).ravel().tolist() == [10, 20, 101, 202, 10, 20]


def star(k):
    return orc_global().to_csr(k + 1, [[0, i] for i in range(1, k + 1)], True)


_ORC = None


def orc_global():
    global _ORC
    if _ORC is None:
        _ORC = Oracle("orc")
    return _ORC


def test_counter_goldens_star(orc):
    # test_engine.cpp:142-178: naive E*d, unit G*d, shared leaders*d
    k = 8
    rp, col = star(k)
    e = 2 * k
    for ngs in (1, 2, 4, 8):
        p = params_arr(ngs=ngs, dw=32, tpb=128, dim=16)
        x = np.ones((k + 1, 16))
        groups = k // ngs + k
        _, naive = orc.aggregate_scheduled(rp, col, x, p, 0, 1)
        _, unit = orc.aggregate_scheduled(rp, col, x, p, 1, 1)
        _, sh = orc.aggregate_scheduled(rp, col, x, p, 2, 1)
        assert naive[0] == e * 16 and naive[2] == e * 16 and naive[1] == e * 16 and naive[4] == 0
        assert unit[0] == groups * 16 and unit[1] == e * 16 and unit[4] == 0
        assert sh[4] == 4 * 16 * 4 and sh[1] == e * 16 and sh[0] == sh[2]
        assert sh[0] <= unit[0] <= naive[0]


def test_transaction_goldens(orc):
    # test_engine.cpp:232-254: dim 32 fills one line -> e + e / e + groups
    k = 8
    rp, col = star(k)
    p = params_arr(ngs=8, dw=32, tpb=128, dim=32)
    x = np.ones((k + 1, 32))
    e, groups = 2 * k, 1 + k
    assert orc.aggregate_scheduled(rp, col, x, p, 0, 1)[1][3] == e + e
    assert orc.aggregate_scheduled(rp, col, x, p, 1, 1)[1][3] == e + groups
    assert orc.aggregate_scheduled(rp, col, x, p, 2, 1)[1][3] == e + groups
    # test_engine.cpp:256-268: cyclic 8, sequential 16
    rp, col = orc.to_csr(2, [[0, 1]], True)
    p = params_arr(ngs=4, dw=32, tpb=32, dim=64)
    x = np.ones((2, 64))
    assert orc.aggregate_scheduled(rp, col, x, p, 1, 1)[1][3] == 8
    assert orc.aggregate_scheduled(rp, col, x, p, 1, 0)[1][3] == 16


def test_lru_goldens(orc):
    # test_engine.cpp:297-318 rows 10,11,10,12,10 in one block
    rp = np.array([0, 1, 2, 3, 4, 5] + [5] * 8, np.uint64)
    col = np.array([10, 11, 10, 12, 10], np.uint32)
    p = params_arr(ngs=1, dw=32, tpb=256, dim=32)
    assert orc.simulate_cache(rp, col, p, (2 * 128, 128), 32) == (2, 5)
    assert orc.simulate_cache(rp, col, p, (128, 128), 32)[0] == 0
    assert orc.simulate_cache(rp, col, p, (64 * 1024, 128), 32)[0] == 2
    # test_engine.cpp:320-333 resets at block boundaries (wpb 1)
    assert orc.simulate_cache(rp, col, params_arr(ngs=1, dw=32, tpb=32, dim=32), (64 * 1024, 128), 32) == (0, 5)
    # test_engine.cpp:335-348 dim 64 rows span two lines
    rp2 = np.array([0, 1, 2, 2], np.uint64)
    col2 = np.array([2, 2], np.uint32)
    assert orc.simulate_cache(rp2, col2, params_arr(ngs=1, dw=32, tpb=64, dim=64), (64 * 1024, 128), 64) == (2, 4)


def test_renumber_goldens(orc):
    # test_renumber.cpp:153-166 mapping goldens
    o2n, n2o = orc.build_mapping(np.array([1, 0, 1, 0], np.uint32), 2)
    assert o2n.tolist() == [2, 0, 3, 1]
    o2n, _ = orc.mapping_from_vector(np.array([2, 1, 0], np.uint32))
    assert o2n.tolist() == [2, 1, 0]
    with pytest.raises(OracleError):
        orc.mapping_from_vector(np.array([0, 0, 1], np.uint32))
    # test_renumber.cpp:139-151 modularity 5/14 of two triangles joined by an edge
    rp, col = orc.to_csr(6, [[0, 1], [1, 2], [0, 2], [3, 4], [4, 5], [3, 5], [2, 3]], True)
    q = orc.modularity(rp, col, np.array([0, 0, 0, 1, 1, 1], np.uint32), 2)
    assert abs(q - 5.0 / 14.0) < 1e-12
    # test_renumber.cpp:81-93: two 4-cliques joined by one edge -> 2 communities
    e = [[a, b] for a in range(4) for b in range(a + 1, 4)] + [[a, b] for a in range(4, 8) for b in range(a + 1, 8)]
    rp, col = orc.to_csr(8, e + [[3, 4]], True)
    com, k = orc.detect_communities(rp, col)
    assert k == 2 and com.tolist() == [0, 0, 0, 0, 1, 1, 1, 1]


# ----------------------------------------------------- 2. reference vectors
def test_golden_csr_and_partition(orc):
    g = golden_cases()
    for i in g.ids("csr"):
        rp, col = orc.to_csr(int(g[f"csr/{i}/n"][0]), g[f"csr/{i}/edges"], bool(g[f"csr/{i}/sym"][0]))
        assert np.array_equal(rp, g[f"csr/{i}/rp"]) and np.array_equal(col, g[f"csr/{i}/col"])
    for i in g.ids("part"):
        rp = g[f"part/{i}/rp"]
        _, tg, bg, en = orc.partition_neighbors(rp, np.zeros(int(rp[-1]), np.uint32), int(g[f"part/{i}/ngs"][0]))
        assert np.array_equal(tg, g[f"part/{i}/target"])
        assert np.array_equal(bg, g[f"part/{i}/begin"]) and np.array_equal(en, g[f"part/{i}/end"])


def test_golden_memplan(orc):
    g = golden_cases()
    for i in g.ids("plan"):
        s, _, lead, smem = orc.build_mem_plan(g[f"plan/{i}/targets"], g[f"plan/{i}/params"])
        assert np.array_equal(s, g[f"plan/{i}/slot"]) and np.array_equal(lead, g[f"plan/{i}/leader"])
        assert smem == int(g[f"plan/{i}/smem"][0])


def test_golden_aggregate_bitwise(orc):
    g = golden_cases()
    for i in g.ids("agg"):
        rp, col, x, p = g[f"agg/{i}/rp"], g[f"agg/{i}/col"], g[f"agg/{i}/x"], g[f"agg/{i}/params"]
        line, cache = int(g[f"agg/{i}/line"][0]), tuple(int(v) for v in g[f"agg/{i}/cache"])
        for s in (0, 1, 2):
            for m in (0, 1):
                y, cost = orc.aggregate_scheduled(rp, col, x, p, s, m, line=line, cache=cache)
                assert np.array_equal(y, g[f"agg/{i}/y_{s}{m}"]), (i, s, m)
                assert np.array_equal(cost, g[f"agg/{i}/cost_{s}{m}"]), (i, s, m)
        assert np.array_equal(orc.aggregate_oracle(rp, col, x), g[f"orc/{i}/y"])


def test_golden_layers_bitwise(orc):
    g = golden_cases()
    for i in g.ids("gcn"):
        rp, col, x, w = g[f"gcn/{i}/rp"], g[f"gcn/{i}/col"], g[f"gcn/{i}/x"], g[f"gcn/{i}/w"]
        sl = bool(g[f"gcn/{i}/self_loops"][0])
        assert np.array_equal(orc.gcn_layer(rp, col, x, w, sl), g[f"gcn/{i}/y"]), i
        eps = float(g[f"gin/{i}/eps"][0])
        assert np.array_equal(orc.gin_layer(rp, col, x, eps, w, g[f"gin/{i}/b"]), g[f"gin/{i}/y"]), i


def test_golden_renumbering(orc):
    g = golden_cases()
    for i in g.ids("com"):
        rp, col, edges = g[f"com/{i}/rp"], g[f"com/{i}/col"], g[f"com/{i}/edges"]
        com, k = orc.detect_communities(rp, col)
        assert np.array_equal(com, g[f"com/{i}/com"]) and k == int(g[f"com/{i}/k"][0])
        assert orc.modularity(rp, col, com, k) == float(g[f"com/{i}/q"][0])
        o2n, n2o = orc.build_mapping(com, k)
        assert np.array_equal(o2n, g[f"com/{i}/o2n"]) and np.array_equal(n2o, g[f"com/{i}/n2o"])
        orp, ocol = orc.apply_mapping_csr(rp, col, o2n, n2o)
        assert np.array_equal(orp, g[f"com/{i}/orp"]) and np.array_equal(ocol, g[f"com/{i}/ocol"])
        n = len(rp) - 1
        assert np.array_equal(orc.apply_mapping_edges(n, edges, o2n, n2o), g[f"com/{i}/oedges"])
        assert orc.aes(n, edges) == float(g[f"aes/{i}/aes"][0])
        a, m, s = orc.degree_stats(rp, col)
        want = g[f"aes/{i}/stats"]
        assert a == want[0] and m == want[1] and abs(s - want[2]) <= 1e-12 * max(1.0, want[2])


# ------------------------------------------------ 3. live differential runs
needs_ref = pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")


@needs_ref
def test_differential_aggregate(orc, ref):
    rng = np.random.default_rng(1001)
    for t in range(60):
        n = int(rng.integers(1, 300))
        edges = rng.integers(0, n, size=(int(rng.integers(0, 12 * n + 1)), 2)).astype(np.uint32)
        rp, col = ref.to_csr(n, edges, True)
        r2, c2 = orc.to_csr(n, edges, True)
        assert np.array_equal(rp, r2) and np.array_equal(col, c2)
        dim = int(rng.choice([1, 2, 7, 16, 32, 33, 64]))
        x = rng.random((n, dim))
        p = params_arr(ngs=1 + int(rng.integers(0, 64)), dw=1 + int(rng.integers(0, 32)),
                       tpb=32 * (1 + int(rng.integers(0, 32))), dim=dim)
        s, m = int(rng.integers(0, 3)), int(rng.integers(0, 2))
        cache = None if t % 3 == 0 else (int(rng.choice([1, 4, 64])) * 128, int(rng.choice([32, 128])))
        line = int(rng.choice([32, 64, 128]))
        y1, c1 = ref.aggregate_scheduled(rp, col, x, p, s, m, workers=3, line=line, cache=cache)
        y2, c2 = orc.aggregate_scheduled(rp, col, x, p, s, m, line=line, cache=cache)
        assert np.array_equal(y1, y2) and np.array_equal(c1, c2), t


@needs_ref
def test_differential_layers_and_renumber(orc, ref):
    rng = np.random.default_rng(77)
    for t in range(20):
        n = int(rng.integers(2, 90))
        edges = rng.integers(0, n, size=(int(rng.integers(1, 5 * n)), 2)).astype(np.uint32)
        rp, col = ref.to_csr(n, edges, True)
        din, dout = int(rng.integers(1, 20)), int(rng.integers(1, 20))
        x = rng.random((n, din)) - 0.5
        w = rng.random((din, dout)) - 0.5
        b = rng.random(dout) - 0.5
        assert np.array_equal(ref.gcn_layer(rp, col, x, w, t % 2 == 0), orc.gcn_layer(rp, col, x, w, t % 2 == 0))
        assert np.array_equal(ref.gin_layer(rp, col, x, 0.1, w, b), orc.gin_layer(rp, col, x, 0.1, w, b))
        c1, k1 = ref.detect_communities(rp, col)
        c2, k2 = orc.detect_communities(rp, col)
        assert k1 == k2 and np.array_equal(c1, c2)
        assert ref.modularity(rp, col, c1, k1) == orc.modularity(rp, col, c2, k2)
        assert ref.aes(n, edges) == orc.aes(n, edges)


# ------------------------------------- backward: parity pinned by the reference forward
@needs_ref
@pytest.mark.parametrize("layer", ["gcn", "gcn_sl", "gin"])
def test_backward_finite_differences_of_reference(orc, ref, layer):
    """No reference backward exists.  The oracle's analytic
    gradients are pinned by central differences of the REFERENCE forward
    (gcn_layer / gin_layer from oracle/_ref) of L = sum(dy * y)."""
    rng = np.random.default_rng(hash(layer) % 1000)
    for t in range(4):
        n = int(rng.integers(3, 40))
        edges = rng.integers(0, n, size=(int(rng.integers(n, 4 * n)), 2)).astype(np.uint32)
        rp, col = ref.to_csr(n, edges, True)
        din, dout = (6, 3) if t % 2 else (3, 6)
        x = rng.random((n, din)) - 0.5
        w = rng.random((din, dout)) - 0.5
        b = rng.random(dout) - 0.5
        dy = rng.random((n, dout)) - 0.5
        eps = 0.15
        if layer == "gin":
            f = lambda xx, ww: float((dy * ref.gin_layer(rp, col, xx, eps, ww, b)).sum())  # noqa: E731
            gx, gw, _, _ = orc.gin_backward(rp, col, x, eps, w, b, dy)
        else:
            sl = layer == "gcn_sl"
            f = lambda xx, ww: float((dy * ref.gcn_layer(rp, col, xx, ww, sl)).sum())  # noqa: E731
            gx, gw = orc.gcn_backward(rp, col, x, w, dy, sl)
        h = 1e-6
        for _ in range(6):
            i, j = int(rng.integers(0, n)), int(rng.integers(0, din))
            xp, xm = x.copy(), x.copy()
            xp[i, j] += h
            xm[i, j] -= h
            assert (f(xp, w) - f(xm, w)) / (2 * h) == pytest.approx(gx[i, j], rel=1e-5, abs=1e-7)
            i, j = int(rng.integers(0, din)), int(rng.integers(0, dout))
            wp, wm = w.copy(), w.copy()
            wp[i, j] += h
            wm[i, j] -= h
            assert (f(x, wp) - f(x, wm)) / (2 * h) == pytest.approx(gw[i, j], rel=1e-5, abs=1e-7)
