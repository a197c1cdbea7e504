"""GPU runs of BASELINE configs C1 and C2 at config size against the
reference itself (oracle/_ref: the unmodified reference compiled from its
sources, run live on the box's CPU), on the SAME synthetic inputs: both arms
take their edges from gnna_gen_sbm (mt19937_64 + rand.hpp draws) and their
features from random_features (pipeline.cpp:57-67).

* C1 (Cora shape, 2,708 nodes, d 16): GCN aggregation.  The F64 layer entry
  (gcn_forward with W = I: normalized_aggregate then an identity matmul) is
  bitwise equal to the reference's gcn_layer; the fp32 fused K3 form is
  within 1e-5.
* C2 (Pubmed shape, 19,717 nodes, ids shuffled, d 64): the reference's
  run_pipeline(force_reorder = true) -- detect_communities, build_mapping,
  apply_mapping, to_csr, auto_params, aggregate_scheduled with the LRU cache
  replay -- against the same chain through the C-ABI on the GPU: mapping,
  community count, modularity, AES after, parameters, every CostReport
  counter and the fp64 output bit for bit; then the GIN sum (eps 0) on the
  renumbered graph in fp32 within 1e-5.
"""
import numpy as np
import pytest
import torch

from conftest import to_dev

pytestmark = pytest.mark.gpu


def host(t, dt):
    return t.cpu().numpy().view(dt)


def edges_of(name):
    from paper_2006_06608_b200 import capi, synth
    cfg = synth.CONFIGS[name]
    e = capi.gen_edges(cfg.kind, cfg.n, cfg.nnz // 2, cfg.seed, shuffle=cfg.shuffle, gamma=cfg.gamma, i0=cfg.i0,
                       communities=cfg.communities, p_intra=cfg.p_intra)
    return cfg, e


def test_c1_gcn_aggregation_vs_reference(ctx, ref):
    from paper_2006_06608_b200.capi import WARP_SHARED, random_features
    cfg, e = edges_of("c1")
    rp, col = ref.to_csr(cfg.n, e, True)
    drp, dcol = ctx.to_csr(cfg.n, to_dev(e.view(np.int32)), True)
    assert np.array_equal(host(drp, np.uint64), rp) and np.array_equal(host(dcol, np.uint32), col)
    x = random_features(cfg.n, cfg.dim, 11, np.float64)
    assert np.array_equal(x, ref.random_features(cfg.n, cfg.dim, 11))  # the same features on both arms
    eye = np.eye(cfg.dim)
    for self_loops in (False, True):
        want = ref.gcn_layer(rp, col, x, eye, self_loops)  # = normalized_aggregate (engine.cpp:338-369)
        got = ctx.gcn_forward(drp, dcol, to_dev(x), to_dev(eye), self_loops).cpu().numpy()
        assert np.array_equal(got, want), self_loops
        # fp32: the fused K3 form (gathered norm[u], self weight, row scale)
        p, _ = ctx.b200_params(drp, cfg.dim)
        plan = ctx.plan(drp, dcol, p, WARP_SHARED)
        rs, sw, _ = ctx.gcn_weights(drp, dcol, self_loops, edge_weights=False)
        got32 = plan.aggregate_ex(to_dev(x.astype(np.float32)), node_weight=rs, self_weight=sw,
                                  row_scale=rs).cpu().numpy()
        want32 = ref.gcn_layer(rp, col, x.astype(np.float32).astype(np.float64), eye, self_loops)
        assert (np.abs(got32 - want32) <= 1e-5 * np.abs(want32) + 1e-30).all(), self_loops


def test_c2_run_pipeline_vs_reference(ctx, ref, orc):
    from paper_2006_06608_b200.capi import DIM_CYCLIC, WARP_SHARED, random_features
    cfg, e = edges_of("c2")
    n, dim, seed = cfg.n, cfg.dim, 5
    want = ref.run_pipeline(n, e, dim, force_reorder=True, seed=seed)  # ~20 s of reference CPU
    assert want["reordered"]
    # the same chain through the C-ABI, every stage on the GPU
    de = to_dev(e.view(np.int32))
    rp0, col0 = ctx.to_csr(n, de, True)
    com, ncom = ctx.detect_communities(rp0, col0)
    assert ncom == want["num_communities"]
    assert ctx.modularity(rp0, col0, com, ncom) == want["modularity"]
    o2n, n2o = ctx.build_mapping(com, ncom)
    assert np.array_equal(host(o2n, np.uint32), want["o2n"])
    moved = ctx.apply_mapping_edges(de, n, o2n)
    assert ctx.aes(de) == want["aes_before"] and ctx.aes(moved) == want["aes_after"]
    rp, col = ctx.to_csr(n, moved, True)
    p = ctx.auto_params(ctx.model_inputs(rp, dim))  # decider.cpp auto_params on the renumbered graph
    assert p.tolist() == want["params"]
    x = random_features(n, p.dim, seed, np.float64)
    plan = ctx.plan(rp, col, p, WARP_SHARED)
    y = plan.aggregate(to_dev(x)).cpu().numpy()
    assert np.array_equal(y, want["output"])  # fp64: the reference's summation tree, bit for bit
    cost = plan.cost(DIM_CYCLIC, 128, (64 * 1024, 128)).tolist()
    assert cost == want["report"]
    # GIN sum (eps 0) on the renumbered graph, fp32 K3 with the self term fused
    rph, colh = host(rp, np.uint64), host(col, np.uint32)
    got = plan.aggregate_ex(to_dev(x.astype(np.float32)), alpha=1.0).cpu().numpy()
    x32 = x.astype(np.float32).astype(np.float64)
    want_gin = ref.aggregate_oracle(rph, colh, x32) + x32
    assert (np.abs(got - want_gin) <= 1e-5 * np.abs(want_gin) + 1e-30).all()
