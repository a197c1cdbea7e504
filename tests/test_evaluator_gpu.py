"""The B200 performance evaluator (north-star subsystem 3)
against the measured-latency tuner on the device.

gnna_tune_params times K3 with CUDA events over a parameter grid on the live
graph (the measured alternative to decider.cpp's analytic latency model);
gnna_b200_plan_params is the analytic B200 model over the device's SM
count, L2 size and measured HBM bandwidth and the graph's degree profile.
The model's pick must run within 5 % of the tuned optimum on the BASELINE
configs C3 (power law, d 16) and C4 (dense communities, d 64)."""
import pytest

pytestmark = pytest.mark.gpu

GS = (32, 64, 128, 256, 512, 1024, 2048, 4096)
TPB = (128, 256, 512)


@pytest.mark.parametrize("workload", ["c3", "c4"])
def test_model_pick_within_5pct_of_tuned_optimum(ctx, workload):
    import torch
    from paper_2006_06608_b200 import synth
    from paper_2006_06608_b200.capi import Decider
    cfg = synth.CONFIGS[workload]
    _, rp, col = synth.build_graph(cfg, lambda n, e: ctx.to_csr(n, e, True), torch.device("cuda", 0))
    dw = Decider().select_dw(cfg.dim)
    p, est_us, window = ctx.b200_params(rp, cfg.dim, window=True)
    assert p.tpb == 512 and p.dw == dw and p.ngs in GS and est_us > 0
    assert window == 0  # x fits in L2: no hub window
    best_ms = min(ctx.tune_params(rp, col, cfg.dim, gs=GS, dw=(dw,), tpb=TPB)[1] for _ in range(2))
    model_ms = min(ctx.tune_params(rp, col, cfg.dim, gs=(p.ngs,), dw=(dw,), tpb=(p.tpb,))[1] for _ in range(3))
    assert model_ms <= 1.05 * best_ms + 1e-3, (p.tolist(), model_ms, best_ms)


def test_window_recommendation_on_a_power_law_graph_beyond_l2(ctx):
    """x above the L2 (2M nodes x 128 fp32 = 1 GB) on a Chung-Lu graph with
    its hubs drawing far more than their uniform share: the evaluator
    recommends the 48 MB hub window; on a uniform graph it does not."""
    import numpy as np
    import torch
    from paper_2006_06608_b200 import capi
    n = 2_000_000
    e = capi.gen_edges("chung_lu", n, 10_000_000, 21)
    rp, _ = ctx.to_csr(n, torch.from_numpy(e.view(np.int32)).cuda(), True)
    _, _, window = ctx.b200_params(rp, 128, window=True)
    assert window == 48 << 20
    u = capi.gen_edges("sbm", n, 10_000_000, 22, communities=1, p_intra=0.0)
    rpu, _ = ctx.to_csr(n, torch.from_numpy(u.view(np.int32)).cuda(), True)
    _, _, window = ctx.b200_params(rpu, 128, window=True)
    assert window == 0
