"""K3 time per units-per-CTA cap (run once per GNNA_K3_UPC_MAX value): C3 / C4
sum in fp32 and fp64, B200-evaluator params, CUDA events, L2 flushed."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2006_06608_b200 import synth  # noqa: E402
from paper_2006_06608_b200.capi import WARP_SHARED, Context  # noqa: E402

dev = torch.device("cuda", 0)
ctx = Context(0)
scratch = bench.l2_flush_buffer(dev)
for w in ("c3", "c4"):
    cfg = synth.CONFIGS[w]
    _, rp, col = synth.build_graph(cfg, lambda n, e: ctx.to_csr(n, e, True), dev)
    x = synth.features(cfg.n, cfg.dim, cfg.seed, dev)
    for dt in (torch.float32, torch.float64):
        xx = x.to(dt)
        y = torch.empty_like(xx)
        p, _ = ctx.b200_params(rp, cfg.dim, dtype=dt)
        plan = ctx.plan(rp, col, p, WARP_SHARED)
        t = bench.time_calls(lambda: plan.aggregate(xx, out=y), 20, scratch)
        print(json.dumps({"upc_max": os.environ.get("GNNA_K3_UPC_MAX", "default"), "workload": w,
                          "dtype": str(dt).split(".")[-1], "ms": round(t, 4)}), flush=True)
