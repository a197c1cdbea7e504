"""A/B of the L2 access-policy window over the front (hub) rows of x for the
C5 gather: K3 time per window size / hit ratio (CUDA events, 10 reps)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_06608_b200 import synth  # noqa: E402
from paper_2006_06608_b200.capi import WARP_SHARED, Context  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c5"
dev = torch.device("cuda", 0)
ctx = Context(0)
cfg = synth.CONFIGS[w]
_, rp, col = synth.build_graph(cfg, lambda n, e: ctx.to_csr(n, e, True), dev)
x = synth.features(cfg.n, cfg.dim, cfg.seed, dev)
y = torch.empty_like(x)
p, _ = ctx.b200_params(rp, cfg.dim)
plan = ctx.plan(rp, col, p, WARP_SHARED)
nnz = int(col.numel())
print(json.dumps({"l2_bytes": torch.cuda.get_device_properties(dev).L2_cache_size}))
for mb, hr in [tuple(float(v) for v in a.split(":")) for a in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0:1", "32:1", "64:1", "0:1"])]:
    mb = int(mb)
    applied = ctx.set_l2_window(x if mb else None, mb << 20, hr)
    for _ in range(2):
        plan.aggregate(x, out=y)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.aggregate(x, out=y)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = float(np.median(ts))
    print(json.dumps({"window_MB": mb, "applied": applied, "hit_ratio": hr, "ms": round(t, 3),
                      "T_edge_dim_s": round(nnz * cfg.dim / t / 1e9, 1)}), flush=True)
ctx.set_l2_window(None, 0)
