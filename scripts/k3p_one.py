"""One C3 sum aggregation (3 warm-up calls + 1), for ncu captures of K3/K3P."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_06608_b200 import synth  # noqa: E402
from paper_2006_06608_b200.capi import WARP_SHARED, Context  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c3"
dev = torch.device("cuda", 0)
ctx = Context(0)
cfg = synth.CONFIGS[w]
_, rp, col = synth.build_graph(cfg, lambda n, e: ctx.to_csr(n, e, True), dev)
x = synth.features(cfg.n, cfg.dim, cfg.seed, dev)
p, _ = ctx.b200_params(rp, cfg.dim)
plan = ctx.plan(rp, col, p, WARP_SHARED)
y = torch.empty_like(x)
for _ in range(4):
    plan.aggregate(x, out=y)
torch.cuda.synchronize()
print(plan.info())
