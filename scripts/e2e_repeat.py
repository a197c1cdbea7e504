"""e2e (host-buffer stream entry) repeated on one box: distribution of ms/step."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_06608_b200 import synth  # noqa: E402
from paper_2006_06608_b200.capi import Context  # noqa: E402

dev = torch.device("cuda", 0)
ctx = Context(0)
cfg = synth.CONFIGS["c5"]
_, rp, col = synth.build_graph(cfg, lambda n, e: ctx.to_csr(n, e, True), dev)
x = synth.features(cfg.n, cfg.dim, cfg.seed, dev)
p, _ = ctx.b200_params(rp, cfg.dim)
if len(sys.argv) > 1 and sys.argv[1] == "pin":
    print(ctx.pin_hot_rows(rp.cpu().numpy().view("uint64"), x))
    ctx.set_l2_window(None, 0)
h_rp, h_col, h_x = rp.cpu().pin_memory(), col.cpu().pin_memory(), x.cpu().pin_memory()
h_y = torch.empty((cfg.n, cfg.dim), dtype=torch.float32).pin_memory()
batches = [(h_rp, h_col, h_x, 0, cfg.n, h_y)] * 8
ctx.aggregate_host_stream(p, batches[:2])
for rep in range(4):
    t0 = time.perf_counter()
    ctx.aggregate_host_stream(p, batches)
    print(json.dumps({"rep": rep, "ms_per_step": round((time.perf_counter() - t0) / 8 * 1e3, 1)}), flush=True)
