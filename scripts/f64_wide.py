"""fp64 K3 at C5 shape (d 128, natural Chung-Lu order = hubs first), tpb 512
(team 16, 4 chunks per lane) and tpb 128 (team 32): CUDA-event median of
5 calls.  GNNA_K3_F64_KMAX4=1 selects the single KMAX-4 pass."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_06608_b200 import synth  # noqa: E402
from paper_2006_06608_b200.capi import WARP_SHARED, Context, Params  # noqa: E402

dev = torch.device("cuda", 0)
ctx = Context(0)
cfg = synth.CONFIGS["c5"]
_, rp, col = synth.build_graph(cfg, lambda n, e: ctx.to_csr(n, e, True), dev)
x = synth.features(cfg.n, cfg.dim, cfg.seed, dev).double()
y = torch.empty_like(x)
for tpb in (512, 128):
    plan = ctx.plan(rp, col, Params.make(ngs=4096, dw=32, tpb=tpb, dim=128), WARP_SHARED)
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.aggregate(x, out=y)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(json.dumps({"tpb": tpb, "kmax4": bool(os.environ.get("GNNA_K3_F64_KMAX4")),
                      "ms": float(np.median(ts[2:]))}), flush=True)
