"""K3 sweep for the B200 evaluator: per workload and dtype,
ngs x tpb, CUDA-event median of 7 calls (L2 flushed between calls when the
features fit in L2).  One JSON line per point, then the best."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2006_06608_b200 import synth  # noqa: E402
from paper_2006_06608_b200.capi import WARP_SHARED, Context, Params  # noqa: E402

dev = torch.device("cuda", 0)
ctx = Context(0)
scratch = bench.l2_flush_buffer(dev)
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
works = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c3", "c4", "c5"]
for w in works:
    cfg = synth.CONFIGS[w]
    _, rp, col = synth.build_graph(cfg, lambda n, e: ctx.to_csr(n, e, True), dev)
    if w == "c5":  # the bench's preprocessing: hubs first
        o2n, n2o = ctx.degree_order(rp)
        rp, col = ctx.apply_mapping_csr(rp, col, o2n, n2o)
    for dt in (torch.float32, torch.float64):
        x = synth.features(cfg.n, cfg.dim, cfg.seed, dev, dtype=dt)
        y = torch.empty_like(x)
        flush = x.numel() * x.element_size() < 4 * l2
        model, est = ctx.b200_params(rp, cfg.dim)
        best = None
        for tpb in (128, 256, 512):
            for ngs in (32, 64, 128, 256, 512, 1024, 2048, 4096):
                plan = ctx.plan(rp, col, Params.make(ngs=ngs, dw=32, tpb=tpb, dim=cfg.dim), WARP_SHARED)
                t = bench.time_calls(lambda: plan.aggregate(x, out=y), 7 if w != "c5" else 3,
                                     scratch if flush else None)
                rec = {"workload": w, "dtype": str(dt)[6:], "ngs": ngs, "tpb": tpb, "ms": round(t, 5)}
                print(json.dumps(rec), flush=True)
                if best is None or t < best["ms"]:
                    best = rec
                del plan
        print(json.dumps({"best": best, "model_pick": model.tolist()[:3], "model_est_us": est}), flush=True)
        del x, y
        torch.cuda.empty_cache()
