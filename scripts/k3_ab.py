"""K3 A/B timing harness (GPU): per workload, build the graph once, then time
the scheduled aggregation for several parameter sets.  Each rep is timed
alone with CUDA events; for L2-sized inputs a 2xL2 scratch write flushes L2
between reps.  Prints one JSON line per (workload, params).

  python scripts/k3_ab.py --workloads c3,c4,c5 --params 256/32/128,16/32/128 [--dtype f32]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2006_06608_b200 import synth  # noqa: E402
from paper_2006_06608_b200.capi import WARP_SHARED, Context, Params  # noqa: E402
from bench import Clocks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="c3,c4,c5")
    ap.add_argument("--params", default="auto")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    ctx = Context(0)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    scratch = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    for w in args.workloads.split(","):
        cfg = synth.CONFIGS[w]
        _, rp, col = synth.build_graph(cfg, lambda n, e: ctx.to_csr(n, e, True), dev)
        dt = torch.float32 if args.dtype == "f32" else torch.float64
        x = synth.features(cfg.n, cfg.dim, cfg.seed, dev, dtype=dt)
        y = torch.zeros_like(x)
        nnz = int(col.numel())
        flush = x.numel() * x.element_size() < 4 * l2
        plist = []
        for ps in args.params.split(","):
            if ps == "auto":
                p = ctx.auto_params(ctx.model_inputs(rp, cfg.dim, b200=True))
            elif ps == "b200":
                p, _ = ctx.b200_params(rp, cfg.dim)
            else:
                g, d, t = (int(v) for v in ps.split("/"))
                p = Params.make(ngs=g, dw=d, tpb=t, dim=cfg.dim)
            plist.append(p)
        for p in plist:
            plan = ctx.plan(rp, col, p, WARP_SHARED)
            for _ in range(3):
                plan.aggregate(x, out=y)
            ts = []
            clk = Clocks(0).__enter__()
            for _ in range(args.reps):
                if flush:
                    scratch.fill_(1.0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                plan.aggregate(x, out=y)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            clk.__exit__(None, None, None)
            cs = clk.summary()
            t = float(np.median(ts))
            balg = synth.b_alg(cfg.n, nnz, cfg.dim, x.element_size())
            print(json.dumps({"tag": args.tag, "workload": w, "params": p.tolist()[:3], "ms": round(t, 5),
                              "Gedps": round(nnz * cfg.dim / t / 1e6, 1),
                              "balg_GBps": round(balg / t / 1e6, 1), "frac": round(balg / t / 1e6 / peak, 3),
                              "flush": flush, "min_ms": round(min(ts), 5), "max_ms": round(max(ts), 5),
                              "sm_mhz": cs.get("sm_mhz"), "power": cs.get("power_w_max"),
                              "reasons": cs.get("reasons"), "info": plan.info()}), flush=True)
            del plan
        del x, y, rp, col
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
