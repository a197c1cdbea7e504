"""The hub L2 window on a graph whose ids are shuffled: without a degree
order the front rows carry ~uniform gather share (no pin); after
gnna_degree_order + apply_mapping the hubs are in front again and the window
applies.  K3 times (CUDA events, median of 10) for C5."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_06608_b200 import synth  # noqa: E402
from paper_2006_06608_b200.capi import WARP_SHARED, Context  # noqa: E402


def time_k3(ctx, rp, col, x, dim):
    p, _ = ctx.b200_params(rp, dim)
    plan = ctx.plan(rp, col, p, WARP_SHARED)
    y = torch.empty_like(x)
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
    return float(np.median(ts))


dev = torch.device("cuda", 0)
ctx = Context(0)
cfg = synth.CONFIGS["c5"]
_, rp, col = synth.build_graph(cfg, lambda n, e: ctx.to_csr(n, e, True), dev)
x = synth.features(cfg.n, cfg.dim, cfg.seed, dev)
n = cfg.n
perm = torch.randperm(n, device=dev, generator=torch.Generator(device=dev).manual_seed(3)).int()
inv = torch.empty_like(perm)
inv[perm.long()] = torch.arange(n, device=dev, dtype=torch.int32)
rps, cols = ctx.apply_mapping_csr(rp, col, perm, inv)     # shuffled ids: old v -> perm[v]
xs = x[inv.long()].contiguous()
del rp, col, x
pin = ctx.pin_hot_rows(rps.cpu().numpy().view(np.uint64), xs)
t_shuf = time_k3(ctx, rps, cols, xs, cfg.dim)
ctx.set_l2_window(None, 0)
print(json.dumps({"graph": "C5 shuffled ids", "pin": pin, "k3_ms": round(t_shuf, 3)}), flush=True)
o2n, n2o = ctx.degree_order(rps)
rpd, cold = ctx.apply_mapping_csr(rps, cols, o2n, n2o)
xd = xs[n2o.long()].contiguous()
del rps, cols, xs
t_nopin = time_k3(ctx, rpd, cold, xd, cfg.dim)
pin = ctx.pin_hot_rows(rpd.cpu().numpy().view(np.uint64), xd)
t_pin = time_k3(ctx, rpd, cold, xd, cfg.dim)
ctx.set_l2_window(None, 0)
print(json.dumps({"graph": "C5 shuffled, then degree-ordered", "pin": pin, "k3_ms_no_window": round(t_nopin, 3),
                  "k3_ms_window": round(t_pin, 3)}), flush=True)
