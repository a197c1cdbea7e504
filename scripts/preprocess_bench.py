"""Preprocessing stages on the GPU vs the reference CPU path (SURVEY §6, §8(a)
H2-H10): to_csr, K1/K2 plan build, renumbering (detect_communities,
modularity, build_mapping, apply_mapping).  One JSON line per stage.

  python scripts/preprocess_bench.py [--ref] [--skip-c4-communities]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2006_06608_b200 import synth  # noqa: E402
from paper_2006_06608_b200.capi import WARP_SHARED, Context, Params  # noqa: E402


def timed(fn, reps=1):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps, out


def emit(**kw):
    print(json.dumps(kw), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", action="store_true", help="also time the reference CPU path where it finishes")
    ap.add_argument("--skip-c4-communities", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    ctx = Context(0)
    ref = None
    if args.ref:
        from oracle.cpu import Oracle, available
        ref = Oracle("ref") if available("ref") else None

    # C5: to_csr + plan build
    cfg = synth.CONFIGS["c5"]
    edges = synth.sample_pairs(cfg, cfg.nnz // 2, cfg.seed, dev)
    ctx.to_csr(cfg.n, edges[:1000], True)  # warm up allocator / CUB
    t, (rp, col) = timed(lambda: ctx.to_csr(cfg.n, edges, True))
    emit(stage="to_csr", workload="c5", edges=int(edges.shape[0]), nnz=int(col.numel()), gpu_s=t)
    p = Params.make(ngs=256, dw=32, tpb=128, dim=128)
    ctx.plan(rp, col, p, WARP_SHARED)
    t, plan = timed(lambda: ctx.plan(rp, col, p, WARP_SHARED), reps=3)
    emit(stage="partition_neighbors+build_mem_plan (K1+K2)", workload="c5", units=plan.info()["groups"], gpu_s=t)
    del edges, rp, col, plan
    torch.cuda.empty_cache()

    for w in ("c2", "c4"):
        cfg = synth.CONFIGS[w]
        edges, rp, col = synth.build_graph(cfg, lambda n, e: ctx.to_csr(n, e, True), dev)
        if w == "c4" and args.skip_c4_communities:
            continue
        t, (com, k) = timed(lambda: ctx.detect_communities(rp, col))
        q = ctx.modularity(rp, col, com, k)
        rec = dict(stage="detect_communities (exact greedy)", workload=w, n=cfg.n, nnz=int(col.numel()),
                   communities=k, modularity=q, gpu_s=t)
        if ref is not None and w == "c2":
            rph, colh = rp.cpu().numpy().view(np.uint64), col.cpu().numpy().view(np.uint32)
            t0 = time.perf_counter()
            rc, rk = ref.detect_communities(rph, colh)
            rec["ref_cpu_s"] = time.perf_counter() - t0
            rec["bit_exact"] = bool(rk == k and np.array_equal(rc, com.cpu().numpy().view(np.uint32)))
        emit(**rec)
        t, (o2n, n2o) = timed(lambda: ctx.build_mapping(com, k), reps=5)
        emit(stage="build_mapping", workload=w, gpu_s=t)
        t, _ = timed(lambda: ctx.apply_mapping_csr(rp, col, o2n, n2o), reps=5)
        emit(stage="apply_mapping (CSR)", workload=w, gpu_s=t)
        e1 = ctx.aes(edges)
        e2 = ctx.aes(ctx.apply_mapping_edges(edges, cfg.n, o2n))
        emit(stage="aes before/after renumbering", workload=w, aes_before=e1, aes_after=e2)


if __name__ == "__main__":
    main()
