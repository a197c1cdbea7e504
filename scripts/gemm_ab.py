"""Skinny GEMM A/B on the C3 training shapes: libgnna K6 kernels vs cuBLAS
(torch.matmul, fp32, no TF32).  Median of 20 CUDA-event timings each."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_06608_b200.capi import Context  # noqa: E402
from paper_2006_06608_b200.gcn import ctx_gemm_tn  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False


def t(fn, reps=20, batch=10):
    """Median over `reps` of (CUDA-event time of `batch` back-to-back calls) / batch:
    the device time per call with host launch overhead overlapped."""
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(batch):
            fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1000 / batch)
    return float(np.median(ts))


def main():
    ctx = Context(0)
    m = 410236
    for (k, n) in ((96, 16), (22, 16), (16, 22), (64, 64)):
        x = torch.rand((m, k), device="cuda")
        w = torch.rand((k, n), device="cuda")
        dt = torch.rand((m, n), device="cuda")
        ideal = (m * k + m * n) * 4 / 6.5e12 * 1e6
        r = {"shape": f"{m}x{k} . {k}x{n}", "ideal_us": round(ideal, 1),
             "gnna_us": round(t(lambda: ctx.gemm(x, w)), 1),
             "cublas_us": round(t(lambda: torch.matmul(x, w)), 1),
             "gnna_tn_us": round(t(lambda: ctx_gemm_tn(ctx, x, dt)), 1),
             "cublas_tn_us": round(t(lambda: torch.matmul(x.t(), dt)), 1)}
        ref = x.double() @ w.double()
        r["gnna_relerr"] = float(((ctx.gemm(x, w) - ref).abs() / ref.abs().clamp_min(1e-6)).max())
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
