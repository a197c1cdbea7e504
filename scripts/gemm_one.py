"""One skinny GEMM shape, a few launches (for ncu captures): m k n [reps] [tn]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_06608_b200.capi import Context  # noqa: E402

m, k, n = (int(v) for v in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
tn = len(sys.argv) > 5 and sys.argv[5] == "tn"
ctx = Context(0)
x = torch.rand((m, k), device="cuda")
w = torch.rand((k, n), device="cuda") if not tn else torch.rand((m, n), device="cuda")
for _ in range(reps):
    if tn:
        from paper_2006_06608_b200.gcn import ctx_gemm_tn
        y = ctx_gemm_tn(ctx, x, w)
    else:
        y = ctx.gemm(x, w)
torch.cuda.synchronize()
print("ok", float(y.sum()))
