"""One skinny GEMM shape, a few launches (for ncu captures): m k n [reps]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_06608_b200.capi import Context  # noqa: E402

m, k, n = (int(v) for v in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
ctx = Context(0)
x = torch.rand((m, k), device="cuda")
w = torch.rand((k, n), device="cuda")
for _ in range(reps):
    y = ctx.gemm(x, w)
torch.cuda.synchronize()
print("ok", float(y.sum()))
