"""C3 output-layer backward (gnna_dense_backward, 410k x 22 -> 16) x4, for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_06608_b200.capi import Context  # noqa: E402

ctx = Context(0)
m = 410236
dy = torch.rand((m, 22), device="cuda") - 0.5
w = torch.rand((16, 22), device="cuda") - 0.5
z = torch.rand((m, 16), device="cuda")
s = torch.rand(m, device="cuda", dtype=torch.float64)
for _ in range(4):
    ctx.dense_backward(dy, w, z, s)
torch.cuda.synchronize()
