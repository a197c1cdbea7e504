"""torch.autograd bindings of the layer entry points, so GCN/GIN layers built
on libgnna train inside ordinary PyTorch code (the role GNNAdvisor's
extension plays for its users).

Forward: gnna_gcn_forward / gnna_gin_forward (gcn_layer / gin_layer,
engine.cpp:373-408).  Backward: gnna_gcn_backward / gnna_gin_backward (the
added entry points; Â^T = Â on the symmetric CSR to_csr(.., true) builds;
pass the transposed CSR otherwise).  fp64 tensors run the bitwise reference
order, fp32 the scheduled fast path.  torch supplies tensors and autograd
bookkeeping only; every FLOP runs in libgnna.so.
"""
from __future__ import annotations

import torch

from .capi import Context


class GCNConvFn(torch.autograd.Function):
    @staticmethod
    def forward(fctx, gctx: Context, row_ptr, col, x, w, self_loops: bool, rt):
        y = gctx.gcn_forward(row_ptr, col, x.contiguous(), w.contiguous(), self_loops)
        fctx.save_for_backward(x, w)
        fctx.graph = (gctx, row_ptr, col, self_loops, rt)
        return y

    @staticmethod
    def backward(fctx, dy):
        x, w = fctx.saved_tensors
        gctx, row_ptr, col, self_loops, rt = fctx.graph
        dx, dw = gctx.gcn_backward(row_ptr, col, x.contiguous(), w.contiguous(), dy.contiguous(), self_loops, rt=rt)
        return None, None, None, dx, dw, None, None


class GINConvFn(torch.autograd.Function):
    @staticmethod
    def forward(fctx, gctx: Context, row_ptr, col, x, eps: float, w, b, rt):
        y = gctx.gin_forward(row_ptr, col, x.contiguous(), eps, w.contiguous(), b.contiguous())
        fctx.save_for_backward(x, w, b)
        fctx.graph = (gctx, row_ptr, col, eps, rt)
        return y

    @staticmethod
    def backward(fctx, dy):
        x, w, b = fctx.saved_tensors
        gctx, row_ptr, col, eps, rt = fctx.graph
        dx, dw, db, _deps = gctx.gin_backward(row_ptr, col, x.contiguous(), eps, w.contiguous(), b.contiguous(),
                                              dy.contiguous(), rt=rt)
        return None, None, None, dx, None, dw, db, None


class GCNConv(torch.nn.Module):
    """gcn_layer as a module: y = D^-1/2 (A [+I]) D^-1/2 x W."""

    def __init__(self, gctx: Context, in_dim, out_dim, self_loops=False, dtype=torch.float32, device="cuda"):
        super().__init__()
        self.gctx, self.self_loops = gctx, self_loops
        bound = 1.0 / in_dim ** 0.5
        self.weight = torch.nn.Parameter((torch.rand((in_dim, out_dim), dtype=dtype, device=device) * 2 - 1) * bound)

    def forward(self, row_ptr, col, x, rt=None):
        return GCNConvFn.apply(self.gctx, row_ptr, col, x, self.weight, self.self_loops, rt)


class GINConv(torch.nn.Module):
    """gin_layer as a module: y = relu(((1+eps) x + sum_N x) W + b)."""

    def __init__(self, gctx: Context, in_dim, out_dim, eps=0.0, dtype=torch.float32, device="cuda"):
        super().__init__()
        self.gctx, self.eps = gctx, float(eps)
        bound = 1.0 / in_dim ** 0.5
        self.weight = torch.nn.Parameter((torch.rand((in_dim, out_dim), dtype=dtype, device=device) * 2 - 1) * bound)
        self.bias = torch.nn.Parameter(torch.zeros(out_dim, dtype=dtype, device=device))

    def forward(self, row_ptr, col, x, rt=None):
        return GINConvFn.apply(self.gctx, row_ptr, col, x, self.eps, self.weight, self.bias, rt)
