"""GNN models on the B200 path: the BASELINE C3 configuration (2-layer GCN,
forward + backward + SGD step) and a GIN layer, composed from the C-ABI's
plan-based kernels (fp32 perf path):

  aggregation  gnna_aggregate_ex on one gnna_plan (K1/K2 built once), with the
               normalisation fused in: per-edge weights norm[col[e]], self
               weight, row scale norm[v], and the ReLU / ReLU-backward mask in
               the flush epilogue
  update       gnna_gemm (K6) and its transposed forms for the gradients

Layer math follows gcn_layer (engine.cpp:373-382): update first iff the layer
shrinks the width, z = D^-1/2 (A [+I]) D^-1/2 x.  The reference has no model
or backward; a ReLU between the two layers makes it the standard
2-layer GCN.  torch supplies device memory and the tiny SGD update (plumbing).
"""
from __future__ import annotations

import math

import torch

from .capi import WARP_SHARED, Context, Params


class GCN2:
    """2-layer GCN: y = Â relu(Â x W1) W2 (each layer ordered as gcn_layer)."""

    def __init__(self, ctx: Context, row_ptr, col, in_dim, hidden, out_dim, self_loops=False, params: Params = None,
                 seed=4, lr=0.01):
        self.ctx, self.torch = ctx, torch
        self.row_ptr, self.col = row_ptr, col
        self.n = row_ptr.numel() - 1
        self.dims = (in_dim, hidden, out_dim)
        dev = row_ptr.device
        if params is None:
            params, _ = ctx.b200_params(row_ptr, min(hidden, in_dim))
        self.params = params
        # one schedule (K1 units + K2 Algorithm-1 plan) for every aggregation of the step
        self.plan = ctx.plan(row_ptr, col, params, WARP_SHARED)
        self.rs, self.sw, _ = ctx.gcn_weights(row_ptr, col, self_loops, edge_weights=False)
        # folded form: the source-side D^-1/2 rides in the producing GEMM's
        # row-scale epilogue (norm), or in the previous aggregation's epilogue
        # (norm^2), so those aggregations are plain sums (no per-edge gather)
        self.norm, _, self.rs2, self.ind = ctx.gcn_fold_weights(row_ptr, col, self_loops)
        if not self_loops:  # no implicit self loops: the self term is identically zero
            self.sw = self.ind = None
        # W ~ U[-1, 1) / sqrt(fan_in) from the reference's random_features stream (seeds 4, 5)
        self.w1 = self._uniform(in_dim, hidden, seed, dev) / math.sqrt(in_dim)
        self.w2 = self._uniform(hidden, out_dim, seed + 1, dev) / math.sqrt(hidden)
        self.zero_b1 = torch.zeros(hidden, device=dev)
        self.lr = lr
        self.side = None

    @staticmethod
    def _uniform(rows, cols, seed, dev):
        from .capi import random_features
        return (torch.from_numpy(random_features(rows, cols, seed)) * 2 - 1).to(dev).contiguous()

    def use_side_stream(self, enable=True):
        """Run the independent dW2 product on a second stream (its own
        gnna context) so it overlaps the dP1 chain; capturable in a CUDA
        graph (fork/join through stream waits)."""
        if not enable:
            self.side = None
            return self

        class _Side:
            pass
        side = _Side()
        side.stream = torch.cuda.Stream(device=self.row_ptr.device)
        side.ctx = Context(self.row_ptr.device.index or 0, side.stream)
        self.side = side
        return self

    def _agg(self, x, relu=False, mask=None, out=None):
        """Â x for an x nobody pre-scaled: K3 gathers norm[u] per edge."""
        return self.plan.aggregate_ex(x, out=out, node_weight=self.rs, self_weight=self.sw, row_scale=self.rs,
                                      relu=relu, mask=mask)

    def _aggf(self, xs, scale, relu=False, mask=None, out=None):
        """Â x given xs = norm * x (pre-scaled by its producer): a plain-sum K3
        with the destination scale (norm, or norm^2 when the result feeds
        another aggregation) and the self term in the epilogue."""
        return self.plan.aggregate_ex(xs, out=out, self_weight=self.ind, row_scale=scale, relu=relu, mask=mask)

    def forward(self, x):
        ctx = self.ctx
        in_dim, hid, out_dim = self.dims
        s = {}
        agg2_first = out_dim >= hid  # layer 2 aggregates first (then h1 feeds an aggregation)
        if hid < in_dim:  # layer 1 update first: h1 = relu(Â (x W1))
            s["t1"] = ctx.gemm(x, self.w1, None, 2, self.norm)  # norm * (x W1)
            # relu(norm^2 * S) = norm * relu(norm * S): h1 comes out pre-scaled for layer 2
            s["h1"] = self._aggf(s["t1"], self.rs2 if agg2_first else self.rs, relu=True)
            s["h1_scaled"] = agg2_first
        else:  # aggregate first: h1 = relu((Â x) W1)
            s["z1"] = self._agg(x)
            s["h1"] = ctx.gemm(s["z1"], self.w1, self.zero_b1, 1)
            s["h1_scaled"] = False
        if not agg2_first:  # layer 2 update first
            s["t2"] = ctx.gemm(s["h1"], self.w2, None, 2, self.norm)
            y = self._aggf(s["t2"], self.rs)
        else:
            s["z2"] = self._aggf(s["h1"], self.rs) if s["h1_scaled"] else self._agg(s["h1"])
            y = ctx.gemm(s["z2"], self.w2)
        self.saved = s
        return y

    def backward(self, x, dy):
        """Gradients of <dy, forward(x)> w.r.t. W1, W2 (Â is symmetric for the
        symmetrised CSR to_csr(.., true) builds, so Â^T = Â)."""
        ctx, s = self.ctx, self.saved
        in_dim, hid, out_dim = self.dims
        if out_dim < hid:
            dt2 = self._agg(dy)                                    # Â^T dY
            dw2 = ctx_gemm_tn(ctx, s["h1"], dt2)                   # h1^T dT2
            dh1 = ctx.gemm(dt2, self.w2.t().contiguous())
            dp1 = dh1 * (s["h1"] > 0)
            dp1_scaled = False
        else:
            # (Â h1)^T dY does not feed the rest of the backward: with a side
            # context it runs on a second stream, overlapped with the dP1 chain
            side = self.side
            if side is not None:
                main = torch.cuda.current_stream()
                side.stream.wait_stream(main)
                with torch.cuda.stream(side.stream):
                    dw2 = ctx_gemm_tn(side.ctx, s["z2"], dy)
                dz2 = ctx.gemm(dy, self.w2.t().contiguous(), None, 2, self.norm)  # norm * (dY W2^T)
            else:
                # one pass over dY and Â h1: dZ2 = norm * (dY W2^T), dW2 = (Â h1)^T dY
                dz2, dw2 = ctx.dense_backward(dy, self.w2, s["z2"], self.norm)
            # Â^T dZ2 masked by relu'(h1) (the sign of a pre-scaled h1 is the same);
            # pre-scaled by norm again when the next aggregation consumes it
            dp1_scaled = hid < in_dim
            dp1 = self._aggf(dz2, self.rs2 if dp1_scaled else self.rs, mask=s["h1"])
        if hid < in_dim:
            dt1 = self._aggf(dp1, self.rs) if dp1_scaled else self._agg(dp1)  # Â^T dP1
            dw1 = ctx_gemm_tn(ctx, x, dt1)                         # x^T dT1
        else:
            dw1 = ctx_gemm_tn(ctx, s["z1"], dp1)
        if out_dim >= hid and self.side is not None:
            torch.cuda.current_stream().wait_stream(self.side.stream)  # join before dW2 is read
        return dw1, dw2

    def sgd(self, dw1, dw2):
        # both weights in one multi-tensor kernel (w += (-lr) * dw, as add_ per weight)
        torch._foreach_add_([self.w1, self.w2], [dw1, dw2], alpha=-self.lr)

    def step(self, x, dy):
        y = self.forward(x)
        dw1, dw2 = self.backward(x, dy)
        self.sgd(dw1, dw2)
        return y, dw1, dw2

    def aggregations_per_step(self):
        """(count, width) of the aggregations one step runs."""
        in_dim, hid, out_dim = self.dims
        widths = [min(hid, in_dim), min(out_dim, hid), min(out_dim, hid)]
        if hid < in_dim:
            widths.append(hid)
        return widths


def ctx_gemm_tn(ctx: Context, a, b):
    """a^T b through the C-ABI (deterministic chunked reduction)."""
    import ctypes as C
    from .capi import _dtype_code, _ptr
    m, p = a.shape
    q = b.shape[1]
    out = torch.empty((p, q), dtype=a.dtype, device=a.device)
    ctx._check(ctx.L.gnna_gemm_tn(ctx.h, C.c_int(_dtype_code(a)), _ptr(a), _ptr(b), C.c_uint32(m), C.c_uint32(p),
                                  C.c_uint32(q), _ptr(out)))
    return out
