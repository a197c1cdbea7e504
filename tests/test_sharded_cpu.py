"""Host orchestration of the row-sharded 2-layer GCN step (paper_2006_06608_b200/
sharded.py) with gloo at world size 2 on CPU.

Each rank runs ShardedGCN2 over its nnz-balanced row range with fp64 CPU
primitives (torch CSR products: the test's stand-in for the GPU kernels),
all-gathers the layer outputs, all-reduces the weight gradients, and the
result must equal the UNSHARDED step computed by the oracle (oracle/
gnnsim_oracle.c: gcn_layer twice with a ReLU between, gcn_backward through
both layers) -- output rows, dW1, dW2 -- to 1e-12, on both ranks, for two
consecutive SGD steps.
"""
import os
import socket
import subprocess
import sys

from conftest import ROOT

_WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["GNNA_ROOT"])
sys.path.insert(0, os.path.join(os.environ["GNNA_ROOT"], "tests"))
import numpy as np, torch, torch.distributed as dist
from oracle.cpu import Oracle
from paper_2006_06608_b200.shard import row_ranges
from paper_2006_06608_b200.sharded import ShardedGCN2, TorchComm

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
orc = Oracle("orc")
rng = np.random.default_rng(17)
n, din, hid, dout = 900, 24, 8, 11
w = 1.0 / np.arange(1, n + 1) ** 0.8
src = rng.choice(n, size=5000, p=w / w.sum())
edges = np.stack([src, rng.integers(0, n, 5000)], 1).astype(np.uint32)
rp, col = orc.to_csr(n, edges, True)
x = rng.random((n, din)) - 0.5
dy = rng.random((n, dout)) - 0.5
w1 = (rng.random((din, hid)) * 2 - 1) / np.sqrt(din)
w2 = (rng.random((hid, dout)) * 2 - 1) / np.sqrt(hid)
ranges = row_ranges(rp, world)
r0, r1 = ranges[rank]


class CpuOps:
    """fp64 CPU stand-ins for GpuOps (torch CSR products), same interface."""

    def __init__(self, rp, col, rows):
        n = len(rp) - 1
        self.n, self.rows = n, rows
        deg = np.diff(rp).astype(np.float64)
        norm = 1.0 / np.sqrt(np.maximum(deg, 1.0))
        self.norm = torch.from_numpy(norm)
        self.rs2 = self.norm ** 2
        self.A = torch.sparse_csr_tensor(torch.from_numpy(rp.astype(np.int64)),
                                         torch.from_numpy(col.astype(np.int64)), torch.ones(len(col), dtype=torch.float64),
                                         (n, n))

    def gemm(self, a, w, scale=None):
        y = a @ w
        return y * scale[:, None] if scale is not None else y

    def agg(self, x, out, scale, relu=False, mask=None, peers=None):
        a, b = self.rows
        s = (self.rs2 if scale == "norm2" else self.norm)[a:b, None]
        y = s * (self.A @ x)[a:b]
        if relu:
            y = y.clamp_min(0)
        if mask is not None:
            y = torch.where(mask[a:b] > 0, y, torch.zeros_like(y))
        out[a:b] = y
        return out

    def dense_backward(self, dy, w, z):
        a, b = self.rows
        return self.norm[a:b, None] * (dy @ w.t()), z.t() @ dy

    def gemm_tn(self, a, b):
        return a.t() @ b

    def empty(self, shape, like):
        return torch.zeros(shape, dtype=like.dtype)


ops = CpuOps(rp, col, (r0, r1))
model = ShardedGCN2(ops, TorchComm(ranges, rank, fused=False), torch.from_numpy(w1.copy()),
                    torch.from_numpy(w2.copy()), lr=0.05)
W1, W2 = w1.copy(), w2.copy()
for step in range(2):
    y_own, dw1, dw2 = model.step(torch.from_numpy(x), torch.from_numpy(dy[r0:r1]).contiguous())
    # the unsharded step (oracle, fp64)
    h1 = np.maximum(orc.gcn_layer(rp, col, x, W1, False), 0.0)
    want_y = orc.gcn_layer(rp, col, h1, W2, False)
    dh1, want_dw2 = orc.gcn_backward(rp, col, h1, W2, dy, False)
    _, want_dw1 = orc.gcn_backward(rp, col, x, W1, dh1 * (h1 > 0), False)
    for got, want, name in ((y_own.numpy(), want_y[r0:r1], "y"), (dw1.numpy(), want_dw1, "dW1"),
                            (dw2.numpy(), want_dw2, "dW2")):
        err = np.abs(got - want).max() / max(np.abs(want).max(), 1e-300)
        assert err <= 1e-12, (rank, step, name, err)
    W1 -= 0.05 * want_dw1
    W2 -= 0.05 * want_dw2
    assert np.allclose(model.w1.numpy(), W1, rtol=1e-12, atol=1e-14)
dist.barrier()
print("rank", rank, "ok", ranges[rank])
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_gcn2_step_gloo_world2(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(_WORKER)
    env = dict(os.environ, GNNA_ROOT=ROOT, OMP_NUM_THREADS="1")
    for attempt in range(3):  # a fresh port per attempt
        r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2", "--master-addr",
                            "127.0.0.1", "--master-port", str(_free_port()), str(script)], capture_output=True,
                           text=True, env=env, timeout=300)
        if r.returncode == 0 or "AssertionError" in r.stderr:
            break
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.count("ok") == 2  # one per rank (the two lines may interleave)
