"""ctypes binding of libgnna.so (include/gnna.h) for Python callers.

Device memory, streams and collectives come from PyTorch (plumbing only); all
compute happens in libgnna.so's sm_100a kernels.  There is no fallback: if the
library is missing or the device is not a B200 the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GNNA_LIB") or os.path.join(HERE, "libgnna.so")  # GNNA_LIB: experiment builds

OK, ERR_DOMAIN, ERR_INTERNAL, ERR_CUDA, ERR_OOM = 0, 1, 2, 3, 4
NAIVE_ATOMIC, UNIT_SYNC, WARP_SHARED = 0, 1, 2
DIM_SEQUENTIAL, DIM_CYCLIC = 0, 1
F32, F64 = 0, 1


class GnnaError(RuntimeError):
    KIND = {ERR_DOMAIN: "DomainError", ERR_INTERNAL: "InternalError", ERR_CUDA: "CudaError",
            ERR_OOM: "OutOfMemory"}

    def __init__(self, code, msg):
        super().__init__(f"{self.KIND.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg


class DomainError(GnnaError):
    pass


class Params(C.Structure):
    """schedule.hpp:14-27 KernelParams."""
    _fields_ = [("ngs", C.c_uint32), ("dw", C.c_uint32), ("tpb", C.c_uint32), ("tpw", C.c_uint32),
                ("dim", C.c_uint32)]

    @classmethod
    def make(cls, ngs=16, dw=32, tpb=128, dim=16, tpw=32):
        return cls(ngs, dw, tpb, tpw, dim)

    def tolist(self):
        return [self.ngs, self.dw, self.tpb, self.tpw, self.dim]


class Cost(C.Structure):
    """engine.hpp:30-53 CostReport."""
    _fields_ = [(k, C.c_uint64) for k in ("atomic_ops", "global_reads", "global_writes",
                                          "global_transactions", "shared_bytes_per_block",
                                          "cache_hits", "cache_accesses")]

    def tolist(self):
        return [getattr(self, k) for k, _ in self._fields_]


class ModelInputs(C.Structure):
    """decider.hpp:12-26 ModelInputs."""
    _fields_ = [("num_nodes", C.c_uint64), ("num_edges", C.c_uint64), ("dim", C.c_uint32),
                ("max_tpb", C.c_uint32), ("avg_degree", C.c_double),
                ("stddev_degree", C.c_double), ("smem_per_block", C.c_uint64),
                ("capability", C.c_uint64), ("alpha", C.c_double)]

    @classmethod
    def make(cls, num_nodes=0, num_edges=0, dim=16, avg_degree=0.0, stddev_degree=0.0,
             max_tpb=1024, smem_per_block=96 * 1024, capability=4096, alpha=0.15):
        return cls(num_nodes, num_edges, dim, max_tpb, avg_degree, stddev_degree, smem_per_block,
                   capability, alpha)


class AggOpts(C.Structure):
    """gnna_agg_opts (include/gnna.h)."""
    _fields_ = [("dim", C.c_uint32), ("node_weight", C.c_void_p), ("self_weight", C.c_void_p), ("alpha", C.c_double),
                ("row_scale", C.c_void_p), ("relu", C.c_int), ("mask", C.c_void_p)]


class HostBatch(C.Structure):
    """gnna_host_batch (include/gnna.h)."""
    _fields_ = [("h_row_ptr", C.c_void_p), ("h_col", C.c_void_p), ("n", C.c_uint32), ("row_begin", C.c_uint32),
                ("row_end", C.c_uint32), ("h_x", C.c_void_p), ("h_y", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build()")
        _lib = C.CDLL(LIB_PATH)
        _lib.gnna_last_error.restype = C.c_char_p
        _lib.gnna_version.restype = C.c_char_p
        _lib.gnna_launch_count.restype = C.c_uint64
        _lib.gnna_get_stream.restype = C.c_void_p
        _lib.gnna_alpha_from_degrees.restype = C.c_double
        _lib.gnna_alpha_from_degrees.argtypes = [C.c_double, C.c_double]
        _lib.gnna_decider_last_error.restype = C.c_char_p
    return _lib


def _ptr(t):
    if t is None:
        return C.c_void_p(0)
    if isinstance(t, np.ndarray):
        return C.c_void_p(t.ctypes.data)
    return C.c_void_p(t.data_ptr())


def _dev(t, what, dtype=None, shape=None):
    """Argument check before a device pointer crosses the C-ABI: a contiguous
    CUDA tensor of the expected dtype / shape (the kernels take raw row-major
    pointers and sizes, so a view or a width mismatch would read or write out
    of bounds instead of failing)."""
    if t is None:
        return t
    if not getattr(t, "is_cuda", False):
        raise ValueError(f"{what}: expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{what}: expected a contiguous tensor (got strides {tuple(t.stride())})")
    if dtype is not None and t.dtype not in (dtype if isinstance(dtype, tuple) else (dtype,)):
        raise TypeError(f"{what}: expected dtype {dtype}, got {t.dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{what}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    return t


def _dtype_code(t):
    import torch
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.float64:
        return F64
    raise TypeError(f"unsupported feature dtype {t.dtype}")


class Context:
    """One gnna_ctx bound to a CUDA device; kernels run on torch's current
    stream (captured at construction, or call set_stream)."""

    def __init__(self, device: int = 0, stream=None):
        import torch
        self.torch = torch
        self.L = lib()
        self.device = device
        h = C.c_void_p()
        rc = self.L.gnna_create(C.c_int(device), C.byref(h))
        if rc:
            raise GnnaError(rc, "gnna_create failed (needs a B200 / sm_100 device)")
        self.h = h
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.set_stream(stream)

    def set_stream(self, stream):
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self._check(self.L.gnna_set_stream(self.h, C.c_void_p(handle)))

    def close(self):
        if getattr(self, "h", None):
            self.L.gnna_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != OK:
            msg = self.L.gnna_last_error(self.h).decode()
            if rc == ERR_DOMAIN:
                raise DomainError(rc, msg)
            raise GnnaError(rc, msg)

    @property
    def launches(self):
        return int(self.L.gnna_launch_count(self.h))

    def synchronize(self):
        self._check(self.L.gnna_synchronize(self.h))

    def pin_hot_rows(self, row_ptr_host, x, cap_bytes=48 << 20, min_gain=4.0):
        """Data-driven L2 residency for the gather (gnna_set_l2_window): when
        the front rows of x (what fits in cap_bytes) receive at least
        min_gain times their uniform share of the gathers -- power-law hubs
        numbered first -- pin them; otherwise leave L2 alone.  The gather
        share of rows [0, k) is row_ptr[k] / nnz (symmetric CSR: in-degree =
        degree).  Inputs smaller than L2 are never pinned.  Returns a dict for
        the bench's config."""
        rp = np.asarray(row_ptr_host).view(np.uint64) if np.asarray(row_ptr_host).dtype != np.uint64 else \
            np.asarray(row_ptr_host)
        n, nnz = len(rp) - 1, int(rp[-1])
        row_bytes = x.shape[1] * x.element_size()
        l2 = self.torch.cuda.get_device_properties(x.device).L2_cache_size
        info = {"pinned": False, "cap_MB": cap_bytes >> 20}
        if n == 0 or nnz == 0 or x.numel() * x.element_size() <= l2:
            return info
        k = min(n, cap_bytes // row_bytes)
        share = float(rp[k]) / nnz
        uniform = k / n
        info.update({"rows": int(k), "gather_share": round(share, 4), "uniform_share": round(uniform, 6)})
        if share >= min_gain * uniform:
            info["applied_bytes"] = self.set_l2_window(x, k * row_bytes, 1.0)
            info["pinned"] = True
        return info

    def set_l2_window(self, base=None, nbytes=0, hit_ratio=1.0):
        """gnna_set_l2_window: persist [base, base+nbytes) in L2 on this
        context's stream (base: tensor or pointer); nbytes 0 clears it."""
        ptr = 0 if base is None else (base if isinstance(base, int) else base.data_ptr())
        applied = C.c_uint64()
        self._check(self.L.gnna_set_l2_window(self.h, C.c_void_p(ptr), C.c_uint64(int(nbytes)),
                                              C.c_double(hit_ratio), C.byref(applied)))
        return applied.value

    def _empty(self, n, dtype):
        return self.torch.empty(n, dtype=dtype, device=f"cuda:{self.device}")

    # ------------------------------------------------------- preprocessing
    def validate_params(self, p: Params):
        self._check(self.L.gnna_validate_params(self.h, C.byref(p)))

    def count_groups(self, row_ptr, ngs):
        g = C.c_uint64()
        self._check(self.L.gnna_count_groups(self.h, _ptr(row_ptr), C.c_uint32(row_ptr.numel() - 1),
                                             C.c_uint32(ngs), C.byref(g)))
        return g.value

    def partition_neighbors(self, row_ptr, ngs):
        """schedule.cpp:16 -> (part_ptr[G+1] int64, part2node[G] int32) device tensors."""
        torch = self.torch
        G = self.count_groups(row_ptr, ngs)
        pp = self._empty(G + 1, torch.int64)
        p2n = self._empty(max(G, 1), torch.int32)
        self._check(self.L.gnna_partition_neighbors(self.h, _ptr(row_ptr), C.c_uint32(row_ptr.numel() - 1),
                                                    C.c_uint32(ngs), _ptr(pp), _ptr(p2n)))
        return pp, p2n[:G]

    def build_mem_plan(self, part2node, p: Params):
        """memplan.cpp:9 -> (slot u8[G], leader u8[G], shared_bytes)."""
        torch = self.torch
        G = part2node.numel()
        slot = self._empty(max(G, 1), torch.uint8)
        lead = self._empty(max(G, 1), torch.uint8)
        sb = C.c_uint64()
        self._check(self.L.gnna_build_mem_plan(self.h, _ptr(part2node), C.c_uint64(G), C.byref(p),
                                               _ptr(slot), _ptr(lead), C.byref(sb)))
        return slot[:G], lead[:G], sb.value

    def plan(self, row_ptr, col, p: Params, strategy=WARP_SHARED, rows=None):
        return Plan(self, row_ptr, col, p, strategy, rows)

    # --------------------------------------------------------- aggregation
    def aggregate_rows(self, row_ptr, col, x, out=None):
        n = row_ptr.numel() - 1
        if out is None:
            out = self.torch.empty_like(x)
        self._check(self.L.gnna_aggregate_rows(self.h, C.c_int(_dtype_code(x)), _ptr(row_ptr), _ptr(col),
                                               C.c_uint32(n), C.c_uint32(x.shape[1]), _ptr(x), _ptr(out)))
        return out

    def features_close(self, a, b, rel_tol):
        """engine.cpp:162 features_close on device tensors (shape check here, elements on the GPU)."""
        if tuple(a.shape) != tuple(b.shape) or a.dtype != b.dtype:
            return False
        out = C.c_int()
        self._check(self.L.gnna_features_close(self.h, C.c_int(_dtype_code(a)), _ptr(a), _ptr(b),
                                               C.c_uint64(a.numel()), C.c_double(rel_tol), C.byref(out)))
        return bool(out.value)

    def aggregate_host(self, row_ptr, col, x, p: Params, strategy=WARP_SHARED, dim_mode=DIM_CYCLIC,
                       out=None, line=128, cache=None, want_cost=True):
        """gnna_aggregate_host: host (numpy / pinned torch CPU) buffers in and out."""
        n = len(row_ptr) - 1
        if out is None:
            out = np.empty_like(x)
        if isinstance(x, np.ndarray):
            if x.dtype not in (np.float32, np.float64):
                raise TypeError(f"unsupported feature dtype {x.dtype}")
            dt = F32 if x.dtype == np.float32 else F64
        else:
            dt = _dtype_code(x)
        cost = Cost()
        cap, cl = cache if cache else (0, 0)
        self._check(self.L.gnna_aggregate_host(self.h, C.c_int(dt), _ptr(row_ptr), _ptr(col), C.c_uint32(n),
                                               C.byref(p), C.c_int(strategy), C.c_int(dim_mode), _ptr(x),
                                               _ptr(out), C.c_uint64(line), C.c_uint64(cap), C.c_uint64(cl),
                                               C.byref(cost) if want_cost else None))
        return out, cost

    # --------------------------------------------------------------- graph
    def to_csr(self, n, edges, symmetrize=True):
        """graph.cpp:76 to_csr on the GPU: edges (E,2) int32 device tensor ->
        (row_ptr int64[n+1], col int32[nnz]) canonical CSR."""
        torch = self.torch
        e = edges.numel() // 2
        nnz = C.c_uint64()
        rp = self._empty(n + 1, torch.int64)
        self._check(self.L.gnna_to_csr(self.h, C.c_uint32(n), _ptr(edges), C.c_uint64(e), C.c_int(int(symmetrize)),
                                       _ptr(rp), C.c_void_p(0), C.byref(nnz)))
        col = self._empty(max(nnz.value, 1), torch.int32)
        self._check(self.L.gnna_to_csr(self.h, C.c_uint32(n), _ptr(edges), C.c_uint64(e), C.c_int(int(symmetrize)),
                                       _ptr(rp), _ptr(col), C.byref(nnz)))
        return rp, col[: nnz.value]

    def csr_transpose(self, row_ptr, col):
        n = row_ptr.numel() - 1
        tp = self._empty(n + 1, self.torch.int64)
        tc = self._empty(max(col.numel(), 1), self.torch.int32)
        self._check(self.L.gnna_csr_transpose(self.h, _ptr(row_ptr), _ptr(col), C.c_uint32(n), _ptr(tp), _ptr(tc)))
        return tp, tc[: col.numel()]

    def aes(self, edges):
        out = C.c_double()
        self._check(self.L.gnna_aes(self.h, _ptr(edges), C.c_uint64(edges.numel() // 2), C.byref(out)))
        return out.value

    def degree_stats(self, row_ptr):
        a, m, s = C.c_double(), C.c_uint64(), C.c_double()
        self._check(self.L.gnna_degree_stats(self.h, _ptr(row_ptr), C.c_uint32(row_ptr.numel() - 1), C.byref(a),
                                             C.byref(m), C.byref(s)))
        return a.value, m.value, s.value

    def model_inputs(self, row_ptr, dim, b200=False):
        mi = ModelInputs()
        self._check(self.L.gnna_model_inputs_from_graph(self.h, _ptr(row_ptr), C.c_uint32(row_ptr.numel() - 1),
                                                        C.c_uint32(dim), C.byref(mi)))
        if b200:
            self._check(self.L.gnna_b200_profile(self.h, C.byref(mi)))
        return mi

    def aggregate_host_rows(self, row_ptr, col, x, p: Params, r0, r1, out, strategy=WARP_SHARED,
                            dim_mode=DIM_CYCLIC):
        """gnna_aggregate_host_rows over host (pinned) torch tensors; out: (r1-r0) x dim."""
        n = row_ptr.numel() - 1
        self._check(self.L.gnna_aggregate_host_rows(self.h, C.c_int(_dtype_code(x)), _ptr(row_ptr), _ptr(col),
                                                    C.c_uint32(n), C.c_uint32(r0), C.c_uint32(r1), C.byref(p),
                                                    C.c_int(strategy), C.c_int(dim_mode), _ptr(x), _ptr(out),
                                                    C.c_uint64(128), C.c_uint64(0), C.c_uint64(0), None))
        return out

    def aggregate_host_stream(self, p: Params, batches, strategy=WARP_SHARED, dim_mode=DIM_CYCLIC):
        """gnna_aggregate_host_stream: batches = [(row_ptr, col, x, r0, r1, out)] of host (pinned) tensors,
        processed with uploads/compute/downloads of consecutive batches overlapped."""
        arr = (HostBatch * len(batches))()
        dt = None
        for i, (rp, col, x, r0, r1, out) in enumerate(batches):
            arr[i] = HostBatch(_ptr(rp).value, _ptr(col).value, rp.numel() - 1, r0, r1, _ptr(x).value, _ptr(out).value)
            dt = _dtype_code(x)
        self._check(self.L.gnna_aggregate_host_stream(self.h, C.c_int(dt), C.byref(p), C.c_int(strategy),
                                                      C.c_int(dim_mode), arr, C.c_uint32(len(batches))))

    # ------------------------------------------------------- layers (K5/K6)
    def gemm(self, a, w, bias=None, epilogue=0, row_scale=None, out=None):
        m, k = a.shape
        n_out = w.shape[1]
        if out is None:
            out = self.torch.empty((m, n_out), dtype=a.dtype, device=a.device)
        _dev(a, "a", (self.torch.float32, self.torch.float64))
        _dev(w, "w", a.dtype, (k, n_out))
        _dev(out, "out", a.dtype, (m, n_out))
        _dev(bias, "bias", a.dtype, (n_out,))
        _dev(row_scale, "row_scale", self.torch.float64, (m,))  # gnna_gemm takes a double row scale
        self._check(self.L.gnna_gemm(self.h, C.c_int(_dtype_code(a)), _ptr(a), C.c_uint32(m), C.c_uint32(k), _ptr(w),
                                     C.c_uint32(n_out), _ptr(bias), C.c_int(epilogue), _ptr(row_scale), _ptr(out)))
        return out

    def dense_backward(self, dy, w, z, row_scale=None):
        """gnna_dense_backward: (dz = row_scale * (dy W^T), dW = z^T dy) for
        y = z W; one fused pass for narrow fp32 layers."""
        torch = self.torch
        m, q = dy.shape
        p = w.shape[0]
        _dev(dy, "dy", (torch.float32, torch.float64))
        _dev(w, "w", dy.dtype, (p, q))
        _dev(z, "z", dy.dtype, (m, p))
        _dev(row_scale, "row_scale", torch.float64, (m,))
        dz = torch.empty((m, p), dtype=dy.dtype, device=dy.device)
        dw = torch.empty((p, q), dtype=dy.dtype, device=dy.device)
        self._check(self.L.gnna_dense_backward(self.h, C.c_int(_dtype_code(dy)), _ptr(dy), C.c_uint32(m),
                                               C.c_uint32(q), _ptr(w), _ptr(z), C.c_uint32(p), _ptr(row_scale),
                                               _ptr(dz), _ptr(dw)))
        return dz, dw

    def gcn_norm(self, row_ptr, col, self_loops=False):
        n = row_ptr.numel() - 1
        norm = self._empty(max(n, 1), self.torch.float64)
        sl = self._empty(max(n, 1), self.torch.uint8)
        self._check(self.L.gnna_gcn_norm(self.h, _ptr(row_ptr), _ptr(col), C.c_uint32(n), C.c_int(int(self_loops)),
                                         _ptr(norm), _ptr(sl)))
        return norm[:n], sl[:n]

    def gcn_weights(self, row_ptr, col, self_loops=False, edge_weights=True):
        """fp32 (row_scale[n], self_weight[n], edge_weight[nnz] or None) of
        D^-1/2 (A [+I]) D^-1/2.  The fused K3 only needs the node arrays
        (edge_weights=False skips the per-edge array)."""
        n = row_ptr.numel() - 1
        torch = self.torch
        rs, sw = self._empty(max(n, 1), torch.float32), self._empty(max(n, 1), torch.float32)
        ew = self._empty(max(col.numel(), 1), torch.float32) if edge_weights else None
        self._check(self.L.gnna_gcn_weights(self.h, _ptr(row_ptr), _ptr(col), C.c_uint32(n), C.c_int(int(self_loops)),
                                            _ptr(rs), _ptr(sw), _ptr(ew)))
        return rs[:n], sw[:n], (ew[: col.numel()] if edge_weights else None)

    def gcn_fold_weights(self, row_ptr, col, self_loops=False):
        """gnna_gcn_fold_weights: (norm f64, row_scale = norm, row_scale2 =
        norm^2, self indicator) for the folded normalisation, whose source-side
        D^-1/2 rides in the producing GEMM's row-scale epilogue."""
        n = row_ptr.numel() - 1
        torch = self.torch
        norm = self._empty(max(n, 1), torch.float64)
        rs, rs2, ind = (self._empty(max(n, 1), torch.float32) for _ in range(3))
        self._check(self.L.gnna_gcn_fold_weights(self.h, _ptr(row_ptr), _ptr(col), C.c_uint32(n),
                                                 C.c_int(int(self_loops)), _ptr(norm), _ptr(rs), _ptr(rs2),
                                                 _ptr(ind)))
        return norm[:n], rs[:n], rs2[:n], ind[:n]

    def normalized_aggregate(self, row_ptr, col, x, norm, selfl, out=None):
        n = row_ptr.numel() - 1
        if out is None:
            out = self.torch.empty_like(x)
        self._check(self.L.gnna_normalized_aggregate(self.h, C.c_int(_dtype_code(x)), _ptr(row_ptr), _ptr(col),
                                                     C.c_uint32(n), C.c_uint32(x.shape[1]), _ptr(norm), _ptr(selfl),
                                                     _ptr(x), _ptr(out)))
        return out

    def gcn_forward(self, row_ptr, col, x, w, self_loops=False):
        n = row_ptr.numel() - 1
        y = self.torch.empty((n, w.shape[1]), dtype=x.dtype, device=x.device)
        self._check(self.L.gnna_gcn_forward(self.h, C.c_int(_dtype_code(x)), _ptr(row_ptr), _ptr(col), C.c_uint32(n),
                                            _ptr(x), C.c_uint32(x.shape[1]), _ptr(w), C.c_uint32(w.shape[1]),
                                            C.c_int(int(self_loops)), _ptr(y)))
        return y

    def gin_forward(self, row_ptr, col, x, eps, w, b):
        n = row_ptr.numel() - 1
        y = self.torch.empty((n, w.shape[1]), dtype=x.dtype, device=x.device)
        self._check(self.L.gnna_gin_forward(self.h, C.c_int(_dtype_code(x)), _ptr(row_ptr), _ptr(col), C.c_uint32(n),
                                            _ptr(x), C.c_uint32(x.shape[1]), C.c_double(eps), _ptr(w),
                                            C.c_uint32(w.shape[1]), _ptr(b), _ptr(y)))
        return y

    def gcn_backward(self, row_ptr, col, x, w, dy, self_loops=False, rt=None):
        n = row_ptr.numel() - 1
        rtp, rtc = rt if rt is not None else (row_ptr, col)
        dx = self.torch.empty_like(x)
        dw = self.torch.empty_like(w)
        self._check(self.L.gnna_gcn_backward(self.h, C.c_int(_dtype_code(x)), _ptr(row_ptr), _ptr(col), _ptr(rtp),
                                             _ptr(rtc), C.c_uint32(n), _ptr(x), C.c_uint32(x.shape[1]), _ptr(w),
                                             C.c_uint32(w.shape[1]), C.c_int(int(self_loops)), _ptr(dy), _ptr(dx),
                                             _ptr(dw)))
        return dx, dw

    def gin_backward(self, row_ptr, col, x, eps, w, b, dy, rt=None):
        n = row_ptr.numel() - 1
        rtp, rtc = rt if rt is not None else (row_ptr, col)
        dx, dw, db = self.torch.empty_like(x), self.torch.empty_like(w), self.torch.empty_like(b)
        de = C.c_double()
        self._check(self.L.gnna_gin_backward(self.h, C.c_int(_dtype_code(x)), _ptr(row_ptr), _ptr(col), _ptr(rtp),
                                             _ptr(rtc), C.c_uint32(n), _ptr(x), C.c_uint32(x.shape[1]),
                                             C.c_double(eps), _ptr(w), C.c_uint32(w.shape[1]), _ptr(b), _ptr(dy),
                                             _ptr(dx), _ptr(dw), _ptr(db), C.byref(de)))
        return dx, dw, db, de.value

    # ----------------------------------------------------------- renumber
    def detect_communities(self, row_ptr, col):
        n = row_ptr.numel() - 1
        com = self._empty(max(n, 1), self.torch.int32)
        k = C.c_uint32()
        self._check(self.L.gnna_detect_communities(self.h, _ptr(row_ptr), _ptr(col), C.c_uint32(n), _ptr(com),
                                                   C.byref(k)))
        return com[:n], k.value

    def modularity(self, row_ptr, col, com, ncom):
        q = C.c_double()
        self._check(self.L.gnna_modularity(self.h, _ptr(row_ptr), _ptr(col), C.c_uint32(row_ptr.numel() - 1),
                                           _ptr(com), C.c_uint32(ncom), C.byref(q)))
        return q.value

    def degree_order(self, row_ptr):
        """gnna_degree_order: (old_to_new, new_to_old) by descending degree, ties by id."""
        n = row_ptr.numel() - 1
        o2n, n2o = self._empty(max(n, 1), self.torch.int32), self._empty(max(n, 1), self.torch.int32)
        self._check(self.L.gnna_degree_order(self.h, _ptr(row_ptr), C.c_uint32(n), _ptr(o2n), _ptr(n2o)))
        return o2n[:n], n2o[:n]

    def build_mapping(self, com, ncom):
        n = com.numel()
        o2n, n2o = self._empty(max(n, 1), self.torch.int32), self._empty(max(n, 1), self.torch.int32)
        self._check(self.L.gnna_build_mapping(self.h, _ptr(com), C.c_uint32(n), C.c_uint32(ncom), _ptr(o2n),
                                              _ptr(n2o)))
        return o2n[:n], n2o[:n]

    def mapping_from_vector(self, vec):
        n = vec.numel()
        o2n, n2o = self._empty(max(n, 1), self.torch.int32), self._empty(max(n, 1), self.torch.int32)
        self._check(self.L.gnna_mapping_from_vector(self.h, _ptr(vec), C.c_uint32(n), _ptr(o2n), _ptr(n2o)))
        return o2n[:n], n2o[:n]

    def apply_mapping_csr(self, row_ptr, col, o2n, n2o):
        n = row_ptr.numel() - 1
        orp = self._empty(n + 1, self.torch.int64)
        oc = self._empty(max(col.numel(), 1), self.torch.int32)
        self._check(self.L.gnna_apply_mapping_csr(self.h, _ptr(row_ptr), _ptr(col), C.c_uint32(n), _ptr(o2n),
                                                  _ptr(n2o), _ptr(orp), _ptr(oc)))
        return orp, oc[: col.numel()]

    def apply_mapping_edges(self, edges, n, o2n):
        out = self.torch.empty_like(edges)
        self._check(self.L.gnna_apply_mapping_edges(self.h, _ptr(edges), C.c_uint64(edges.numel() // 2),
                                                    C.c_uint32(n), _ptr(o2n), _ptr(out)))
        return out

    def tune_params(self, row_ptr, col, dim, gs=(1, 2, 4, 8, 16, 32, 64, 128, 256), dw=(4, 8, 16, 32),
                    tpb=(32, 64, 128, 256)):
        g, d, t = (np.asarray(v, np.uint32) for v in (gs, dw, tpb))
        best = Params()
        ms = C.c_float()
        self._check(self.L.gnna_tune_params(self.h, _ptr(row_ptr), _ptr(col), C.c_uint32(row_ptr.numel() - 1),
                                            C.c_uint32(dim), _ptr(g), C.c_uint32(len(g)), _ptr(d), C.c_uint32(len(d)),
                                            _ptr(t), C.c_uint32(len(t)), C.byref(best), C.byref(ms)))
        return best, ms.value

    # ------------------------------------------------------------- decider
    def b200_params(self, row_ptr, dim, hbm_gbs=0.0, dtype=None, window=False):
        """The B200 evaluator (gnna_b200_plan_params) on this device graph:
        (Params, model K3 microseconds), plus the recommended L2 window bytes
        for the hub rows when window=True.  dtype: torch.float32 (default) or
        torch.float64 (element size of the features)."""
        if not hbm_gbs:
            try:
                import json
                hbm_gbs = float(json.load(open(os.path.join(os.path.dirname(HERE), "MEASURED_PEAKS.json")))["hbm_gbs"])
            except Exception:
                hbm_gbs = 0.0
        dt = F64 if dtype is not None and dtype == self.torch.float64 else F32
        p = Params()
        est = C.c_double()
        win = C.c_uint64()
        self._check(self.L.gnna_b200_plan_params(self.h, _ptr(row_ptr), C.c_uint32(row_ptr.numel() - 1),
                                                 C.c_uint32(dim), C.c_int(dt), C.c_double(hbm_gbs), C.byref(p),
                                                 C.byref(est), C.byref(win)))
        return (p, est.value, win.value) if window else (p, est.value)

    def auto_params(self, inputs: ModelInputs) -> Params:
        p = Params()
        rc = self.L.gnna_auto_params(C.byref(inputs), C.byref(p))
        if rc:
            raise DomainError(rc, "auto_params")
        return p


class Plan:
    def __init__(self, ctx: Context, row_ptr, col, p: Params, strategy=WARP_SHARED, rows=None):
        self.ctx = ctx
        self.row_ptr, self.col = row_ptr, col  # keep alive
        self.params = Params(*p.tolist())
        self.strategy = strategy
        n = row_ptr.numel() - 1
        r0, r1 = rows if rows is not None else (0, n)
        self.n, self.rows = n, (r0, r1)
        h = C.c_void_p()
        ctx._check(ctx.L.gnna_plan_create(ctx.h, _ptr(row_ptr), _ptr(col), C.c_uint32(n), C.c_uint32(r0),
                                          C.c_uint32(r1), C.byref(self.params), C.c_int(strategy),
                                          C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                self.ctx.L.gnna_plan_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def info(self):
        g, r, s, c = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.ctx._check(self.ctx.L.gnna_plan_info(self.h, C.byref(g), C.byref(r), C.byref(s), C.byref(c)))
        return {"groups": g.value, "runs": r.value, "split_nodes": s.value, "carries": c.value}

    def _feat(self, x, out, width=None):
        torch = self.ctx.torch
        width = x.shape[1] if width is None else width
        _dev(x, "x", (torch.float32, torch.float64), (self.n, width))
        _dev(out, "out", x.dtype, (self.n, width))

    def aggregate(self, x, out=None, dim_mode=DIM_CYCLIC):
        if out is None:
            out = self.ctx.torch.zeros_like(x)
        # gnna_aggregate uses the plan's dim: x must have exactly that width
        self._feat(x, out, self.params.dim)
        self.ctx._check(self.ctx.L.gnna_aggregate(self.ctx.h, self.h, C.c_int(_dtype_code(x)),
                                                  C.c_int(dim_mode), _ptr(x), _ptr(out)))
        return out

    def aggregate_ex(self, x, out=None, node_weight=None, self_weight=None, alpha=0.0, row_scale=None, relu=False,
                     mask=None, dim_mode=DIM_CYCLIC):
        """gnna_aggregate_ex: y = relu?(row_scale * (A (node_weight x) + self_weight * x)) [masked]; any width."""
        if out is None:
            out = self.ctx.torch.empty_like(x)
        self._feat(x, out)
        f32 = self.ctx.torch.float32
        for t, nm in ((node_weight, "node_weight"), (self_weight, "self_weight"), (row_scale, "row_scale")):
            _dev(t, nm, f32, (self.n,))
        _dev(mask, "mask", x.dtype, tuple(x.shape))
        o = AggOpts(int(x.shape[1]), _ptr(node_weight), _ptr(self_weight), float(alpha), _ptr(row_scale), int(relu),
                    _ptr(mask))
        self.ctx._check(self.ctx.L.gnna_aggregate_ex(self.ctx.h, self.h, C.c_int(_dtype_code(x)), C.c_int(dim_mode),
                                                     _ptr(x), _ptr(out), C.byref(o)))
        return out

    def aggregate_fanout(self, x, out, peers=(), mc=None, node_weight=None, self_weight=None, alpha=0.0,
                         row_scale=None, relu=False, mask=None, dim_mode=DIM_CYCLIC):
        """gnna_aggregate_fanout: aggregate_ex on this plan's rows, every final
        row also written into each peer replica (device pointers or tensors:
        the other ranks' y, P2P-mapped) or, with `mc`, only through the NVLS
        multicast address of the replicated y."""
        self._feat(x, out)
        f32 = self.ctx.torch.float32
        for t, nm in ((node_weight, "node_weight"), (self_weight, "self_weight"), (row_scale, "row_scale")):
            _dev(t, nm, f32, (self.n,))
        _dev(mask, "mask", x.dtype, tuple(x.shape))
        peers = [p if isinstance(p, int) else p.data_ptr() for p in peers]
        if len(peers) > 7:
            raise ValueError("at most 7 peer replicas (GNNA_MAX_PEERS)")
        arr = (C.c_void_p * max(1, len(peers)))(*peers)
        o = AggOpts(int(x.shape[1]), _ptr(node_weight), _ptr(self_weight), float(alpha), _ptr(row_scale), int(relu),
                    _ptr(mask))
        mcp = None if mc is None else (mc if isinstance(mc, int) else mc.data_ptr())
        self.ctx._check(self.ctx.L.gnna_aggregate_fanout(self.ctx.h, self.h, C.c_int(_dtype_code(x)),
                                                         C.c_int(dim_mode), _ptr(x), _ptr(out), C.byref(o), arr,
                                                         C.c_uint32(len(peers)), C.c_void_p(mcp)))
        return out

    def cost(self, dim_mode=DIM_CYCLIC, line=128, cache=None):
        c = Cost()
        cap, cl = cache if cache else (0, 0)
        self.ctx._check(self.ctx.L.gnna_cost_report(self.ctx.h, self.h, C.c_int(dim_mode), C.c_uint64(line),
                                                    C.c_uint64(cap), C.c_uint64(cl), C.byref(c)))
        return c

    def simulate_cache(self, cache, dim):
        h, a = C.c_uint64(), C.c_uint64()
        self.ctx._check(self.ctx.L.gnna_simulate_cache(self.ctx.h, self.h, C.c_uint64(cache[0]),
                                                       C.c_uint64(cache[1]), C.c_uint32(dim), C.byref(h),
                                                       C.byref(a)))
        return h.value, a.value


# ---------------------------------------- synthetic inputs (host, no GPU)
def gen_edges(kind, n, pairs, seed, shuffle=False, gamma=2.3, i0=10.0, communities=1, p_intra=0.8, out=None):
    """gnna_gen_chung_lu / gnna_gen_sbm: (pairs, 2) uint32 node pairs drawn
    with the reference's mt19937_64 draws (rand.hpp:13-21), into `out` (a
    uint32 numpy array or a pinned CPU tensor's numpy view) when given."""
    if out is None:
        out = np.empty((pairs, 2), np.uint32)
    L = lib()
    if kind == "chung_lu":
        rc = L.gnna_gen_chung_lu(C.c_uint32(n), C.c_uint64(pairs), C.c_double(gamma), C.c_double(i0),
                                 C.c_uint64(seed), C.c_int(int(shuffle)), _ptr(out))
    else:
        rc = L.gnna_gen_sbm(C.c_uint32(n), C.c_uint64(pairs), C.c_uint32(communities), C.c_double(p_intra),
                            C.c_uint64(seed), C.c_int(int(shuffle)), _ptr(out))
    if rc:
        raise DomainError(rc, f"gen_edges({kind}): arguments outside the generator's domain")
    return out


def random_features(n, dim, seed, dtype=np.float32, out=None):
    """gnna_random_features = random_features(n, dim, seed) of
    pipeline.cpp:57-67 (fp32: the same doubles rounded)."""
    dt = F32 if np.dtype(dtype) == np.float32 else F64
    if out is None:
        out = np.empty((n, dim), dtype)
    rc = lib().gnna_random_features(C.c_uint32(n), C.c_uint32(dim), C.c_uint64(seed), C.c_int(dt), _ptr(out))
    if rc:
        raise DomainError(rc, "random_features: dim must be positive")
    return out


# ------------------------------------------------- evaluator (host, no GPU)
# decider.hpp:46-94: these run on the host inside libgnna.so and need no
# device, so the CPU test suite checks them against the reference.
class Decider:
    def __init__(self):
        self.L = lib()
        self.L.gnna_alpha_from_degrees.restype = C.c_double

    def _chk(self, rc, what):
        if rc:
            raise DomainError(rc, what)

    def alpha_from_degrees(self, avg, sd):
        return self.L.gnna_alpha_from_degrees(C.c_double(avg), C.c_double(sd))

    def select_dw(self, dim, tpw=32):
        out = C.c_uint32()
        self._chk(self.L.gnna_select_dw(C.c_uint32(dim), C.c_uint32(tpw), C.byref(out)), "select_dw")
        return out.value

    def select_ngs(self, dw, tpb, inputs):
        out = C.c_uint32()
        self._chk(self.L.gnna_select_ngs(C.c_uint32(dw), C.c_uint32(tpb), C.byref(inputs), C.byref(out)), "select_ngs")
        return out.value

    def dp_size(self, smem, avg):
        out = C.c_double()
        self._chk(self.L.gnna_dp_size(C.c_uint64(smem), C.c_double(avg), C.byref(out)), "dp_size")
        return out.value

    def estimate_latency(self, p: Params, inputs):
        out = C.c_double()
        self._chk(self.L.gnna_estimate_latency(C.byref(p), C.byref(inputs), C.byref(out)), "estimate_latency")
        return out.value

    def feasible(self, p: Params, inputs):
        return (bool(self.L.gnna_candidate_feasible(C.byref(p), C.byref(inputs))),
                bool(self.L.gnna_feasibility(C.byref(p), C.byref(inputs))))

    def auto_params(self, inputs) -> Params:
        p = Params()
        self._chk(self.L.gnna_auto_params(C.byref(inputs), C.byref(p)), "auto_params")
        return p

    def search_params(self, inputs, iterations=15, population=32, seed=1, gs=(1, 2, 4, 8, 16, 32, 64),
                      dw=(8, 16, 32), tpb=(32, 64, 128, 256)):
        g, d, t = (np.asarray(v, np.uint32) for v in (gs, dw, tpb))
        best = Params()
        lat, feas = C.c_double(), C.c_int()
        trace = np.zeros(iterations + 1, np.float64)
        tl = C.c_uint32()
        self._chk(self.L.gnna_search_params(C.byref(inputs), C.c_uint32(iterations), C.c_uint32(population),
                                            C.c_uint64(seed), _ptr(g), C.c_uint32(len(g)), _ptr(d), C.c_uint32(len(d)),
                                            _ptr(t), C.c_uint32(len(t)), C.byref(best), C.byref(lat), C.byref(feas),
                                            _ptr(trace), C.byref(tl)), "search_params")
        return best, lat.value, bool(feas.value), trace[: tl.value].copy()
