"""TEST INFRASTRUCTURE ONLY — ctypes front end for the two CPU checkers.

* ``Oracle("orc")``  -> oracle/liboracle.so, the plain-C restatement
  (oracle/gnnsim_oracle.c).
* ``Oracle("ref")``  -> oracle/_ref/libgnnsim_ref.so, the UNMODIFIED reference
  (/root/reference/proj/src) compiled from its own sources plus the POD shim
  oracle/ref_shim.cpp.

Both libraries export the same POD signatures (prefix ``orc_`` / ``ref_``), so a
test runs one case through either and through the CUDA C-ABI.  Only tests/,
``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl reference``
legs may import this module, and only as the checker or the CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "orc": os.path.join(HERE, "liboracle.so"),
    "ref": os.path.join(HERE, "_ref", "libgnnsim_ref.so"),
}

STATUS = {0: "ok", 1: "DomainError", 2: "InternalError", 3: "ParseError", 4: "IoError",
          5: "error", 6: "buffer too small"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg


class PodInputs(C.Structure):
    """POD mirror of ModelInputs (decider.hpp:12-26), see ref_shim.cpp."""
    _fields_ = [("num_nodes", C.c_uint64), ("num_edges", C.c_uint64),
                ("dim", C.c_uint32), ("max_tpb", C.c_uint32),
                ("avg_degree", C.c_double), ("stddev_degree", C.c_double),
                ("smem_per_block", C.c_uint64), ("capability", C.c_uint64),
                ("alpha", C.c_double)]


def model_inputs(num_nodes=0, num_edges=0, dim=16, avg_degree=0.0, stddev_degree=0.0,
                 max_tpb=1024, smem_per_block=96 * 1024, capability=4096, alpha=0.15):
    """Defaults equal the reference's ModelInputs (decider.hpp:12-26)."""
    return PodInputs(num_nodes, num_edges, dim, max_tpb, avg_degree, stddev_degree,
                     smem_per_block, capability, alpha)


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else C.c_void_p(0)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def params_arr(ngs=16, dw=32, tpb=128, dim=16, tpw=32):
    return np.array([ngs, dw, tpb, tpw, dim], dtype=np.uint32)


class Oracle:
    def __init__(self, kind: str = "orc", path: str | None = None):
        self.kind = kind
        self.path = path or PATHS[kind]
        if not os.path.exists(self.path):
            raise FileNotFoundError(f"{self.path} not built (run __graft_entry__.build())")
        self.lib = C.CDLL(self.path)
        self._err = getattr(self.lib, f"{kind}_last_error")
        self._err.restype = C.c_char_p

    def _fn(self, name):
        return getattr(self.lib, f"{self.kind}_{name}")

    def _call(self, name, *args):
        f = self._fn(name)
        f.restype = C.c_int
        rc = f(*args)
        if rc != 0:
            msg = self._err().decode()
            raise OracleError(rc, msg)

    # ------------------------------------------------------------- graph
    def to_csr(self, n, edges, symmetrize=True):
        e = _u32(edges).reshape(-1, 2)
        cap = 2 * len(e) if symmetrize else len(e)
        row_ptr = np.zeros(n + 1, np.uint64)
        col = np.zeros(max(cap, 1), np.uint32)
        nnz = C.c_uint64()
        self._call("to_csr", C.c_uint32(n), _p(e), C.c_uint64(len(e)), C.c_int(int(symmetrize)),
                   _p(row_ptr), _p(col), C.c_uint64(cap), C.byref(nnz))
        return row_ptr, col[: nnz.value].copy()

    def aes(self, n, edges):
        e = _u32(edges).reshape(-1, 2)
        out = C.c_double()
        self._call("aes", C.c_uint32(n), _p(e), C.c_uint64(len(e)), C.byref(out))
        return out.value

    def should_reorder(self, n, edges):
        e = _u32(edges).reshape(-1, 2)
        out = C.c_int()
        self._call("should_reorder", C.c_uint32(n), _p(e), C.c_uint64(len(e)), C.byref(out))
        return bool(out.value)

    def degree_stats(self, row_ptr, col):
        row_ptr, col = _u64(row_ptr), _u32(col)
        a, m, s = C.c_double(), C.c_uint64(), C.c_double()
        self._call("degree_stats", C.c_uint32(len(row_ptr) - 1), _p(row_ptr), _p(col),
                   C.byref(a), C.byref(m), C.byref(s))
        return a.value, m.value, s.value

    # ---------------------------------------------------------- schedule
    def validate_params(self, p):
        self._call("validate_params", _p(_u32(p)))

    def partition_neighbors(self, row_ptr, col, ngs):
        row_ptr, col = _u64(row_ptr), _u32(col)
        n = len(row_ptr) - 1
        cap = max(int(row_ptr[-1]), 1)
        ids = np.zeros(cap, np.uint32)
        tg = np.zeros(cap, np.uint32)
        bg = np.zeros(cap, np.uint64)
        en = np.zeros(cap, np.uint64)
        g = C.c_uint64()
        self._call("partition_neighbors", C.c_uint32(n), _p(row_ptr), _p(col), C.c_uint32(ngs),
                   C.c_uint64(cap), C.byref(g), _p(ids), _p(tg), _p(bg), _p(en))
        k = g.value
        return ids[:k].copy(), tg[:k].copy(), bg[:k].copy(), en[:k].copy()

    def partition_dims(self, dim, dw, mode):
        lp = np.zeros(dw + 1, np.uint32)
        dims = np.zeros(max(dim, 1), np.uint32)
        self._call("partition_dims", C.c_uint32(dim), C.c_uint32(dw), C.c_int(mode), _p(lp), _p(dims))
        return [dims[lp[t]:lp[t + 1]].tolist() for t in range(dw)]

    def build_mem_plan(self, targets, p):
        t = _u32(targets)
        g = len(t)
        slots = np.zeros(max(g, 1), np.uint32)
        nodes = np.zeros(max(g, 1), np.uint32)
        lead = np.zeros(max(g, 1), np.uint8)
        smem = C.c_uint64()
        self._call("build_mem_plan", _p(t), C.c_uint64(g), _p(_u32(p)), _p(slots), _p(nodes),
                   _p(lead), C.byref(smem))
        return slots[:g].copy(), nodes[:g].copy(), lead[:g].copy(), smem.value

    # ------------------------------------------------------------ engine
    def aggregate_scheduled(self, row_ptr, col, x, p, strategy=2, dim_mode=1, workers=1,
                            line=128, cache=None):
        row_ptr, col, x, p = _u64(row_ptr), _u32(col), _f64(x), _u32(p)
        n = len(row_ptr) - 1
        y = np.zeros((n, int(p[4])), np.float64)
        cost = np.zeros(7, np.uint64)
        on = cache is not None
        cap, cl = cache if on else (0, 0)
        self._call("aggregate_scheduled", C.c_uint32(n), _p(row_ptr), _p(col), _p(x), _p(p),
                   C.c_int(strategy), C.c_int(dim_mode), C.c_uint32(workers), C.c_uint64(line),
                   C.c_int(int(on)), C.c_uint64(cap), C.c_uint64(cl), _p(y), _p(cost))
        return y, cost

    def aggregate_oracle(self, row_ptr, col, x):
        row_ptr, col, x = _u64(row_ptr), _u32(col), _f64(x)
        n = len(row_ptr) - 1
        dim = x.shape[1] if x.ndim == 2 else x.size // max(n, 1)
        y = np.zeros((n, dim), np.float64)
        self._call("aggregate_oracle", C.c_uint32(n), _p(row_ptr), _p(col), _p(x),
                   C.c_uint32(dim), _p(y))
        return y

    def count_transactions(self, addr, line=128):
        a = _u64(addr)
        out = C.c_uint64()
        self._call("count_transactions", _p(a) if len(a) else C.c_void_p(0), C.c_uint64(len(a)),
                   C.c_uint64(line), C.byref(out))
        return out.value

    def simulate_cache(self, row_ptr, col, p, cache, dim):
        row_ptr, col, p = _u64(row_ptr), _u32(col), _u32(p)
        h, a = C.c_uint64(), C.c_uint64()
        self._call("simulate_cache", C.c_uint32(len(row_ptr) - 1), _p(row_ptr), _p(col), _p(p),
                   C.c_uint64(cache[0]), C.c_uint64(cache[1]), C.c_uint32(dim), C.byref(h),
                   C.byref(a))
        return h.value, a.value

    def gcn_layer(self, row_ptr, col, x, w, self_loops=False):
        row_ptr, col, x, w = _u64(row_ptr), _u32(col), _f64(x), _f64(w)
        n = len(row_ptr) - 1
        y = np.zeros((n, w.shape[1]), np.float64)
        self._call("gcn_layer", C.c_uint32(n), _p(row_ptr), _p(col), _p(x), C.c_uint32(x.shape[1]),
                   _p(w), C.c_uint32(w.shape[1]), C.c_int(int(self_loops)), _p(y))
        return y

    def gin_layer(self, row_ptr, col, x, eps, w, b):
        row_ptr, col, x, w, b = _u64(row_ptr), _u32(col), _f64(x), _f64(w), _f64(b)
        n = len(row_ptr) - 1
        y = np.zeros((n, w.shape[1]), np.float64)
        self._call("gin_layer", C.c_uint32(n), _p(row_ptr), _p(col), _p(x), C.c_uint32(x.shape[1]),
                   C.c_double(eps), _p(w), C.c_uint32(w.shape[1]), _p(b), _p(y))
        return y

    def gcn_backward(self, row_ptr, col, x, w, dy, self_loops=False):
        row_ptr, col, x, w, dy = _u64(row_ptr), _u32(col), _f64(x), _f64(w), _f64(dy)
        n = len(row_ptr) - 1
        dx = np.zeros_like(x)
        dw = np.zeros_like(w)
        self._call("gcn_backward", C.c_uint32(n), _p(row_ptr), _p(col), _p(x),
                   C.c_uint32(x.shape[1]), _p(w), C.c_uint32(w.shape[1]),
                   C.c_int(int(self_loops)), _p(dy), _p(dx), _p(dw))
        return dx, dw

    def gin_backward(self, row_ptr, col, x, eps, w, b, dy):
        row_ptr, col, x, w, b, dy = (_u64(row_ptr), _u32(col), _f64(x), _f64(w), _f64(b),
                                     _f64(dy))
        n = len(row_ptr) - 1
        dx, dw, db = np.zeros_like(x), np.zeros_like(w), np.zeros_like(b)
        de = C.c_double()
        self._call("gin_backward", C.c_uint32(n), _p(row_ptr), _p(col), _p(x),
                   C.c_uint32(x.shape[1]), C.c_double(eps), _p(w), C.c_uint32(w.shape[1]),
                   _p(b), _p(dy), _p(dx), _p(dw), _p(db), C.byref(de))
        return dx, dw, db, de.value

    # ---------------------------------------------------------- renumber
    def detect_communities(self, row_ptr, col):
        row_ptr, col = _u64(row_ptr), _u32(col)
        n = len(row_ptr) - 1
        com = np.zeros(max(n, 1), np.uint32)
        k = C.c_uint32()
        self._call("detect_communities", C.c_uint32(n), _p(row_ptr), _p(col), _p(com), C.byref(k))
        return com[:n].copy(), k.value

    def modularity(self, row_ptr, col, com, ncom):
        row_ptr, col, com = _u64(row_ptr), _u32(col), _u32(com)
        q = C.c_double()
        self._call("modularity", C.c_uint32(len(row_ptr) - 1), _p(row_ptr), _p(col), _p(com),
                   C.c_uint32(ncom), C.byref(q))
        return q.value

    def build_mapping(self, com, ncom):
        com = _u32(com)
        n = len(com)
        o2n, n2o = np.zeros(max(n, 1), np.uint32), np.zeros(max(n, 1), np.uint32)
        self._call("build_mapping", C.c_uint32(n), _p(com), C.c_uint32(ncom), _p(o2n), _p(n2o))
        return o2n[:n].copy(), n2o[:n].copy()

    def mapping_from_vector(self, v):
        v = _u32(v)
        n = len(v)
        o2n, n2o = np.zeros(max(n, 1), np.uint32), np.zeros(max(n, 1), np.uint32)
        self._call("mapping_from_vector", C.c_uint32(n), _p(v), _p(o2n), _p(n2o))
        return o2n[:n].copy(), n2o[:n].copy()

    def apply_mapping_csr(self, row_ptr, col, o2n, n2o):
        row_ptr, col, o2n, n2o = _u64(row_ptr), _u32(col), _u32(o2n), _u32(n2o)
        n = len(row_ptr) - 1
        orp = np.zeros(n + 1, np.uint64)
        oc = np.zeros(max(len(col), 1), np.uint32)
        self._call("apply_mapping_csr", C.c_uint32(n), _p(row_ptr), _p(col), _p(o2n), _p(n2o),
                   _p(orp), _p(oc))
        return orp, oc[: len(col)].copy()

    def apply_mapping_edges(self, n, edges, o2n, n2o):
        e = _u32(edges).reshape(-1, 2)
        out = np.zeros_like(e)
        self._call("apply_mapping_edges", C.c_uint32(n), _p(e), C.c_uint64(len(e)), _p(_u32(o2n)),
                   _p(_u32(n2o)), _p(out))
        return out

    # ----------------------------------------------------------- pipeline
    def random_features(self, n, dim, seed):
        out = np.zeros((n, dim), np.float64)
        self._call("random_features", C.c_uint32(n), C.c_uint32(dim), C.c_uint64(seed), _p(out))
        return out

    def planted_partition(self, communities, size, p_in, p_out, shuffle, seed):
        n = communities * size
        cap = max(n * (n - 1) // 2, 1)
        edges = np.zeros((cap, 2), np.uint32)
        ne, nn = C.c_uint64(), C.c_uint32()
        self._call("planted_partition", C.c_uint32(communities), C.c_uint32(size),
                   C.c_double(p_in), C.c_double(p_out), C.c_int(int(shuffle)), C.c_uint64(seed),
                   C.c_uint64(cap), _p(edges), C.byref(ne), C.byref(nn))
        return nn.value, edges[: ne.value].copy()

    # ------------------------------------------------ ref-only (decider)
    def reorder_edges(self, n, edges):
        e = _u32(edges).reshape(-1, 2)
        o2n, n2o = np.zeros(max(n, 1), np.uint32), np.zeros(max(n, 1), np.uint32)
        k, q, a0, a1 = C.c_uint32(), C.c_double(), C.c_double(), C.c_double()
        self._call("reorder_edges", C.c_uint32(n), _p(e), C.c_uint64(len(e)), _p(o2n), _p(n2o),
                   C.byref(k), C.byref(q), C.byref(a0), C.byref(a1))
        return o2n[:n].copy(), n2o[:n].copy(), k.value, q.value, a0.value, a1.value

    def run_pipeline(self, n, edges, dim, params=None, strategy=2, dim_mode=1, force_reorder=None, seed=1,
                     cache=(64 * 1024, 128), workers=1):
        """pipeline.cpp:93-124 run_pipeline (reference only: "ref")."""
        e = _u32(edges).reshape(-1, 2)
        p_in = _u32(params if params is not None else [0, 0, 0, 0, 0])
        reordered, ncom, q = C.c_int(), C.c_uint32(), C.c_double()
        o2n = np.zeros(max(n, 1), np.uint32)
        aes = np.zeros(3, np.float64)
        p_out = np.zeros(5, np.uint32)
        rep = np.zeros(7, np.uint64)
        fr = -1 if force_reorder is None else int(bool(force_reorder))
        cap, line = cache if cache else (0, 0)
        # the output's width is the params' dim (auto: the config dim)
        width = int(p_in[4]) if params is not None else dim
        out = np.zeros((n, width), np.float64)
        self._call("run_pipeline", C.c_uint32(n), _p(e), C.c_uint64(len(e)), C.c_uint32(dim), _p(p_in),
                   C.c_int(strategy), C.c_int(dim_mode), C.c_int(fr), C.c_uint64(seed), C.c_uint64(cap),
                   C.c_uint64(line), C.c_uint(workers), C.byref(reordered), _p(o2n), C.byref(ncom), C.byref(q),
                   _p(aes), _p(p_out), _p(rep), _p(out))
        return {"reordered": bool(reordered.value), "o2n": o2n[:n], "num_communities": ncom.value,
                "modularity": q.value, "aes": aes[0], "aes_before": aes[1], "aes_after": aes[2],
                "params": p_out.tolist(), "report": rep.tolist(), "output": out}

    def model_inputs(self, row_ptr, col, dim):
        row_ptr, col = _u64(row_ptr), _u32(col)
        out = PodInputs()
        self._call("model_inputs", C.c_uint32(len(row_ptr) - 1), _p(row_ptr), _p(col),
                   C.c_uint32(dim), C.byref(out))
        return out

    def alpha_from_degrees(self, avg, sd):
        f = self._fn("alpha_from_degrees")
        f.restype = C.c_double
        return f(C.c_double(avg), C.c_double(sd))

    def select_dw(self, dim, tpw=32):
        out = C.c_uint32()
        self._call("select_dw", C.c_uint32(dim), C.c_uint32(tpw), C.byref(out))
        return out.value

    def select_ngs(self, dw, tpb, inputs):
        out = C.c_uint32()
        self._call("select_ngs", C.c_uint32(dw), C.c_uint32(tpb), C.byref(inputs), C.byref(out))
        return out.value

    def dp_size(self, smem_bytes, avg):
        out = C.c_double()
        self._call("dp_size", C.c_uint64(smem_bytes), C.c_double(avg), C.byref(out))
        return out.value

    def estimate_latency(self, p, inputs):
        out = C.c_double()
        self._call("estimate_latency", _p(_u32(p)), C.byref(inputs), C.byref(out))
        return out.value

    def feasible(self, p, inputs):
        a, b = C.c_int(), C.c_int()
        self._call("feasible", _p(_u32(p)), C.byref(inputs), C.byref(a), C.byref(b))
        return bool(a.value), bool(b.value)

    def auto_params(self, inputs):
        p = np.zeros(5, np.uint32)
        self._call("auto_params", C.byref(inputs), _p(p))
        return p

    def search_params(self, inputs, iterations=15, population=32, seed=1,
                      gs=(1, 2, 4, 8, 16, 32, 64), dw=(8, 16, 32), tpb=(32, 64, 128, 256)):
        gs, dw, tpb = _u32(gs), _u32(dw), _u32(tpb)
        p = np.zeros(5, np.uint32)
        lat, feas = C.c_double(), C.c_int()
        trace = np.zeros(iterations + 1, np.float64)
        tl = C.c_uint32()
        self._call("search_params", C.byref(inputs), C.c_uint32(iterations),
                   C.c_uint32(population), C.c_uint64(seed), _p(gs), C.c_uint32(len(gs)), _p(dw),
                   C.c_uint32(len(dw)), _p(tpb), C.c_uint32(len(tpb)), _p(p), C.byref(lat),
                   C.byref(feas), _p(trace), C.byref(tl))
        return p, lat.value, bool(feas.value), trace[: tl.value].copy()


def available(kind: str) -> bool:
    return os.path.exists(PATHS[kind])
