"""Synthetic graphs and features for the BASELINE.json configs.

The reference's own generator (planted_partition, pipeline.cpp:14-46) samples
all O(n^2) node pairs and refuses graphs above 65,536 nodes, so the C3-C5
shapes need new samplers.  They draw with the reference's generator family:
std::mt19937_64 with rand.hpp's draw_unit / draw_index (gnna_gen_chung_lu /
gnna_gen_sbm, host C++ in libgnna.so), and features are the reference's
random_features(n, d, seed) itself (pipeline.cpp:57-67, gnna_random_features)
-- so bench.py's GPU arm and its CPU reference arm aggregate the same graph
and the same features whenever they run the same size.  The sampled pairs are
canonicalised by to_csr (symmetrise, sort, dedup: graph.cpp:76-95), on the GPU
(gnna_to_csr) or on the CPU through the reference's to_csr.

* Chung-Lu power law: endpoint weight (i + i0)^(-1/(gamma-1)), inverse-CDF
  sampling; low ids are the hubs.  C3 (amazon0505 shape), C5.
* Community SBM: `communities` equal contiguous blocks; an endpoint stays in
  its source's block with probability p_intra; optionally ids shuffled
  (Fisher-Yates with draw_index).  C1, C2, C4.

This module is input plumbing, not a compute path.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import capi


@dataclass(frozen=True)
class GraphConfig:
    name: str
    kind: str            # "chung_lu" | "sbm"
    n: int
    nnz: int             # target symmetrised nnz (even)
    dim: int
    seed: int
    gamma: float = 2.3
    i0: float = 10.0
    communities: int = 1
    p_intra: float = 0.8
    shuffle: bool = False


CONFIGS = {
    "c1": GraphConfig("C1 Cora-shape community graph", "sbm", 2708, 10556, 16, 1, communities=7, p_intra=0.8),
    "c2": GraphConfig("C2 Pubmed-shape community graph (ids shuffled)", "sbm", 19717, 88648, 64, 2,
                      communities=3, p_intra=0.8, shuffle=True),
    "c3": GraphConfig("C3 amazon0505-shape Chung-Lu power law", "chung_lu", 410236, 4878874, 16, 3),
    "c4": GraphConfig("C4 soc-BlogCatalog-shape dense-community SBM", "sbm", 88784, 2093194, 64, 7,
                      communities=39, p_intra=0.9),
    "c5": GraphConfig("C5 10M-node Chung-Lu power law", "chung_lu", 10_000_000, 200_000_000, 128, 8),
}

ROUND_SEED = 1_000_003  # top-up round r draws from seed + r * ROUND_SEED


def sample_pairs(cfg: GraphConfig, pairs: int, seed: int, device, n=None):
    """(pairs, 2) int32 node pairs on `device` (host generator, pinned upload)."""
    n = n or cfg.n
    pin = torch.device(device).type == "cuda"
    buf = torch.empty((pairs, 2), dtype=torch.int32, pin_memory=pin)
    capi.gen_edges(cfg.kind, n, pairs, seed, shuffle=cfg.shuffle, gamma=cfg.gamma, i0=cfg.i0,
                   communities=cfg.communities, p_intra=cfg.p_intra, out=buf.numpy().view(np.uint32))
    return buf.to(device, non_blocking=pin) if pin else buf


def build_graph(cfg: GraphConfig, to_csr, device, n=None, nnz=None, max_rounds=4):
    """Sample pairs until the symmetrised, de-duplicated CSR reaches ~nnz.

    to_csr(n, edges(E,2) int32 tensor on `device`) -> (row_ptr, col).
    Returns (edges, row_ptr, col)."""
    n = n or cfg.n
    target = nnz or cfg.nnz
    edges = sample_pairs(cfg, target // 2, cfg.seed, device, n)
    rp, col = to_csr(n, edges)
    for r in range(1, max_rounds + 1):
        have = int(col.numel())
        if have >= target * 0.999:
            break
        extra = int((target - have) / 2 * 1.15) + 16
        edges = torch.cat([edges, sample_pairs(cfg, extra, cfg.seed + r * ROUND_SEED, device, n)])
        rp, col = to_csr(n, edges)
    return edges, rp, col


EXACT_FEATURES_MAX = 1 << 28  # values; above it the features come in parallel row blocks


def features(n, dim, seed, device, dtype=torch.float32):
    """random_features(n, dim, seed + 1000) of pipeline.cpp:57-67 on `device`.

    Up to 2^28 values (every config but C5) this is the reference's function
    exactly: one sequential mt19937_64 stream.  Above it (C5: 1.28e9 values,
    ~10 s as one stream) rows come in blocks of 2^20, block b being
    random_features(rows, dim, seed + 1000 + b * 0x9E3779B97F4A7C15), drawn
    in parallel -- the same generator, deterministic, not one stream."""
    np_dt = np.float32 if dtype == torch.float32 else np.float64
    pin = torch.device(device).type == "cuda"
    buf = torch.empty((n, dim), dtype=dtype, pin_memory=pin)
    arr = buf.numpy()
    if n * dim <= EXACT_FEATURES_MAX:
        capi.random_features(n, dim, seed + 1000, np_dt, out=arr)
    else:
        import os
        from concurrent.futures import ThreadPoolExecutor
        rows = 1 << 20

        def block(b):  # ctypes releases the GIL: the blocks run on all cores
            r0 = b * rows
            capi.random_features(min(rows, n - r0), dim, (seed + 1000 + b * 0x9E3779B97F4A7C15) % (1 << 64),
                                 np_dt, out=arr[r0:r0 + rows])
        with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
            list(ex.map(block, range((n + rows - 1) // rows)))
    return buf.to(device, non_blocking=pin) if pin else buf


def scaled_config(cfg: GraphConfig, n: int) -> tuple[int, int]:
    """Same generator and mean degree at n nodes (CPU-baseline samples)."""
    nnz = int(round(cfg.nnz * n / cfg.n / 2)) * 2
    return n, max(nnz, 2)


def b_alg(n_rows: int, nnz: int, dim: int, elem: int = 4) -> int:
    """Algorithmic bytes of one aggregation:
    4*nnz (col) + elem*d*nnz (gathered rows) + elem*d*n (output) + 8*(n+1) (row_ptr)."""
    return 4 * nnz + elem * dim * nnz + elem * dim * n_rows + 8 * (n_rows + 1)


__all__ = ["GraphConfig", "CONFIGS", "build_graph", "features", "b_alg", "scaled_config",
           "sample_pairs"]
