"""Synthetic graphs and features for the BASELINE.json configs.

The reference's own generator (planted_partition, pipeline.cpp:14-46) samples
all O(n^2) node pairs and refuses graphs above 65,536 nodes, so the C3-C5
shapes need a new generator.  These are edge samplers; the graph is then
canonicalised by to_csr (symmetrise, sort, dedup: graph.cpp:76-95), on the GPU
through libgnna (gnna_to_csr) or on the CPU through the reference's to_csr.

* Chung-Lu power law: endpoint i is drawn with weight (i + i0)^(-beta),
  beta = 1/(gamma-1), by inverting the continuous CDF of that weight.  Low
  ids are the hubs.  Used for C3 (amazon0505 shape) and C5.
* Community SBM: nodes are split into `communities` equal contiguous blocks
  (optionally shuffled); an edge's destination stays in the source's block
  with probability p_intra.  Used for C1, C2, C4.

Edge samples are drawn with torch generators (CPU or CUDA); this module is
input plumbing, not a compute path.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


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


def _gen(device, seed):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def chung_lu_pairs(n, pairs, gamma, i0, gen, device):
    beta = 1.0 / (gamma - 1.0)
    a = 1.0 - beta
    lo = i0 ** a
    hi = (n + i0) ** a
    u = torch.rand((pairs, 2), generator=gen, device=device, dtype=torch.float64)
    x = torch.pow(lo + u * (hi - lo), 1.0 / a) - i0
    return torch.clamp(x.floor(), 0, n - 1).to(torch.int32)


def sbm_pairs(n, pairs, communities, p_intra, gen, device, perm=None):
    size = max(1, n // communities)
    src = torch.randint(0, n, (pairs,), generator=gen, device=device, dtype=torch.int64)
    intra = torch.rand(pairs, generator=gen, device=device) < p_intra
    com = torch.clamp(src // size, max=communities - 1)
    base = com * size
    span = torch.where(com == communities - 1, n - base, torch.full_like(base, size))
    r = torch.rand(pairs, generator=gen, device=device, dtype=torch.float64)
    dst_in = base + (r * span).floor().to(torch.int64)
    dst_out = torch.randint(0, n, (pairs,), generator=gen, device=device, dtype=torch.int64)
    dst = torch.where(intra, dst_in, dst_out)
    e = torch.stack([src, dst], 1)
    if perm is not None:
        e = perm[e]
    return e.to(torch.int32)


def sample_pairs(cfg: GraphConfig, pairs: int, gen, device, n=None):
    n = n or cfg.n
    if cfg.kind == "chung_lu":
        return chung_lu_pairs(n, pairs, cfg.gamma, cfg.i0, gen, device)
    perm = None
    if cfg.shuffle:
        perm = torch.randperm(n, generator=gen, device=device)
    return sbm_pairs(n, pairs, cfg.communities, cfg.p_intra, gen, device, perm)


def build_graph(cfg: GraphConfig, to_csr, device, n=None, nnz=None, max_rounds=4):
    """Sample edges until the symmetrised, de-duplicated CSR reaches ~nnz.

    to_csr(n, edges(E,2) int32 tensor on `device`) -> (row_ptr, col).
    Returns (edges, row_ptr, col)."""
    n = n or cfg.n
    target = nnz or cfg.nnz
    gen = _gen(device, cfg.seed)
    edges = sample_pairs(cfg, target // 2, gen, device, n)
    rp, col = to_csr(n, edges)
    for _ in range(max_rounds):
        have = int(col.numel())
        if have >= target * 0.999:
            break
        extra = int((target - have) / 2 * 1.15) + 16
        edges = torch.cat([edges, sample_pairs(cfg, extra, gen, device, n)])
        rp, col = to_csr(n, edges)
    return edges, rp, col


def features(n, dim, seed, device, dtype=torch.float32):
    """U[0,1) features (random_features semantics, pipeline.cpp:57-67)."""
    return torch.rand((n, dim), generator=_gen(device, seed + 1000), device=device, dtype=dtype)


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
