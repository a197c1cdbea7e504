"""Generate tests/golden/ref_golden.npz from the REFERENCE itself.

Runs the unmodified reference (oracle/_ref/libgnnsim_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile) on seeded small cases and stores
inputs and outputs, so the parity tests have reference-produced vectors even
where /root/reference (and so oracle/_ref) is absent, e.g. on the GPU box.

    python tests/golden/make_golden.py      # needs oracle/_ref built

Cases (all n <= 300 so the file stays small):
  csr/*    to_csr (graph.cpp:76)           on random edge lists, sym and not
  part/*   partition_neighbors (schedule.cpp:16)
  plan/*   build_mem_plan (memplan.cpp:9)  on random consecutive-run targets
  agg/*    aggregate_scheduled (engine.cpp:200), 3 strategies x 2 dim modes,
           fp64 outputs + the full CostReport (LRU cache on)
  orc/*    aggregate_oracle (engine.cpp:149)
  gcn/*    gcn_layer (engine.cpp:373), both update orders, with/without self loops
  gin/*    gin_layer (engine.cpp:384)
  com/*    detect_communities / modularity / build_mapping / apply_mapping
  aes/*    aes, degree_stats
  dec/*    auto_params on ModelInputs::from_graph
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.cpu import Oracle  # noqa: E402

OUT = os.path.join(HERE, "ref_golden.npz")


def main():
    ref = Oracle("ref")
    rng = np.random.default_rng(20260101)
    d = {}

    def graph(n, e, sym=True):
        edges = rng.integers(0, n, size=(e, 2)).astype(np.uint32)
        rp, col = ref.to_csr(n, edges, sym)
        return edges, rp, col

    # to_csr
    for i in range(12):
        n = int(rng.integers(1, 120))
        edges, rp, col = graph(n, int(rng.integers(0, 6 * n + 1)), bool(i % 2))
        d[f"csr/{i}/n"] = np.array([n])
        d[f"csr/{i}/sym"] = np.array([i % 2])
        d[f"csr/{i}/edges"] = edges
        d[f"csr/{i}/rp"] = rp
        d[f"csr/{i}/col"] = col

    # partition_neighbors
    for i in range(12):
        n = int(rng.integers(1, 200))
        _, rp, col = graph(n, int(rng.integers(0, 8 * n + 1)))
        ngs = int(rng.choice([1, 2, 3, 7, 16, 64]))
        ids, tg, bg, en = ref.partition_neighbors(rp, col, ngs)
        d[f"part/{i}/rp"] = rp
        d[f"part/{i}/ngs"] = np.array([ngs])
        d[f"part/{i}/target"] = tg
        d[f"part/{i}/begin"] = bg
        d[f"part/{i}/end"] = en

    # build_mem_plan
    for i in range(40):
        t = []
        for v in range(1 + int(rng.integers(0, 40))):
            t += [v] * int(rng.integers(0, 6))
        t = np.array(t or [0], np.uint32)
        p = np.array([16, 32, 32 * int(rng.integers(1, 33)), 32, int(rng.integers(1, 65))], np.uint32)
        s, nodes, lead, smem = ref.build_mem_plan(t, p)
        d[f"plan/{i}/targets"] = t
        d[f"plan/{i}/params"] = p
        d[f"plan/{i}/slot"] = s
        d[f"plan/{i}/leader"] = lead
        d[f"plan/{i}/smem"] = np.array([smem], np.uint64)

    # aggregate_scheduled + cost report, aggregate_oracle
    dims = [1, 3, 16, 33, 64, 8]
    for i in range(24):
        n = int(rng.integers(2, 120))
        _, rp, col = graph(n, int(rng.integers(1, 10 * n)))
        dim = dims[i % len(dims)]
        x = rng.random((n, dim))
        p = np.array([1 + int(rng.integers(0, 40)), 1 + int(rng.integers(0, 32)), 32 * (1 + int(rng.integers(0, 16))),
                      32, dim], np.uint32)
        line = int(rng.choice([32, 128]))
        cache = (int(rng.choice([2, 16, 512])) * 128, 128)
        d[f"agg/{i}/rp"] = rp
        d[f"agg/{i}/col"] = col
        d[f"agg/{i}/x"] = x
        d[f"agg/{i}/params"] = p
        d[f"agg/{i}/line"] = np.array([line])
        d[f"agg/{i}/cache"] = np.array(cache)
        for s in (0, 1, 2):
            for m in (0, 1):
                y, cost = ref.aggregate_scheduled(rp, col, x, p, s, m, workers=2, line=line, cache=cache)
                d[f"agg/{i}/y_{s}{m}"] = y
                d[f"agg/{i}/cost_{s}{m}"] = cost
        d[f"orc/{i}/y"] = ref.aggregate_oracle(rp, col, x)

    # GCN / GIN layers (signed weights)
    for i in range(10):
        n = int(rng.integers(2, 150))
        _, rp, col = graph(n, int(rng.integers(1, 6 * n)))
        din, dout = int(rng.integers(1, 24)), int(rng.integers(1, 24))
        x = rng.random((n, din)) - 0.3
        w = rng.random((din, dout)) * 2 - 1
        b = rng.random(dout) - 0.5
        sl = bool(i % 2)
        eps = float(rng.choice([0.0, 0.1, -0.25]))
        d[f"gcn/{i}/rp"], d[f"gcn/{i}/col"], d[f"gcn/{i}/x"], d[f"gcn/{i}/w"] = rp, col, x, w
        d[f"gcn/{i}/self_loops"] = np.array([int(sl)])
        d[f"gcn/{i}/y"] = ref.gcn_layer(rp, col, x, w, sl)
        d[f"gin/{i}/b"], d[f"gin/{i}/eps"] = b, np.array([eps])
        d[f"gin/{i}/y"] = ref.gin_layer(rp, col, x, eps, w, b)

    # renumbering
    for i in range(8):
        n = int(rng.integers(4, 120))
        edges, rp, col = graph(n, int(rng.integers(n, 4 * n)))
        com, k = ref.detect_communities(rp, col)
        q = ref.modularity(rp, col, com, k)
        o2n, n2o = ref.build_mapping(com, k)
        orp, ocol = ref.apply_mapping_csr(rp, col, o2n, n2o)
        oe = ref.apply_mapping_edges(n, edges, o2n, n2o)
        d[f"com/{i}/edges"], d[f"com/{i}/rp"], d[f"com/{i}/col"] = edges, rp, col
        d[f"com/{i}/com"], d[f"com/{i}/k"], d[f"com/{i}/q"] = com, np.array([k]), np.array([q])
        d[f"com/{i}/o2n"], d[f"com/{i}/n2o"] = o2n, n2o
        d[f"com/{i}/orp"], d[f"com/{i}/ocol"], d[f"com/{i}/oedges"] = orp, ocol, oe
        d[f"aes/{i}/aes"] = np.array([ref.aes(n, edges)])
        d[f"aes/{i}/stats"] = np.array(ref.degree_stats(rp, col), dtype=np.float64)
        mi = ref.model_inputs(rp, col, int(rng.choice([16, 64, 128])))
        d[f"dec/{i}/inputs"] = np.array([mi.num_nodes, mi.num_edges, mi.dim], np.uint64)
        d[f"dec/{i}/fin"] = np.array([mi.avg_degree, mi.stddev_degree, mi.alpha])
        d[f"dec/{i}/auto"] = ref.auto_params(mi)

    np.savez_compressed(OUT, **d)
    print(f"wrote {OUT}: {len(d)} arrays, {os.path.getsize(OUT)} bytes")
    c2_communities(ref)


def c2_communities(ref):
    """tests/golden/c2_communities.npz: the reference's detect_communities on
    the C2 (Pubmed-shape) synthetic graph — ~30 s of reference CPU time, kept
    as a fixture so the GPU test does not need the reference."""
    import torch
    from paper_2006_06608_b200 import synth
    cfg = synth.CONFIGS["c2"]

    def to_csr(n, e):
        rp, col = ref.to_csr(n, e.numpy().astype(np.uint32), True)
        return rp, torch.from_numpy(col.view(np.int32))

    _, rp, col = synth.build_graph(cfg, to_csr, "cpu")
    col = col.numpy().view(np.uint32)
    com, k = ref.detect_communities(rp, col)
    q = ref.modularity(rp, col, com, k)
    out = os.path.join(HERE, "c2_communities.npz")
    np.savez_compressed(out, rp=rp, col=col, com=com, k=np.array([k]), q=np.array([q]))
    print(f"wrote {out}: n={len(rp) - 1} nnz={len(col)} communities={k}")


if __name__ == "__main__":
    main()
