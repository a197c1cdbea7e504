"""K3P A/B (GPU): the C3 forms (sum, gcn layer form, gcn gather, gin; fp32
and the fp64 sum) and the C4 sum with whatever libgnna.so GNNA_LIB selects
(GNNA_K3P=0 forces the plain K3).  Every form is checked against an fp64
torch-sparse recompute (1e-5 / 1e-12) and timed as the median of `reps`
CUDA-event calls with L2 flushed between calls.  One JSON line per form."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2006_06608_b200.capi import Context  # noqa: E402


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("GNNA_LIB", "default")
    dev = torch.device("cuda", 0)
    ctx = Context(0)
    scratch = bench.l2_flush_buffer(dev)
    for w, cfg, agg, call, y, balg, form, nnz, p, reference in bench.agg_cases(ctx, dev):
        t = bench.time_calls(call, 20, scratch)
        call()
        par = bench.rel_check(y, reference(), tol=1e-12 if agg.endswith("f64") else 1e-5)
        l0 = ctx.launches
        call()
        print(json.dumps({"tag": tag, "case": f"{w}/{agg}", "ms": round(t, 5), "launches": ctx.launches - l0,
                          "ok": par["ok"], "max_rel_err": par["max_rel_err"],
                          "eff_frac": round(balg / (t * 1e-3) / 1e9 / 6544.7, 3)}), flush=True)


if __name__ == "__main__":
    main()
