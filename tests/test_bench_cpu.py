"""bench.py's measurement helpers on CPU (no GPU): the ncu raw-page parser and
traffic summary the roofline's DRAM bytes come from, the per-call launch
grouping, the error-aware parity rule and the sampled spot check the JSON
line's parity fields use, and the peak lookup."""
import json
import os
import sys

import numpy as np
import pytest
import torch

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402

RAW = '''==PROF== Connected to process 1
"ID","Process ID","Kernel Name","dram__bytes_read.sum","dram__bytes_write.sum","gpu__time_duration.sum","lts__t_bytes.sum","lts__t_sector_hit_rate.pct","dram__throughput.avg.pct_of_peak_sustained_elapsed","lts__throughput.avg.pct_of_peak_sustained_elapsed"
"","","","byte","byte","nsecond","byte","%","%","%"
"0","77","void k3_aggregate<float, 4, 16, 2, 0, 0>(AggArgs)","70,000,000,000","6,000,000,000","11,800,000","158,000,000,000","22.4","78.7","51.3"
"1","77","void k3b_split<float, 4, 16, 0>(AggArgs, unsigned long)","1,000,000","2,000,000","7,000","9,000,000","10","5","4"
"2","77","broken row"
'''


def test_parse_ncu_raw_and_traffic_summary(tmp_path):
    p = tmp_path / "raw.csv"
    p.write_text(RAW)
    rows = bench.parse_ncu_raw(str(p))
    assert len(rows) == 2  # the header / units lines and the malformed row are skipped
    assert rows[0]["Kernel Name"].startswith("void k3_aggregate")
    assert rows[0]["dram__bytes_read.sum"] == 70e9 and rows[1]["gpu__time_duration.sum"] == 7000.0
    t = bench.traffic_summary(rows)
    assert t["dram_bytes"] == 70_000_000_000 + 6_000_000_000 + 1_000_000 + 2_000_000
    assert t["dram_read_bytes"] == 70_001_000_000
    assert t["lts_bytes"] == 158_009_000_000
    assert t["ncu_us"] == pytest.approx(11_807.0)
    # the dominant launch's percentages
    assert (t["l2_hit_pct"], t["dram_throughput_pct"], t["lts_throughput_pct"]) == (22.4, 78.7, 51.3)
    assert bench.traffic_summary([]) is None
    assert bench.parse_ncu_raw(str(tmp_path / "raw.csv")) == rows
    (tmp_path / "empty.csv").write_text("==PROF== nothing profiled\n")
    assert bench.parse_ncu_raw(str(tmp_path / "empty.csv")) == []


def test_split_rows_groups_launches_in_order():
    rows = [{"i": i} for i in range(7)]
    out = bench.split_rows(rows, [("sum", 2), ("gin", 1), ("gcn", 3)])
    assert [d["i"] for d in out["sum"]] == [0, 1]
    assert [d["i"] for d in out["gin"]] == [2]
    assert [d["i"] for d in out["gcn"]] == [3, 4, 5]
    assert bench.split_rows([], [("sum", 1)]) == {} and bench.split_rows(rows, None) == {}


def test_rel_check_is_error_aware():
    want = torch.tensor([1.0, -1.0, 1e-9, 0.0], dtype=torch.float64)
    bound = torch.tensor([1.0, 1.0, 2.0, 0.0], dtype=torch.float64)  # sum |terms|: cancellation at index 2
    got = want + torch.tensor([5e-6, -1e-6, 1e-5, 0.0], dtype=torch.float64)
    r = bench.rel_check(got.float(), want, bound)
    assert r["ok"] and r["elements"] == 4 and r["max_rel_err"] <= 1e-5
    bad = bench.rel_check((want + torch.tensor([0, 0, 1e-3, 0], dtype=torch.float64)).float(), want, bound)
    assert not bad["ok"]
    # non-negative inputs: bound defaults to |want| (a plain relative bar, halved)
    assert bench.rel_check(torch.tensor([1.00001]), torch.tensor([1.0], dtype=torch.float64))["ok"]


def _small_graph(n=300, seed=4):
    rng = np.random.default_rng(seed)
    deg = rng.integers(0, 9, n)
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
    col = rng.integers(0, n, int(rp[-1])).astype(np.uint32)
    return rp, col


@pytest.mark.parametrize("agg", ["sum", "gcn", "gin"])
def test_spot_check_matches_the_forms(agg):
    rp, col = _small_graph()
    n, dim = len(rp) - 1, 8
    x = torch.rand((n, dim), dtype=torch.float32, generator=torch.Generator().manual_seed(1))
    x64 = x.double().numpy()
    deg = np.diff(rp).astype(np.float64)
    norm = 1.0 / np.sqrt(np.maximum(deg, 1.0))
    y = np.zeros((n, dim))
    for v in range(n):
        nb = col[rp[v]:rp[v + 1]]
        if agg == "gcn":
            y[v] = norm[v] * (norm[nb][:, None] * x64[nb]).sum(0)
        else:
            y[v] = x64[nb].sum(0) + (1.1 * x64[v] if agg == "gin" else 0)
    yt = torch.from_numpy(y).float()
    colt = torch.from_numpy(col.view(np.int32))
    r = bench.spot_check(rp, colt, x, yt, [(0, n)], dim, rows=200, agg=agg)
    assert r["ok"] and r["max_rel_err"] <= 1e-6, r
    yt[5] += 1.0  # a wrong row is caught when sampled (row 5 is in the pick with this seed or the ends)
    r2 = bench.spot_check(rp, colt, x, yt, [(0, n)], dim, rows=n * 4, agg=agg)
    assert not r2["ok"]


def test_peaks_reads_the_measured_file():
    hbm, src = bench.peaks()
    d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    assert hbm == float(d["hbm_gbs"]) and src.startswith("measured")
