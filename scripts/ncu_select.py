"""Reduce an `ncu --page raw --csv` export to the metrics worth committing:
metric,unit,value for time, DRAM/L2/L1 traffic, throughput, occupancy,
registers, tensor-pipe and TMEM activity and warp-stall samples."""
import csv
import sys

KEYS = ("gpu__time_duration", "dram__bytes", "dram__throughput", "lts__t_sector", "lts__throughput",
        "l1tex__throughput", "l1tex__data_bank_conflicts", "sm__throughput", "sm__warps_active",
        "launch__", "achieved_occupancy", "sm__pipe_tensor", "sm__inst_executed_pipe_tensor", "sm__mem_tensor",
        "sm__inst_executed_pipe_tmem", "smsp__pcsamp_warps_issue_stalled", "Kernel Name")


def main(src, dst):
    rows = list(csv.reader(open(src)))
    head, units, vals = rows[0], rows[1], rows[2]
    with open(dst, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["metric", "unit", "value"])
        for h, u, v in zip(head, units, vals):
            if any(k in h for k in KEYS) and not h.endswith("not_issued"):
                w.writerow([h, u, v])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
