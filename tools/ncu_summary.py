"""Summarise an ncu report (raw page) for the judged metrics: time, DRAM
bytes, L2/L1 hit rates, occupancy, pipe utilisation, top stall reasons.
  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second"]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def main():
    path = sys.argv[1]
    hdr, units, data = load(path)
    idx = {h: i for i, h in enumerate(hdr)}
    res = []
    for r in data:
        d = {"kernel": r[idx["Kernel Name"]][:60]}
        for k in KEYS:
            if k in idx:
                d[k] = r[idx[k]]
        stalls = {h: r[i] for h, i in idx.items()
                  if h.startswith("smsp__average_warp_latency_issue_stalled") or
                  (h.startswith("smsp__warp_issue_stalled_") and h.endswith("_per_warp_active.pct"))}
        top = sorted(((float(v), k) for k, v in stalls.items() if v.replace(".", "").replace("-", "").isdigit()),
                     reverse=True)[:8]
        d["top_stalls"] = [(k.replace("smsp__", ""), round(v, 2)) for v, k in top]
        res.append(d)
    for d in res:
        print(json.dumps(d, indent=1))
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
