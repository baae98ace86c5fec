"""Summarise ncu captures for profiles/ (run here, no GPU needed).

  python profiles/ncu_summary.py launches <launches.csv>        # share of each kernel
  python profiles/ncu_summary.py full <prof.ncu-rep> [algo_bytes]  # key metrics of a --set full capture
"""

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_shared_mem", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard", "sm__inst_executed.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        agg[d["Kernel Name"].split("(")[0][:70]][0] += 1
        agg[d["Kernel Name"].split("(")[0][:70]][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print("| launches | total ns | share | kernel |\n|---:|---:|---:|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {v[0]} | {v[1]:.0f} | {100 * v[1] / tot:.2f}% | `{k}` |")


def full(path, algo_bytes=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        print(f"### {d['Kernel Name'][:120]}\n")
        print("| metric | value | unit |\n|---|---:|---|")
        for k in KEYS[1:]:
            if k in d:
                print(f"| {k} | {d[k]} | {u.get(k, '')} |")
        if algo_bytes and "dram__bytes_read.sum" in d:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rb = float(d["dram__bytes_read.sum"].replace(",", "")) * scale.get(u["dram__bytes_read.sum"], 1)
            wb = float(d["dram__bytes_write.sum"].replace(",", "")) * scale.get(u["dram__bytes_write.sum"], 1)
            print(f"\ntraffic = {rb + wb:.4g} B vs algorithmic {float(algo_bytes):.4g} B "
                  f"(ratio {(rb + wb) / float(algo_bytes):.3f})\n")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
