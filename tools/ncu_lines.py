"""Per-CUDA-line share of executed instructions and stall samples of one kernel in an ncu report
(run here, no GPU): python tools/ncu_lines.py <report.ncu-rep> [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
h = rows[hi]
iE, iS = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
lines, tot, tots = [], 0.0, 0.0
for r in rows[hi + 1:]:
    if len(r) > max(iE, iS) and r[0]:
        try:
            e, s = float(r[iE] or 0), float(r[iS] or 0)
        except ValueError:
            continue
        lines.append((e, s, r[0], r[1][:90]))
        tot += e
        tots += s
print(f"total warp instructions {tot:.0f}, stall samples {tots:.0f}")
for e, s, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{e / tot * 100:5.1f}% inst {s / tots * 100:5.1f}% samp  L{ln:5s} {src}")
