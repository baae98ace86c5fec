#!/bin/bash
# tools/clock_probe.sh <command...>: runs the command while nvidia-smi samples SM clock and power
# every 50 ms; prints the command's output, then median / min SM MHz and median / max W of the
# samples taken while the GPU was busy (utilization > 50 %)
nvidia-smi --query-gpu=clocks.sm,power.draw,utilization.gpu,clocks_event_reasons.active --format=csv,noheader,nounits -lms 50 > /tmp/clk.csv &
P=$!
sleep 1
"$@"
kill $P
python - <<'PY'
import statistics
rows=[l.split(',') for l in open('/tmp/clk.csv') if l.strip()]
busy=[(float(r[0]),float(r[1]),r[3].strip()) for r in rows if r[2].strip().isdigit() and int(r[2])>50]
if busy:
    sm=[b[0] for b in busy]; w=[b[1] for b in busy]
    print("busy samples %d: SM MHz median %.0f min %.0f; power W median %.0f max %.0f; reasons %s" % (
        len(busy), statistics.median(sm), min(sm), statistics.median(w), max(w), sorted({b[2] for b in busy})))
PY
