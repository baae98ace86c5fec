# full GPU tests + config-2 / config-5 bench lines (TAG names the outputs)
TAG=${TAG:-r02u}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${TAG}_gputests.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
[ -n "$C5" ] && { timeout 600 python bench.py --workload config5 > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; echo "c5 rc=$?"; }
python - <<'PY'
import json,os
t=os.environ.get("TAG","r02u")
d=json.load(open(f"gpurun_out/{t}_bench.json"))
print(d["value"], d["e2e"]["value"], d["ms_per_step"], d["roofline"]["frac"], d["parity"]["ok"])
for k,v in d["components"].items(): print(k, v.get("value"), v.get("launch_ms"), (v.get("roofline") or {}).get("frac"))
PY
