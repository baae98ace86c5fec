cp paper_2605_05696_b200/engine.py /tmp/engine_new.py
i=0
for v in old new old new; do
  i=$((i+1))
  if [ $v = old ]; then cp tools/_engine_old.py.txt paper_2605_05696_b200/engine.py; else cp /tmp/engine_new.py paper_2605_05696_b200/engine.py; fi
  timeout 600 python bench.py --no-cpu --steps 20 > gpurun_out/serve_${v}_$i.json 2> gpurun_out/serve_${v}_$i.err; echo "rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/serve_${v}_$i.json')); s=d['components']['serve_api']; print('$v', round(s['value']/1e6,2), round(s['seconds']*1e3,1))" 2>&1 | tail -1
done
cp /tmp/engine_new.py paper_2605_05696_b200/engine.py
