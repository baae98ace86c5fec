timeout 600 python bench.py --workload config5 > gpurun_out/r02v_c5.json 2> gpurun_out/r02v_c5.err; echo "c5 rc=$?"
wc -l gpurun_out/r02v_c5.json; tail -3 gpurun_out/r02v_c5.err
python -c "
import json; d=json.load(open('gpurun_out/r02v_c5.json')); print(d['value'], d['exchange'])"
