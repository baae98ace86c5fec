summ() { python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,1), round(d['ms_per_step'],3), d['parity']['ok'])"; }
for i in 1 2; do
echo -n "default: "; timeout 300 python bench.py --workload config5 --no-cpu --steps 100 2>/dev/null | summ
echo -n "k4sms120: "; IRM_K4_SMS=120 timeout 300 python bench.py --workload config5 --no-cpu --steps 100 2>/dev/null | summ
echo -n "nok0: "; timeout 300 python tools/exp_front.py nok0 --workload config5 --no-cpu --steps 100 2>/dev/null | summ
done
