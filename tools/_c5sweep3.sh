summ() { python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,1), round(d['ms_per_step'],3), d['parity']['ok'])"; }
for n in 136 140 144 146; do
echo -n "c2 sharded k4sms $n: "; IRM_K4_SMS=$n timeout 300 python bench.py --sharded --no-cpu --no-attn --steps 100 2>/dev/null | summ
echo -n "c5 k4sms $n: "; IRM_K4_SMS=$n timeout 300 python bench.py --workload config5 --no-cpu --steps 100 2>/dev/null | summ
done
