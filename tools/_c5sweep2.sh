summ() { python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,1), round(d['ms_per_step'],3), d['parity']['ok'])"; }
for ch in 1 2 4; do
for n in 0 128 140; do
echo -n "c2 sharded nch $ch k4sms $n: "; NCCL_MAX_NCHANNELS=$ch NCCL_MIN_NCHANNELS=1 IRM_K4_SMS=$n timeout 300 python bench.py --sharded --no-cpu --no-attn --steps 100 2>/dev/null | summ
done; done
echo -n "c2 sharded default 112: "; timeout 300 python bench.py --sharded --no-cpu --no-attn --steps 100 2>/dev/null | summ
