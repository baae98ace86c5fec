#!/bin/bash
# one gpurun call: GPU tests, config-2 and config-5 bench lines, reference arm, K4 config-5 capture
set -x
TAG=${TAG:-r02t}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${TAG}_gputests.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --workload config5 > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; echo "c5 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rotate_gather_ws -s 6 -c 1 \
  -o gpurun_out/${TAG}_k4c5 -f python bench.py --workload config5 --steps 2 --warmup 3 --no-cpu --no-attn > gpurun_out/${TAG}_k4c5.log 2>&1; echo "ncu rc=$?"
