for d in 0 8 4 12; do
  echo "== IRM_CDC_DEBUG=$d (8: walker skipped, 4: chain skipped)"
  IRM_CDC_DEBUG=$d K1_FORMS=v1,v2,v1,v2 timeout 120 python tools/k1_bench.py 8 32900 296 32768 2>&1 | tail -4
done
