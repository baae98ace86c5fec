for ls in 3 2 4 8 3 2 4 8; do
  IRM_PROD_LSPLIT=$ls timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import bench
d=bench.producer_component(6458.1)
print('lsplit $ls', round(d['launch_ms']*1e3,1), 'us', round(d['roofline']['frac'],3))"
done
for ls in 2 4 8; do IRM_PROD_LSPLIT=$ls timeout 200 python -m pytest tests/test_gpu_rotate.py tests/test_gpu_registry_store.py -q -x 2>&1 | tail -1; done
