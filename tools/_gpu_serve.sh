timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench
for i in range(3):
    d = bench.serve_api_component()
    print(round(d['value']/1e6,2), 'M tok/s', round(d['seconds']*1e3,1), 'ms', d['reference']['events_identical'] if 'reference' in d else '')
"
