import cProfile, pstats, sys, io, time
sys.path.insert(0, ".")
import bench, torch
bench.serve_api_component()  # warm
pr = cProfile.Profile()
pr.enable()
d = bench.serve_api_component()
pr.disable()
print(d["value"], d["seconds"])
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(30)
print(s.getvalue()[:6000])
