import sys, time
sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import mla_bench
t0 = time.time()
while time.time() - t0 < float(sys.argv[1]):
    mla_bench.main(65536, 4096, reps=20)
