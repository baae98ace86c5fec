"""Where the drop-in serve API's time goes (bench.py components.serve_api workload):
parse_trace, EngineState, run_trace, timed separately over a few passes."""
import io
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2605_05696_b200 import engine, model  # noqa: E402
from paper_2605_05696_b200.chunking import canonical_marker  # noqa: E402

shared = np.random.default_rng(7)
header = tuple(int(t) for t in shared.integers(0, 2**32, size=bench.HEADER, dtype=np.uint64))
body = tuple(int(t) for t in shared.integers(0, 2**32, size=bench.BODY, dtype=np.uint64))
marker = tuple(canonical_marker())
rng = np.random.default_rng(99)
reqs = []
for i in range(9):
    meta = tuple(int(t) for t in rng.integers(0, 2**32, size=int(rng.integers(30, 71)), dtype=np.uint64))
    reqs.append(model.Request(f"s{i}", 0, (model.Segment("system", header, "agent_header"),
                                           model.Segment("header", meta), model.Segment("marker", marker),
                                           model.Segment("body", body, "agent_body"))))
text = model.serialize_trace(model.Trace(tuple(reqs)))
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    trace = model.parse_trace(io.StringIO(text))
    t1 = time.perf_counter()
    state = engine.EngineState(engine.ServeConfig())
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    results, row = engine.run_trace(state, trace)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"pass {it}: parse {1e3 * (t1 - t0):.2f} ms, state {1e3 * (t2 - t1):.2f} ms, run_trace {1e3 * (t3 - t2):.2f} ms")
    del state, trace
if "--prof" in sys.argv:
    import cProfile
    import pstats
    trace = model.parse_trace(io.StringIO(text))
    state = engine.EngineState(engine.ServeConfig())
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    engine.run_trace(state, trace)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
if "--state" in sys.argv:
    import cProfile
    import pstats
    for _ in range(2):
        s = engine.EngineState(engine.ServeConfig())
        torch.cuda.synchronize()
        del s
    pr = cProfile.Profile()
    pr.enable()
    s = engine.EngineState(engine.ServeConfig())
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumtime").print_stats(25)
