"""GPU: bench.py's own arm keeps the driver's JSON contract (one line; metric /
value / e2e with copy bytes / roofline with a measured peak / clocks /
gpu_launches from the library's counter / the CPU leg), on a short run."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("mode", [[], ["--serial"], ["--sharded"]])
def test_bench_json_line(mode):
    import bench

    p = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-attn"] + mode, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    # NCCL's own banner may precede it on stdout (sharded runs); the bench prints one JSON line
    lines = [l for l in p.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["metric"] == bench.METRIC and d["unit"] == bench.UNIT and d["n_gpus"] == 1
    assert d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["value"] > 1e7 and d["ms_per_step"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1.05 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["gpu_launches"] > 0 and d["gpu_launches"] % 3 == 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    c = d["cpu_baseline"]
    assert c["value"] > 0 and c["kind"] == "port" and c["cores"] >= 1
    assert {"cdc_hash", "cdc_hash_wide", "store_lookup"} <= set(d["components"])
    # in-run parity of the timed path: a fresh wave vs the sequential oracle
    par = d["parity"]
    assert par["ok"] and par["service_map_bit_exact"] and par["ckv_bit_exact"] and par["kv_rows_checked"] > 0, par


def test_bench_config5_json_line():
    """BASELINE configs[4] on the sharded path at N = 1 (64 sessions per GPU is the
    default; 16 keeps the test short): one JSON line, weak scaling, in-run parity."""
    p = subprocess.run([sys.executable, "bench.py", "--workload", "config5", "--steps", "3", "--warmup", "3",
                        "--sessions-per-gpu", "16"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["scaling"] == "weak" and d["value"] > 1e7 and d["e2e"]["value"] > 0
    assert d["config"]["sessions_per_gpu"] == 16 and d["parity"]["ok"], d["parity"]
    assert d["gpu_launches"] > 0


@pytest.mark.parametrize("workload", ["config2", "config5"])
def test_bench_two_ranks_on_one_gpu(workload):
    """The N-rank code path (sharded store, all-to-all exchange, CUDA-IPC peer pools,
    replica fetch) with two ranks on one GPU over gloo: it runs to one JSON line
    (timings not meaningful: the ranks share the GPU)."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = {**os.environ, "IRM_BENCH_ONE_DEVICE": "1", "IRM_BENCH_BACKEND": "gloo"}
    extra = ["--sessions-per-gpu", "16"] if workload == "config5" else ["--no-cpu", "--no-attn"]
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--workload", workload,
                        "--steps", "3", "--warmup", "3"] + extra, cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    # every rank's check wave against one global oracle over both ranks (config 5: the shared tool
    # document's rows were first written by one rank, so the other reads them through its replica)
    par = d["parity"]
    assert par["ok"] and par["kv_rows_checked"] > 0 and par["kv_rows_first_written_by_another_gpu"] > 0, par
