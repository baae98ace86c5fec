"""K1 timing: irm_cdc_xxh64 over n_streams random streams, eager launches between
CUDA events (v1 = IRM_CDC_FORM=fused, v2 = split; the library reads it per call, so both forms time in one
process; t1 / t2 = the same forms reading the Gear table instead of computing it from the seed).
Usage: python tools/k1_bench.py [n_streams n_tok ...]"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_05696_b200 import ops  # noqa: E402


def time_k1(n_streams, n_tok, reps=int(os.environ.get("K1_REPS", "20")), forms=os.environ.get("K1_FORMS", "v1,v2,v1,v2")):
    rng = np.random.default_rng(21)
    tok = torch.from_numpy(rng.integers(0, 2**32, size=n_streams * n_tok, dtype=np.uint64).astype(np.uint32)
                           .view(np.int32)).cuda()
    off = torch.arange(0, (n_streams + 1) * n_tok, n_tok, dtype=torch.int64, device="cuda")
    ws = ops.CdcWorkspace()
    table = [False]
    run = lambda: ops.cdc_xxh64(tok, off, None, None, 7, 32, 512, True, ws=ws, n_tokens=tok.numel(),
                                gear_from_table=table[0])
    out = {}
    for form in forms.split(","):
        os.environ["IRM_CDC_FORM"] = {"1": "fused", "2": "split"}[form[1]]
        table[0] = form[0] == "t"
        t = run()
        torch.cuda.synchronize()
        ref = (t.start.clone(), t.fp.clone(), int(t.chunk_off[-1].item()))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            run()
        b.record()
        torch.cuda.synchronize()
        out[form] = (a.elapsed_time(b) / reps, ref)
    same = None
    if len(out) > 1:
        same = True
        (_, r1) = next(iter(out.values()))
        for _, r2 in out.values():
            same &= r1[2] == r2[2] and torch.equal(r1[0][:r1[2]], r2[0][:r2[2]]) and torch.equal(r1[1][:r1[2]], r2[1][:r2[2]])
    for form in out:
        ms = out[form][0]
        print(f"{n_streams:4d} x {n_tok:6d} {form}: {ms * 1e3:8.1f} us  {n_streams * n_tok / ms / 1e6:8.2f} G tok/s"
              f"  identical={same}")


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]] or [8, 32900, 296, 32768, 64, 32768]
    for i in range(0, len(a), 2):
        time_k1(a[i], a[i + 1])
