"""Config 4 precision sweep (BASELINE.json): delta-rotation error vs |delta| on B200.

Unit k_r rows entangled at p_src = 5000 (kr_base = R(p_src) raw, f64), stored in the
pool at fp32 or bf16, re-rotated by K4 (irm_rotate_gather) by delta = +-2^e; rel-L2
against the f64 truth R(p_src + delta) raw (registry.py:146-166, rotary.py:98-108).
Prints a markdown table (one row per |delta|, worst sign) per theta.

  python tools/delta_sweep.py > profiles/r01_delta_sweep.md
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402  (test oracle: the f64 truth)
from paper_2605_05696_b200 import _native as N, ops  # noqa: E402


def sweep(theta, layout, n=4096, p_src=5000):
    rng = np.random.default_rng(int(theta) % 997)
    inv = O.make_inv_freq(theta)
    raw = rng.standard_normal((n, 64))
    raw /= np.linalg.norm(raw, axis=1, keepdims=True)
    interleaved = layout == N.LAYOUT_INTERLEAVED
    rot = (lambda x, pos: O.rotate_rows(x, pos, inv, interleaved=True)) if interleaved else \
        (lambda x, pos: O.rotate_rows(x, pos, inv))
    base = rot(raw, np.full(n, p_src))
    deltas = np.array([s * 2**e for e in range(18) for s in (1, -1)], np.int64)
    deltas = deltas[p_src + deltas >= 0]
    pool = np.zeros((1, n, 576))
    pool[0, :, 512:] = base
    d = lambda a: torch.from_numpy(a).cuda()
    res = {}
    for name, dt in (("fp32", torch.float32), ("bf16", torch.bfloat16)):
        out = torch.empty(1, n * deltas.size, 576, dtype=dt, device="cuda")
        ops.rotate_gather(d(pool).to(dt), out, d(np.zeros(deltas.size, np.int64)),
                          d(np.arange(deltas.size, dtype=np.int64) * n), d(np.full(deltas.size, n, np.int32)),
                          d(deltas), ops.inv_freq_device(inv), layout=layout)
        got = out.to(torch.float64).cpu().numpy()[0, :, 512:].reshape(deltas.size, n, 64)
        for i, dl in enumerate(deltas):
            e = O.rel_l2(got[i], rot(raw, np.full(n, p_src + dl)))
            res[(name, abs(int(dl)))] = max(res.get((name, abs(int(dl))), 0.0), e)
    return sorted({abs(int(x)) for x in deltas}), res


def main():
    print("# Config 4: delta-rotation error vs |delta| (B200, K4 `irm_rotate_gather`)\n")
    print("rel-L2 of the re-rotated k_r against the f64 truth, worst of +-delta, 4096 unit rows "
          "entangled at p_src = 5000; bounds: fp32 1e-5, bf16 4.7e-3 (BASELINE.json north_star).\n")
    for theta, layout, lname in ((1e4, N.LAYOUT_INTERLEAVED, "DSv2 interleaved"), (5e4, N.LAYOUT_HALF_SPLIT, "DSv3 half-split"),
                                 (3.2e7, N.LAYOUT_HALF_SPLIT, "DSv3 half-split")):
        ds, res = sweep(theta, layout)
        print(f"## theta {theta:g} ({lname})\n\n| abs(delta) | fp32 rel-L2 | bf16 rel-L2 |\n|---:|---:|---:|")
        for dl in ds:
            print(f"| 2^{int(np.log2(dl))} | {res[('fp32', dl)]:.2e} | {res[('bf16', dl)]:.2e} |")
        print(f"| **worst** | **{max(res[('fp32', x)] for x in ds):.2e}** | **{max(res[('bf16', x)] for x in ds):.2e}** |\n")


if __name__ == "__main__":
    main()
