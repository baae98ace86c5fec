"""TEST INFRASTRUCTURE ONLY -- fp64 restatement of the fused reattach attention (K5).

No reference implementation exists (the fused
kernel is a "deliberate follow-up"); the attention is therefore UNPINNED by the
reference and this oracle restates the semantics from the paper. Its rotation
input is pinned: tests/golden/mla.npz (make_golden.py) feeds keys rotated by
the reference's KvRegistry.materialize, checked in tests/test_oracle_golden.py.
  * absorbed MLA: attention runs on the 512-dim latent
    c_KV with the 64-dim decoupled rotary key, scores over the 576-wide key;
  * reattach: the cached k_r is kr_base rotated by
    R(delta) = R(p - p_src) (rotary.py:98-108 math, fp64 angles);
  * causal prefill of the query positions q_pos0 .. q_pos0 + n_q - 1.
Everything in float64 from the same bf16 inputs the kernel sees. At the
benchmarked shapes (64K-128K keys) the checker samples query rows
(``q_index``) and may run its fp64 arithmetic on a torch device (``device``):
the same restated math, only executed where it finishes in seconds.
"""

from __future__ import annotations

import numpy as np
import torch

try:
    from . import oracle as O
except ImportError:  # pragma: no cover
    import oracle as O


def rotate_kr(kr_base: np.ndarray, delta_per_key: np.ndarray, inv_freq: np.ndarray, interleaved: bool):
    return O.rotate_rows(kr_base, delta_per_key, inv_freq, interleaved=interleaved)


def mla_reattach_ref(q: torch.Tensor, kv: torch.Tensor, q_pos0: int, scale: float,
                     delta_per_key: np.ndarray | None = None, inv_freq: np.ndarray | None = None,
                     interleaved: bool = False, q_index: np.ndarray | None = None, device: str = "cpu",
                     block: int = 32):
    """q [n_q, H, 576], kv [n_kv, 576] (c_KV || kr_base), both in REQUEST order.
    Returns (out [m, H, 512], lse [m, H]) float64 on the CPU for the query rows
    ``q_index`` (default: all n_q), query i sitting at position q_pos0 + i."""
    kv64 = kv.to(torch.float64).cpu().numpy().copy()
    if delta_per_key is not None:
        kv64[:, 512:] = rotate_kr(kv64[:, 512:], delta_per_key, inv_freq, interleaved)
    kvt = torch.from_numpy(kv64).to(device)
    n_q = q.shape[0]
    idx = np.arange(n_q) if q_index is None else np.asarray(q_index, np.int64)
    n_kv = kvt.shape[0]
    keys = torch.arange(n_kv, device=device).view(1, 1, n_kv)
    outs, lses = [], []
    for b0 in range(0, idx.size, block):
        sel = idx[b0:b0 + block]
        q64 = q[torch.from_numpy(sel).to(q.device)].to(device=device, dtype=torch.float64)
        s = torch.einsum("qhd,kd->qhk", q64, kvt) * scale
        pos = (q_pos0 + torch.from_numpy(sel).to(device)).view(-1, 1, 1)
        s = s.masked_fill(keys > pos, float("-inf"))
        lse = torch.logsumexp(s, dim=-1)
        p = torch.exp(s - lse.unsqueeze(-1))
        outs.append(torch.einsum("qhk,kd->qhd", p, kvt[:, :512]).cpu())
        lses.append(lse.cpu())
    return torch.cat(outs), torch.cat(lses)
