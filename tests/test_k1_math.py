"""CPU: the arithmetic the K1 kernels rest on, checked against the oracle's Gear
states (oracle_gear_states, the restated chunking.py:107-118 loop):

  h_t = G_t + B_t (mod 2^64), G_t = sum_{k<64} g_{t-k} << k, B_{t+1} = (B_t << 1) + msb(h_t)

and the split form's region-start correction of a G computed over the flat
token array, G_local_t = G_flat_t - (G_flat_{rs-1} << (t - rs + 1)) for the
first 63 tokens of a region starting at rs (cdc.cu, cdc_region_split_kernel)."""

import numpy as np

from oracle import oracle as O


def test_gear_decomposition_and_region_correction():
    rng = np.random.default_rng(17)
    n = 3000
    tok = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    pins = [700, 701, 1999]  # two adjacent pins: a one-token region
    g = O.gear_table()[tok & 0xFFFF].astype(np.uint64)
    with np.errstate(over="ignore"):
        G = np.zeros(n, np.uint64)
        for k in range(64):
            G[k:] += g[:n - k] << np.uint64(k)
        h = O.gear_states(tok, pins)
        starts = [0] + [p + 1 for p in pins]
        ends = pins + [n - 1]
        checked = 0
        for rs, re in zip(starts, ends):
            B = np.uint64(0)
            for t in range(rs, re + 1):
                if t - rs < 63 and rs > 0:
                    Gl = G[t] - (G[rs - 1] << np.uint64(t - rs + 1))
                else:
                    Gl = G[t]
                ht = Gl + B
                if t != re or t not in pins:  # a pin token's state is reset (chunking.py:116-118)
                    assert ht == h[t], (rs, t)
                    checked += 1
                B = (B << np.uint64(1)) + (ht >> np.uint64(63))
    assert checked >= n - len(pins)
