"""Small-shape launches of every hot-path kernel, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck) under gpurun:

  compute-sanitizer --tool memcheck --target-processes all python tools/sanitize_cases.py [names]

Each case checks its own result against the oracle so a sanitizer run is also a
parity run. Cases: k1_fused k1_split k1_fused_table k1_split_table k2 k3 k4 k4_fanout k0 rebase producer k5_v3 k5_v2 k5_1sm"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2605_05696_b200 import _native as N, ops  # noqa: E402


def k1(form, table=False):
    import functools

    os.environ["IRM_CDC_FORM"] = form
    rng = np.random.default_rng(1)
    streams = [rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32) for n in (3000, 1, 777, 5000)]
    pins = [[100, 101, 2000], [], [5], [4095]]
    from paper_2605_05696_b200 import chunking

    orig = ops.cdc_xxh64
    if table:  # the Gear table read from memory instead of computed from the seed
        ops.cdc_xxh64 = functools.partial(orig, gear_from_table=True)
    try:
        t = chunking.cdc_chunk_batch(streams, chunking.ChunkerParams(), [set(p) for p in pins])
    finally:
        ops.cdc_xxh64 = orig
    st, ln, fp, fo, off = t.to_host()
    for i, s in enumerate(streams):
        o = O.cdc_chunk(s, pins=pins[i])
        assert np.array_equal(st[off[i]:off[i + 1]], o[0]) and np.array_equal(fp[off[i]:off[i + 1]], o[2])
    os.environ.pop("IRM_CDC_FORM")


def k2():
    from paper_2605_05696_b200.fingerprint import fingerprint_spans

    toks = np.arange(1000, dtype=np.uint32)
    fps = fingerprint_spans(toks, np.array([0, 10, 500]), np.array([1000 - 0, 7, 128]))
    assert int(fps[1]) == O.fingerprint(toks[10:17])


def k3():
    store = ops.ChunkStore(max_entries=64, pool_rows=10_000)
    fp = torch.tensor([5, 6, 5, 7, -1, 6], dtype=torch.int64, device="cuda")
    n = fp.numel()
    hit, entry, p_src, row = store.lookup_insert(fp, torch.arange(n, device="cuda"), torch.arange(n, device="cuda") * 10,
                                                 torch.full((n,), 3, dtype=torch.int32, device="cuda"))
    assert hit.tolist() == [0, 0, 1, 0, 0, 1]


def k4(fan):
    L, rows = 2, 600
    pool = torch.randn(L, rows, 576, device="cuda").to(torch.bfloat16)
    src = np.array([0, 100, 0, 300], np.int64)
    ln = np.array([40, 33, 40, 100], np.int32)
    dst = np.array([0, 40, 73, 113], np.int64)
    delta = np.array([5, -9, 77, 1 << 18], np.int64)
    out = torch.zeros(L, 213, 576, dtype=torch.bfloat16, device="cuda")
    d = lambda a: torch.from_numpy(a).cuda()
    inv = O.make_inv_freq(1e4)
    status = torch.zeros(1, dtype=torch.int64, device="cuda")
    if fan:
        g = ops.SourceGroups.alloc(4, "cuda")
        ops.group_by_source(d(src), d(dst), d(ln), d(delta), g)
        ops.rotate_gather_fanout(pool, out, g, ops.inv_freq_device(inv), layout=1, status=status)
    else:
        ops.rotate_gather(pool, out, d(src), d(dst), d(ln), d(delta), ops.inv_freq_device(inv), layout=1,
                          status=status)
    torch.cuda.synchronize()
    pu = pool.view(torch.int16).cpu().numpy().view(np.uint16)
    exp = np.zeros((L, 213, 576), np.uint16)
    O.rotate_gather_bf16(pu, exp, src, dst, ln, delta, inv, interleaved=True)
    assert np.array_equal(out.view(torch.int16).cpu().numpy().view(np.uint16), exp) and int(status) == 0


def k0():
    from paper_2605_05696_b200.radix import DeviceRadixTree

    tree = DeviceRadixTree(max_prefixes=1 << 12, max_tokens=1 << 14, max_sequences=64)
    seqs = [np.array([1, 2, 3, 4], np.uint32), np.array([1, 2, 9], np.uint32), np.array([1, 2, 3, 4, 5], np.uint32)]
    m, w = tree.match_insert(seqs, [0, 1, 2])
    assert m == [0, 2, 4]


def rebase():
    from paper_2605_05696_b200.radix import WavePrefixIndex

    idx = WavePrefixIndex(max_prefixes=1 << 12, arena_tokens=1 << 14, max_sequences=64)
    tok = torch.tensor([1, 2, 3, 4, 5, 1, 2, 3, 9, 9, 9], dtype=torch.int32, device="cuda")
    off = torch.tensor([0, 5, 11], dtype=torch.int64, device="cuda")
    m = torch.zeros(2, dtype=torch.int64, device="cuda")
    idx.match_insert_wave(tok, off, 2, m)
    tail = torch.zeros(11, dtype=torch.int32, device="cuda")
    toff = torch.zeros(3, dtype=torch.int64, device="cuda")
    poff = torch.zeros(3, dtype=torch.int64, device="cuda")
    pins = torch.zeros(4, dtype=torch.int64, device="cuda")
    ops.wave_rebase(tok, off, m, 2, torch.tensor([0, 1, 2], dtype=torch.int64, device="cuda"),
                    torch.tensor([1, 2, 4, 5], dtype=torch.int64, device="cuda"), tail, toff, poff, pins)
    torch.cuda.synchronize()
    assert m.tolist() == [0, 3] and toff.tolist() == [0, 5, 8] and tail[5:8].tolist() == [9, 9, 9]


def producer():
    pool = torch.randn(3, 50, 576, device="cuda").to(torch.bfloat16)
    kr = pool[:, :40, 512:]
    ops.rotate_rows_layered(kr, torch.arange(40, dtype=torch.float64, device="cuda"),
                            ops.inv_freq_device(O.make_inv_freq(1e4)), 1, out=kr)
    torch.cuda.synchronize()


def k5(kind):
    from oracle.mla_ref import mla_reattach_ref

    env = {"v3": {}, "v2": {"IRM_MLA_V2": "1"}, "1sm": {"IRM_MLA_1SM": "1"}}[kind]
    for k in ("IRM_MLA_V2", "IRM_MLA_1SM"):
        os.environ.pop(k, None)
    os.environ.update(env)
    g = torch.Generator(device="cuda").manual_seed(1)
    n_kv, n_q = 300, 70
    q = torch.randn(n_q, 16, 576, device="cuda", generator=g).to(torch.bfloat16)
    kv = torch.randn(n_kv, 576, device="cuda", generator=g).to(torch.bfloat16)
    chunk = (torch.arange(n_kv, device="cuda") // 100).to(torch.int32)
    deltas = torch.tensor([0, 77, -300], dtype=torch.int64, device="cuda")
    inv = O.make_inv_freq(1e4)
    cs = ops.chunk_cossin(deltas, ops.inv_freq_device(inv))
    out, _ = ops.mla_reattach_prefill(q, kv, n_kv, n_kv - n_q, 192 ** -0.5, kv_chunk=chunk, chunk_cs=cs)
    torch.cuda.synchronize()
    ref, _ = mla_reattach_ref(q, kv, n_kv - n_q, 192 ** -0.5, deltas.cpu().numpy()[chunk.cpu().numpy()], inv)
    assert float((out.double().cpu() - ref).norm() / ref.norm()) < 4.7e-3
    for k in env:
        os.environ.pop(k, None)


CASES = {"k1_fused": lambda: k1("fused"), "k1_split": lambda: k1("split"),
         "k1_fused_table": lambda: k1("fused", True), "k1_split_table": lambda: k1("split", True), "k2": k2, "k3": k3,
         "k4": lambda: k4(False), "k4_fanout": lambda: k4(True), "k0": k0, "rebase": rebase, "producer": producer,
         "k5_v3": lambda: k5("v3"), "k5_v2": lambda: k5("v2"), "k5_1sm": lambda: k5("1sm")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        print("case ok:", n, flush=True)
