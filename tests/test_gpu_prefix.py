"""GPU parity of K0 (csrc/prefix.cu, radix.DeviceRadixTree) against the
reference RadixTree's own outputs (tests/golden/radix.npz, made by
make_golden.py from radix.py:31-83) and the brute-force oracle the reference
tests pin it with (test_radix.py:15-23): longest match m bit-exact and the
earliest-inserted witness, for op sequences run as one batch, in small
batches, and one op at a time through the scalar API."""

import numpy as np
import pytest
import torch

from goldens import load_npz
from inputs import RADIX_CASES, radix_case_inputs
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _tree(**kw):
    from paper_2605_05696_b200.radix import DeviceRadixTree

    args = dict(max_prefixes=1 << 20, max_tokens=1 << 22, max_sequences=1 << 14)
    args.update(kw)
    return DeviceRadixTree(**args)


@pytest.mark.parametrize("batch", [None, 7, 1])
@pytest.mark.parametrize("case", sorted(RADIX_CASES))
def test_prefix_ops_golden(case, batch):
    g = load_npz("radix")[case]
    ops = radix_case_inputs(RADIX_CASES[case])
    if batch == 1 and len(ops) > 500:
        ops = ops[:500]
    tree = _tree()
    bs = batch or len(ops)
    got_m, got_w = np.full(len(ops), -1), np.full(len(ops), -1)
    for b0 in range(0, len(ops), bs):
        part = ops[b0:b0 + bs]
        ins = [o[0] for o in part]
        m, w = tree.run_ops([o[1] for o in part], ins, [not x for x in ins], handles=list(range(b0, b0 + len(part))))
        m, w = m.cpu().numpy(), w.cpu().numpy()
        for k, (is_ins, _) in enumerate(part):
            if not is_ins:
                got_m[b0 + k] = m[k]
                got_w[b0 + k] = tree.handles[w[k]] if m[k] > 0 else -1
    tree.check()
    q = np.array([not o[0] for o in ops])
    assert np.array_equal(got_m[q], g["m"][:len(ops)][q])
    assert np.array_equal(got_w[q], g["witness"][:len(ops)][q])


def test_prefix_scalar_api():
    """insert / match_prefix one call at a time, as RadixTree (radix.py:31-83)."""
    tree = _tree()
    assert tree.match_prefix([1, 2, 3]) == (0, None)  # test_radix.py:26-27
    tree.insert([1, 2, 3], "a")
    assert tree.match_prefix([]) == (0, None)
    tree.insert([1, 2, 3, 4], "b")
    tree.insert([1, 2], "c")
    assert tree.match_prefix([1, 2, 3, 4, 5]) == (4, "b")
    assert tree.match_prefix([1, 2, 3]) == (3, "a")  # earliest witness at depth 3
    assert tree.match_prefix([1, 2, 9]) == (2, "a")
    assert tree.match_prefix([9]) == (0, None)
    tree.insert([], "empty")
    assert tree.match_prefix([7]) == (0, None)
    tree.check()


def test_prefix_match_insert_sessions():
    """The serve-loop form at scale: 256 agent sessions x 4 turns of 8K-16K tokens
    (shared system header, per-session history growing turn by turn), each
    request matched against every earlier one then inserted (engine.py:170,
    228); checked against the host radix and, for a sample, the brute force."""
    from paper_2605_05696_b200.radix import RadixTree

    rng = np.random.default_rng(12)
    header = rng.integers(0, 2**32, size=2000, dtype=np.uint64).astype(np.uint32)
    hist = [np.concatenate([header, rng.integers(0, 2**32, size=int(rng.integers(6000, 14000)),
                                                 dtype=np.uint64).astype(np.uint32)]) for _ in range(256)]
    reqs = []
    for turn in range(4):
        for s in range(256):
            if turn:
                hist[s] = np.concatenate([hist[s], rng.integers(0, 2**32, size=int(rng.integers(50, 500)),
                                                                dtype=np.uint64).astype(np.uint32)])
            cut = hist[s].size - int(rng.integers(0, 64))  # sometimes an edited tail
            reqs.append(hist[s][:cut].copy())
    tree = _tree(max_prefixes=1 << 23, max_tokens=1 << 24)
    torch.cuda.synchronize()
    ms, ws = [], []
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for t in range(4):  # one batch per turn
        part = reqs[t * 256:(t + 1) * 256]
        ev[0].record()
        m, w = tree.match_insert(part, list(range(t * 256, (t + 1) * 256)))
        ev[1].record()
        ms += m
        ws += w
    torch.cuda.synchronize()
    host = RadixTree()
    for i, r in enumerate(reqs):
        hm, hw = host.match_prefix(r)
        assert (ms[i], ws[i]) == (hm, hw), i
        host.insert(r, i)
    for i in rng.choice(len(reqs), size=24, replace=False):
        bm, bw = O.prefix_match(list(enumerate(reqs[:i])), reqs[i])
        assert (ms[i], ws[i]) == (bm, bw)
    assert sum(m > 0 for m in ms) > 900
    tree.check()
    print(f"K0 match_insert: {sum(r.size for r in reqs[-256:])} tokens in {ev[0].elapsed_time(ev[1]):.3f} ms "
          f"(last batch), {tree.n_prefixes} prefixes stored")


def test_prefix_region_boundaries():
    """The K0 table places the keys of depths 64b + 1 .. 64b + 64 of a sequence in one
    region chosen by its prefix of length 64b, with a region step and then per-key double
    hashing on collisions: 1,800 sequences diverging from a shared trunk at and around the
    region boundaries (and from each other inside blocks, over a 3-letter alphabet), plus
    duplicates and strict prefixes, all match the host radix tree exactly, batch after batch."""
    from paper_2605_05696_b200.radix import RadixTree

    rng = np.random.default_rng(64)
    trunk = rng.integers(0, 2**32, size=5000, dtype=np.uint64).astype(np.uint32)
    cuts = [0, 1, 50, 62, 63, 64, 65, 127, 128, 129, 1023, 1024, 1025, 2048, 4999, 5000]
    reqs = []
    for i in range(1800):
        p = cuts[i % len(cuts)] if i % 3 else int(rng.integers(0, 5000))
        tail = rng.integers(0, 3, size=int(rng.integers(0, 200))).astype(np.uint32)
        r = np.concatenate([trunk[:p], tail])
        if i % 97 == 5 and reqs:  # an exact repeat or a strict prefix of an earlier sequence
            prev = reqs[int(rng.integers(0, len(reqs)))]
            r = prev[:int(rng.integers(0, prev.size + 1))].copy()
        reqs.append(r)
    tree = _tree(max_prefixes=1 << 22, max_tokens=1 << 23)
    host = RadixTree()
    for b0 in range(0, len(reqs), 300):
        part = reqs[b0:b0 + 300]
        m, w = tree.match_insert(part, list(range(b0, b0 + len(part))))
        for k, r in enumerate(part):
            assert (m[k], w[k]) == host.match_prefix(r), b0 + k
            host.insert(r, b0 + k)
    tree.check()


@pytest.mark.parametrize("case", ["long_shared", "small_alphabet"])
def test_prefix_growth_golden(case):
    """Tiny initial capacities: the arena, the per-sequence arrays and the table
    (rebuilt from the arena with the original epochs) grow as batches arrive;
    results still equal the reference RadixTree's."""
    g = load_npz("radix")[case]
    ops = radix_case_inputs(RADIX_CASES[case])
    tree = _tree(max_prefixes=8, max_tokens=64, max_sequences=2)
    got_m, got_w = np.full(len(ops), -1), np.full(len(ops), -1)
    bs = 13
    for b0 in range(0, len(ops), bs):
        part = ops[b0:b0 + bs]
        ins = [o[0] for o in part]
        m, w = tree.run_ops([o[1] for o in part], ins, [not x for x in ins], handles=list(range(b0, b0 + len(part))))
        m, w = m.cpu().numpy(), w.cpu().numpy()
        for k, (is_ins, _) in enumerate(part):
            if not is_ins:
                got_m[b0 + k] = m[k]
                got_w[b0 + k] = tree.handles[w[k]] if m[k] > 0 else -1
    tree.check()
    q = np.array([not o[0] for o in ops])
    assert np.array_equal(got_m[q], g["m"][q]) and np.array_equal(got_w[q], g["witness"][q])
    assert tree.n_slots > 16 and tree.arena.numel() > 64


@pytest.mark.parametrize("case", sorted(RADIX_CASES))
def test_prefix_collisions_answered_exactly(case):
    """With degenerate hash keys (hash_key 1: every prefix of one length collides,
    the worst an adversary could do) every query still gets the reference tree's
    answer: the verification catches each false match and the exact on-device
    scan answers it (a collision must not poison later queries)."""
    g = load_npz("radix")[case]
    ops = radix_case_inputs(RADIX_CASES[case])[:300]
    tree = _tree(hash_key=1)
    for b0 in range(0, len(ops), 37):
        part = ops[b0:b0 + 37]
        ins = [o[0] for o in part]
        m, w = tree.run_ops([o[1] for o in part], ins, [not x for x in ins], handles=list(range(b0, b0 + len(part))))
        m, w = m.cpu().numpy(), w.cpu().numpy()
        for j, (is_ins, _seq) in enumerate(part):
            if not is_ins:
                assert m[j] == g["m"][b0 + j], (case, b0 + j)
                assert (tree.handles[w[j]] if m[j] > 0 else -1) == g["witness"][b0 + j], (case, b0 + j)
    tree.check()  # no error: collisions are resolved, not raised
    assert tree.collisions_resolved or not any(not o[0] for o in ops)


def test_prefix_keyed_hash_differs_per_index():
    a, b = _tree(), _tree()
    assert a.hash_key != b.hash_key
