"""TEST INFRASTRUCTURE ONLY -- restated workload generators and a sequential
observer-mode serve loop, so the GPU box can regenerate the golden traces and
check hit sets / deltas without /root/reference.

Restates (reference = /root/reference/pkg/src/irminsul):
  workloads._gen_agent_meta/_sysvar/_compact/_rerank/_tool_variants
                                        workloads.py:67-195
  engine.serve (observer mode, S1 off) engine.py:158-238
  radix.RadixTree.match_prefix         radix.py:61-89 (as a brute-force LCP)
Requests are plain lists of (kind, tokens tuple, shared_id) segments.
"""

from __future__ import annotations

import numpy as np

try:  # package-relative when imported as oracle.workloads
    from . import oracle as O
except ImportError:  # pragma: no cover - imported with oracle/ on sys.path
    import oracle as O

MARKER_LEN = 64
_POOL_LABEL = 0x504F4F4C
_REQ_LABEL = 0x524551


def _rng(seed: int, *labels: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(O.derive_seed(seed, *labels)))


def _tokens(rng, n: int) -> tuple[int, ...]:
    return tuple(int(t) for t in rng.integers(0, 2**32, size=n, dtype=np.uint64))


def _marker():
    return ("marker", O.canonical_marker(), None)


def _strip(markers: bool, segs):
    return segs if markers else [s for s in segs if s[0] != "marker"]


def generate(pattern: str, n_req: int = 80, body_len: int = 2500, header_len: int = 50,
             variant_pool: int = 8, seed: int = 0, markers: bool = True):
    """Returns a list of requests; each request is a list of segments."""
    reqs = []
    if pattern == "agent_meta":
        shared = _rng(seed, _POOL_LABEL, 0)
        header = _tokens(shared, header_len)
        body = _tokens(shared, body_len)
        for i in range(n_req):
            rng = _rng(seed, _REQ_LABEL, i)
            meta_len = int(rng.integers(30, 71))
            reqs.append(_strip(markers, [("system", header, "agent_header"),
                                         ("header", _tokens(rng, meta_len), None), _marker(),
                                         ("body", body, "agent_body")]))
    elif pattern == "sysvar":
        shared = _rng(seed, _POOL_LABEL, 1)
        prefix = _tokens(shared, 1700 + header_len)
        tail = _tokens(shared, 750)
        variants = [_tokens(shared, 8) for _ in range(variant_pool)]
        for i in range(n_req):
            rng = _rng(seed, _REQ_LABEL, i)
            variant = variants[int(rng.integers(variant_pool))]
            slot = variant + _tokens(rng, 32)
            reqs.append(_strip(markers, [("system", prefix, "sysvar_prefix"), ("tool", slot, None),
                                         _marker(), ("body", tail, "sysvar_tail")]))
    elif pattern == "compact":
        rng = _rng(seed, _POOL_LABEL, 2)
        append_len = max(body_len // 25, MARKER_LEN)
        content = list(_tokens(rng, body_len))
        compaction_turn = n_req // 2
        for i in range(n_req):
            if i > 0:
                if i == compaction_turn:
                    content = content[len(content) // 10:]
                content = content + list(_tokens(rng, append_len))
            reqs.append([("history", tuple(content), None)])
    elif pattern == "rerank":
        shared = _rng(seed, _POOL_LABEL, 3)
        prefix = _tokens(shared, 500)
        docs = [_tokens(shared, 256) for _ in range(8)]
        order = list(range(8))
        for i in range(n_req):
            rng = _rng(seed, _REQ_LABEL, i)
            if i > 0 and rng.random() < 0.12:
                j = int(rng.integers(8 - 3, 8 - 1))
                order[j], order[j + 1] = order[j + 1], order[j]
            segs = [("system", prefix, "rerank_prefix")]
            for j in order:
                segs.append(_marker())
                segs.append(("doc", docs[j], f"doc{j}"))
            reqs.append(_strip(markers, segs))
    elif pattern == "tool_variants":
        shared = _rng(seed, _POOL_LABEL, 4)
        prefix = _tokens(shared, 2000)
        tail = _tokens(shared, 500)
        schemas = [_tokens(shared, 100) for _ in range(variant_pool)]
        for i in range(n_req):
            rng = _rng(seed, _REQ_LABEL, i)
            schema = schemas[int(rng.integers(variant_pool))]
            reqs.append(_strip(markers, [("system", prefix, "tool_prefix"), ("tool", schema, None),
                                         _marker(), ("body", tail, "tool_tail")]))
    else:
        raise ValueError(pattern)
    return reqs


def flatten(req) -> tuple[int, ...]:
    out: list[int] = []
    for _, toks, _ in req:
        out.extend(toks)
    return tuple(out)


def marker_spans(req) -> list[tuple[int, int]]:
    spans, pos = [], 0
    for kind, toks, _ in req:
        if kind == "marker":
            spans.append((pos, pos + len(toks)))
        pos += len(toks)
    return spans


KLASS = ("prefix_hit", "pic_hit", "s1_hit", "carveout_prefill", "novel_prefill")


def serve_trace(reqs, k: int = 7, min_size: int = 32, max_size: int = 512, carve: int = 32,
                s1: bool = False, window: int = 128):
    """Sequential observer-mode serve (engine.py:158-238); returns events
    (req, start, len, klass, fp, delta). ``s1``: the sub-window fallback
    (engine.py:116-139, 211-226): a missed chunk's aligned full windows are
    probed against the fingerprints of every earlier novel chunk's windows."""
    seen: list[np.ndarray] = []
    registry: dict[int, int] = {}  # fp -> p_src
    subwindows: set[int] = set()
    events = []
    for ri, req in enumerate(reqs):
        flat = flatten(req)
        arr = np.asarray(flat, dtype=np.uint64)
        m = 0
        for prev in seen:  # brute-force longest common prefix
            n = min(prev.size, arr.size)
            neq = np.nonzero(prev[:n] != arr[:n])[0]
            m = max(m, int(neq[0]) if neq.size else n)
        if m > 0:
            events.append((ri, 0, m, 0, -1, None))
        tail = flat[m:]
        pins = O.marker_pin_offsets((max(s - m, 0), e - m) for s, e in marker_spans(req) if e - 1 >= m)
        st, ln, fp, _ = O.cdc_chunk(tail, k, min_size, max_size, pins) if tail else ([], [], [], [])
        for s, l, f in zip(st, ln, fp):
            p, l, f = m + int(s), int(l), int(f)
            if p < carve:
                carved = min(carve - p, l)
                events.append((ri, p, carved, 3, -1, None))
                if l > carved:
                    events.append((ri, p + carved, l - carved, 4, -1, None))
                continue
            if f in registry:
                events.append((ri, p, l, 1, f, p - registry[f]))
                continue
            novel = [(p, l)]
            if s1:
                chunk = tail[p - m:p - m + l]
                wins = [(o, O.fingerprint(chunk[o:o + window])) for o in range(0, l - window + 1, window)]
                hits = [(p + o, wf) for o, wf in wins if wf in subwindows]
                for hs, wf in hits:
                    events.append((ri, hs, window, 2, wf, None))
                novel, pos = [], p
                for hs, _ in hits:  # _subtract_spans (engine.py:211-226)
                    if hs > pos:
                        novel.append((pos, hs - pos))
                    pos = hs + window
                if pos < p + l:
                    novel.append((pos, p + l - pos))
                subwindows.update(wf for _, wf in wins)
            for s_, l_ in novel:
                events.append((ri, s_, l_, 4, -1, None))
            registry[f] = p
        seen.append(arr)
    return events, len(registry)
