"""GPU parity: the batched serve path reproduces the reference's events
(hit sets, deltas, fingerprints, counts) on the golden traces, bit-exact, and
live mode passes / trips the rotation check like engine.py:142-155."""

import numpy as np
import pytest

from inputs import TRACE_CASES, custom_trace
from oracle import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    from paper_2605_05696_b200 import chunking, engine, model, rotary

    return engine, model, chunking, rotary


def to_requests(model, reqs):
    return [model.Request(f"s{i}", 0, tuple(model.Segment(k, tuple(t), sid) for k, t, sid in r))
            for i, r in enumerate(reqs)]


@pytest.mark.parametrize("batch", [1, 4])
@pytest.mark.parametrize("name", sorted(TRACE_CASES))
def test_trace_events_golden(E, name, batch, golden_traces):
    engine, model, chunking, _ = E
    case = dict(TRACE_CASES[name])
    k = case.pop("k", 7)
    s1, window = case.pop("s1", False), case.pop("window", 128)
    reqs = to_requests(model, custom_trace(TRACE_CASES[name]) if "custom" in case else W.generate(**case))
    cfg = engine.ServeConfig(chunker=chunking.ChunkerParams(mask_exponent=k), s1_enabled=s1, s1_window=window)
    state = engine.EngineState(cfg)
    results, _ = engine.run_trace(state, model.Trace(tuple(reqs)), batch=batch)
    g = golden_traces[name]
    ev = [(ri, e.start, e.length, list(engine.ServiceClass).index(e.klass), e.fingerprint, e.delta)
          for ri, r in enumerate(results) for e in r.events]
    assert len(ev) == g["req"].size
    for i, (ri, s, l, kl, fp, d) in enumerate(ev):
        assert (ri, s, l, kl) == (g["req"][i], g["start"][i], g["length"][i], g["klass"][i]), i
        want_fp = None if int(g["fp"][i]) == 2**64 - 1 else int(g["fp"][i])  # -1 encodes None
        assert fp == want_fp, i
        if g["has_delta"][i]:
            assert d == int(g["delta"][i])
        else:
            assert d is None
    counts = np.array([[r.counts[k] for k in engine.ServiceClass] for r in results])
    assert np.array_equal(counts, g["counts"])
    assert len(state.registry) == int(g["registry_len"][0])
    assert state.registry.pool_bytes() == int(g["pool_bytes"][0])


def _marker_trace(model, chunking):
    rng = np.random.default_rng(85)
    marker = chunking.canonical_marker()
    body = tuple(int(t) for t in rng.integers(0, 2**32, size=1200, dtype=np.uint64))
    reqs = []
    for i in range(8):
        hdr = tuple(int(t) for t in np.random.default_rng(200 + i).integers(0, 2**32, size=40 + 7 * i, dtype=np.uint64))
        reqs.append(model.Request(f"s{i}", 0, (model.Segment("header", hdr), model.Segment("marker", marker),
                                                model.Segment("body", body))))
    return model.Trace(tuple(reqs))


@pytest.mark.parametrize("precision", ["f64", "f32", "bf16e"])
def test_live_equals_observer(E, precision):
    engine, model, chunking, rotary = E
    trace = _marker_trace(model, chunking)
    obs, _ = engine.run_trace(engine.EngineState(engine.ServeConfig()), trace)
    live_state = engine.EngineState(engine.ServeConfig(mode=engine.Mode.LIVE, precision=rotary.Precision(precision)))
    live, _ = engine.run_trace(live_state, trace)
    for a, b, r in zip(obs, live, trace.requests):
        assert a.counts == b.counts and a.events == b.events
        assert b.live_rows == r.num_tokens
    assert sum(r.rotation_multiplies for r in live) > 0


def test_live_tripwire_wrong_theta(E):
    engine, model, chunking, rotary = E
    trace = _marker_trace(model, chunking)
    state = engine.EngineState(engine.ServeConfig(mode=engine.Mode.LIVE))
    state.registry.spec = rotary.make_spec(3.2e7)
    with pytest.raises(engine.LiveVerificationError):
        engine.run_trace(state, trace)


def test_serve_basics(E):
    engine, model, chunking, _ = E
    rng = np.random.default_rng(0)
    toks = tuple(int(t) for t in rng.integers(0, 2**32, size=500, dtype=np.uint64))
    state = engine.EngineState(engine.ServeConfig())
    r = engine.serve(state, model.Request("a", 0, (model.Segment("body", toks),)))
    assert r.counts[engine.ServiceClass.CARVEOUT_PREFILL] == 32
    assert r.counts[engine.ServiceClass.NOVEL_PREFILL] == 468
    r2 = engine.serve(state, model.Request("b", 0, (model.Segment("body", toks),)))
    assert r2.tprefix == 1.0
    with pytest.raises(ValueError):
        engine.serve(state, model.Request("c", 0, ()))


def test_s1_recovery(E):
    engine, model, chunking, _ = E
    rng = np.random.default_rng(95)
    t = lambda n: tuple(int(x) for x in rng.integers(0, 2**32, size=n, dtype=np.uint64))
    content = t(1024)
    cfg = engine.ServeConfig(s1_enabled=True, chunker=chunking.ChunkerParams(mask_exponent=20))
    state = engine.EngineState(cfg)
    engine.serve(state, model.Request("a", 0, (model.Segment("body", content),)))
    shifted = t(512) + content[640:1024] + t(128)
    res = engine.serve(state, model.Request("b", 0, (model.Segment("body", shifted),)))
    assert res.counts[engine.ServiceClass.S1_HIT] == 384
    assert res.counts[engine.ServiceClass.PIC_HIT] == 0
