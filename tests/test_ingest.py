"""CPU: native trace ingest (csrc/ingest.cpp, model.load_trace_arrays /
parse_trace) against the reference's own parse_trace outputs and errors
(tests/golden/ingest.json, made by make_golden.py from model.py:80-166).

Checked: flattened tokens, segment offsets, marker spans, sessions, turns,
kinds and shared ids of every request; byte-exact serialize(parse(text)) round
trips (test_model.py:57-63); the exception class, line number, field and
message of every malformed record (test_model.py:109-153; for invalid JSON the
message is Python json's own text, so only its prefix is compared); and
universal newlines when the trace is read from a file."""

import io
import json
import os

import numpy as np
import pytest

from goldens import GOLDEN

from paper_2605_05696_b200 import model as M

FX = json.load(open(os.path.join(GOLDEN, "ingest.json")))


@pytest.mark.parametrize("name", sorted(FX["good"]))
def test_parse_trace_golden(name):
    g = FX["good"][name]
    trace = M.parse_trace(io.StringIO(g["text"]))
    assert [list(M.flatten(r)[0]) for r in trace.requests] == g["tokens"]
    assert [M.flatten(r)[1] for r in trace.requests] == g["offsets"]
    assert [[list(s) for s in M.marker_spans(r)] for r in trace.requests] == g["markers"]
    assert [r.session_id for r in trace.requests] == g["sessions"]
    assert [r.turn_index for r in trace.requests] == g["turns"]
    assert [[s.kind for s in r.segments] for r in trace.requests] == g["kinds"]
    assert [[s.shared_id for s in r.segments] for r in trace.requests] == g["shared"]
    if not g["text"].startswith("\n"):
        assert M.serialize_trace(trace) == g["text"]  # round trip, byte-exact


@pytest.mark.parametrize("name", sorted(FX["good"]))
def test_trace_arrays_golden(name, tmp_path):
    g = FX["good"][name]
    ta = M.load_trace_arrays(text=g["text"], pinned=False)
    assert ta.n_requests == len(g["tokens"])
    for i, want in enumerate(g["tokens"]):
        got = ta.tokens[ta.req_tok_off[i]:ta.req_tok_off[i + 1]]
        assert got.dtype == np.uint32 and got.tolist() == want
    off, spans = ta.marker_pins()
    for i, want in enumerate(g["markers"]):
        assert spans[off[i]:off[i + 1]].tolist() == want
    # the same file with CRLF line ends, read the way open() reads text files
    p = tmp_path / "t.jsonl"
    p.write_bytes(g["text"].replace("\n", "\r\n").encode())
    tb = M.load_trace_arrays(path=str(p), pinned=False)
    assert np.array_equal(tb.tokens, ta.tokens) and np.array_equal(tb.req_tok_off, ta.req_tok_off)
    assert tb.sessions == ta.sessions and tb.turns.tolist() == ta.turns.tolist()
    p.write_bytes(g["text"].replace("\n", "\r").encode())  # old-Mac line ends: universal newlines too
    tc = M.load_trace_arrays(path=str(p), pinned=False)
    assert np.array_equal(tc.tokens, ta.tokens) and tc.sessions == ta.sessions


@pytest.mark.parametrize("name", sorted(FX["bad"]))
def test_trace_errors_golden(name):
    b = FX["bad"][name]
    if b["error"] is None:
        M.parse_trace(io.StringIO(b["text"]))
        return
    with pytest.raises(ValueError) as exc:
        M.parse_trace(io.StringIO(b["text"]))
    if b["error"] == "TraceFormatError":
        assert isinstance(exc.value, M.TraceFormatError)
        assert (exc.value.line_no, exc.value.field) == (b["line"], b["field"])
        if "invalid JSON" in b["message"]:
            assert str(exc.value).startswith(f"line {b['line']}, field '<line>': invalid JSON:")
        else:
            assert str(exc.value) == b["message"]
    else:
        assert not isinstance(exc.value, M.TraceFormatError) and str(exc.value) == b["message"]


def test_parse_trace_empty_and_blank():
    assert M.parse_trace(io.StringIO("")) == M.Trace(())  # test_model.py:41-42
    assert M.parse_trace(io.StringIO("\n  \n\t\n")) == M.Trace(())


def test_stringio_keeps_lone_cr_inside_a_line():
    """io.StringIO splits on '\\n' only: a lone '\\r' is JSON whitespace inside the line."""
    line = '{"session_id": "a",\r "turn": 0, "segments": []}\n'
    assert M.parse_trace(io.StringIO(line)).requests[0].session_id == "a"
