"""The reference's own serve API on a JSONL trace, ours vs the reference.

Generates an agent_meta trace (oracle/workloads.py restates workloads.generate)
as JSONL, then times parse + run_trace (observer mode):
  python tools/serve_compare.py ours [n_req body_len]       # on the B200: model.parse_trace + engine.run_trace
  python tools/serve_compare.py reference [n_req body_len]  # here: irminsul.model / irminsul.engine (CPU)
Prints requests, tokens, seconds, tokens/s and a digest of every request's
events (start, len, class, fp, delta) so the two runs can be compared.
"""
import hashlib
import io
import sys
import time

sys.path.insert(0, ".")
from oracle import workloads as W  # noqa: E402  (generator only: the trace content)


def trace_text(n_req, body_len):
    reqs = W.generate("agent_meta", n_req=n_req, body_len=body_len, seed=7)
    import json

    lines = []
    for i, r in enumerate(reqs):
        lines.append(json.dumps({"session_id": f"s{i % 8}", "turn": i // 8, "segments": [
            {"kind": k, "tokens": list(t), "shared_id": sid} for k, t, sid in r]}, separators=(", ", ": ")))
    return "\n".join(lines) + "\n"


def digest(results):
    h = hashlib.sha256()
    for r in results:
        for e in r.events:
            h.update(f"{e.start},{e.length},{e.klass.value if hasattr(e.klass, 'value') else e.klass},"
                     f"{getattr(e, 'fingerprint', None)},{getattr(e, 'delta', None)};".encode())
        h.update(b"|")
    return h.hexdigest()[:16]


def main():
    which = sys.argv[1]
    n_req = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    body = int(sys.argv[3]) if len(sys.argv) > 3 else 16000
    text = trace_text(n_req, body)
    if which == "ours":
        import torch

        from paper_2605_05696_b200 import engine, model

        engine.run_trace(engine.EngineState(engine.ServeConfig()), model.parse_trace(io.StringIO(trace_text(4, 500))))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tr = model.parse_trace(io.StringIO(text))
        res, _ = engine.run_trace(engine.EngineState(engine.ServeConfig()), tr)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    else:
        sys.path.insert(0, "/root/reference/pkg/src")
        from irminsul import engine, model

        t0 = time.perf_counter()
        tr = model.parse_trace(io.StringIO(text))
        res, _ = engine.run_trace(engine.EngineState(engine.ServeConfig()), tr)
        dt = time.perf_counter() - t0
    n_tok = sum(r.num_tokens for r in res)
    print(f"{which}: {len(res)} requests, {n_tok} tokens, {dt:.3f} s, {n_tok / dt / 1e6:.3f} M tok/s, "
          f"events digest {digest(res)}")


if __name__ == "__main__":
    main()
