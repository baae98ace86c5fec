"""Experiment (not a bench line): the config-2 overlapped step with parts of the next wave's
front replaced, to see what the front costs K4.  python tools/exp_front.py <mode> [bench args]
  mode normal | nok0 (phase 1 replaced by m = HEADER, the value it finds on this workload)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_05696_b200 import radix  # noqa: E402

mode = sys.argv.pop(1)
if mode == "nok0":
    def _skip(self, tok, off, R, m, wit_out=None):
        m.fill_(bench.HEADER)
    radix.WavePrefixIndex.match_insert_wave = _skip
bench.main()
