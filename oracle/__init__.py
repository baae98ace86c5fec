"""TEST INFRASTRUCTURE ONLY: the CPU oracle (restated reference algorithm).

Importable by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg
only; the product package never imports it.
"""
