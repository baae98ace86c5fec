"""Loading the committed golden fixtures (tests/golden/*.npz), made by make_golden.py."""

import os

import numpy as np

GOLDEN = os.path.dirname(os.path.abspath(__file__))


def load_npz(name: str) -> dict[str, dict[str, np.ndarray]]:
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    out: dict[str, dict[str, np.ndarray]] = {}
    for key in z.files:
        case, field = key.split("/", 1)
        out.setdefault(case, {})[field] = z[key]
    return out
