"""TEST INFRASTRUCTURE ONLY -- the reference's own hot-path test files, run
unmodified against the B200 drop-in (VERDICT r1 "next round" item 2).

The test_*.py files here and _support/{analyzer,roc,workloads}.py plus
_support/data/* are verbatim copies of /root/reference/pkg/tests/*.py and
/root/reference/pkg/src/irminsul/{analyzer,roc,workloads}.py and data/ (see
README.md). This conftest makes ``import irminsul.X`` resolve to the drop-in:

  irminsul.{chunking, fingerprint, rotary, registry, engine, radix, model, rng}
      -> paper_2605_05696_b200.X  (the product: C-ABI library + CUDA kernels)
  irminsul.{analyzer, roc, workloads}
      -> the vendored reference modules (not on the hot path); their
         relative imports land on the drop-in modules above
  irminsul.data -> the vendored reference data files (importlib.resources)

Every test collected here is marked ``gpu``: the drop-in has no CPU fallback.
The product package never imports anything from tests/.
"""

from __future__ import annotations

import importlib
import importlib.util
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SUPPORT = os.path.join(HERE, "_support")
ROOT = os.path.dirname(os.path.dirname(HERE))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

DROP_IN = ("chunking", "fingerprint", "rotary", "registry", "engine", "radix", "model", "rng")
VENDORED = ("workloads", "analyzer", "roc")  # import order: analyzer / workloads need the drop-in only


def _alias():
    if getattr(sys.modules.get("irminsul"), "__irminsul_drop_in__", False):
        return
    pkg = importlib.import_module("paper_2605_05696_b200")
    alias = importlib.util.module_from_spec(importlib.machinery.ModuleSpec("irminsul", None, is_package=True))
    alias.__path__ = []  # nothing is found on disk: every submodule is registered below
    alias.__irminsul_drop_in__ = True
    alias.__doc__ = pkg.__doc__
    sys.modules["irminsul"] = alias
    for name in DROP_IN:
        mod = importlib.import_module(f"paper_2605_05696_b200.{name}")
        sys.modules[f"irminsul.{name}"] = mod
        setattr(alias, name, mod)
    # irminsul.data: a package whose files are the reference's data files
    spec = importlib.util.spec_from_file_location("irminsul.data", os.path.join(SUPPORT, "data", "__init__.py"),
                                                  submodule_search_locations=[os.path.join(SUPPORT, "data")])
    data = importlib.util.module_from_spec(spec)
    sys.modules["irminsul.data"] = data
    spec.loader.exec_module(data)
    alias.data = data
    for name in VENDORED:
        spec = importlib.util.spec_from_file_location(f"irminsul.{name}", os.path.join(SUPPORT, f"{name}.py"))
        mod = importlib.util.module_from_spec(spec)
        sys.modules[f"irminsul.{name}"] = mod
        spec.loader.exec_module(mod)
        setattr(alias, name, mod)


_alias()


def pytest_collection_modifyitems(config, items):
    for item in items:
        if str(item.fspath).startswith(HERE):
            item.add_marker(pytest.mark.gpu)
