"""Alias: the reference's test-suite imports `meshreg`; give it this package."""
import importlib
import sys

import paper_1411_2141_b200 as _p

sys.modules[__name__] = _p
for _s in ("solver", "image", "mesh", "densefield", "baseline", "cli", "delaunay", "meshgen",
           "meshio", "synthetic"):
    try:
        sys.modules[f"meshreg.{_s}"] = importlib.import_module(f"paper_1411_2141_b200.{_s}")
    except ImportError:
        pass
