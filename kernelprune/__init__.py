"""Alias package: `import kernelprune` resolves to paper_2003_06795_b200."""
import importlib
import sys

_real = importlib.import_module("paper_2003_06795_b200")
_MODS = ("errors", "rng", "dataset", "synthetic", "clustering", "decomposition", "pruning",
         "selector_models", "codegen", "report", "cli", "hdbscan")
for _m in _MODS:
    sys.modules[f"{__name__}.{_m}"] = importlib.import_module(f"paper_2003_06795_b200.{_m}")
    globals()[_m] = sys.modules[f"{__name__}.{_m}"]
__version__ = _real.__version__
