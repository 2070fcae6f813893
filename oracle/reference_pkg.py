"""TEST INFRASTRUCTURE ONLY -- import the reference `kernelprune` package.

The reference is pure Python (/root/reference/pkg/src/kernelprune, numpy
only), so it is imported in place (read-only, no bytecode written) under the
alias ``kernelprune_ref`` to generate golden vectors and for differential
tests. /root/reference exists only in the build container: on the GPU box
``load()`` returns None and the differential tests skip; the committed
fixtures in tests/golden/ carry the same evidence there.
"""

from __future__ import annotations

import importlib.util
import os
import sys
from pathlib import Path

REF_SRC = Path(os.environ.get("KERNELPRUNE_REFERENCE_SRC", "/root/reference/pkg/src"))
ALIAS = "kernelprune_ref"


def available() -> bool:
    return (REF_SRC / "kernelprune" / "__init__.py").exists()


def load():
    """The reference package as module `kernelprune_ref`, or None."""
    if ALIAS in sys.modules:
        return sys.modules[ALIAS]
    if not available():
        return None
    sys.dont_write_bytecode = True
    pkg_dir = REF_SRC / "kernelprune"
    spec = importlib.util.spec_from_file_location(
        ALIAS, pkg_dir / "__init__.py", submodule_search_locations=[str(pkg_dir)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules[ALIAS] = mod
    spec.loader.exec_module(mod)
    for name in ("errors", "rng", "dataset", "synthetic", "clustering", "decomposition",
                 "pruning", "selector_models", "codegen", "report", "cli"):
        importlib.import_module(f"{ALIAS}.{name}")
    return mod
