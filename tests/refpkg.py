"""Locate the reference package `btpsim` for interop tests: the offline install under
baseline/_ref (travels to the GPU box) or, in the build container, /root/reference/pkg/src.
Returns None when neither exists (the tests that need it skip)."""

import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
_CANDIDATES = (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src"))


def load_btpsim():
    for path in _CANDIDATES:
        if (path / "btpsim" / "__init__.py").exists():
            if str(path) not in sys.path:
                sys.path.append(str(path))
            return importlib.import_module("btpsim")
    return None
