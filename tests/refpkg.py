"""Import the unmodified reference package (`convbench`) for integration tests.

Search order: baseline/_ref (the pip --target install, git-ignored; it travels to the GPU
box with the repo snapshot), then -- CPU tests in the build container only --
/root/reference/pkg/src.  GPU tests pass allow_source=False: nothing on the GPU box may
read /root/reference."""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CANDIDATES = [ROOT / "baseline" / "_ref"]
SOURCE = Path("/root/reference/pkg/src")


def reference(allow_source: bool = True):
    """The reference `convbench` package, or None when it is not installed here."""
    paths = CANDIDATES + ([SOURCE] if allow_source else [])
    for p in paths:
        if (p / "convbench" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.append(str(p))
            mod = importlib.import_module("convbench")
            for sub in ("harness", "algos", "cli", "report", "timing", "descriptor", "tensor"):
                importlib.import_module(f"convbench.{sub}")
            return mod
    return None
