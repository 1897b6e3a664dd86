"""Locate the reference package ``probestream`` for side-by-side tests.

Search order: ``$PROBESTREAM_REF``, the driver's offline install
``baseline/_ref`` (git-ignored; travels to the GPU box with the snapshot),
then the read-only source tree ``/root/reference/pkg/src`` (this container
only).  Returns None when none is importable."""

from __future__ import annotations

import importlib
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def candidates():
    env = os.environ.get("PROBESTREAM_REF")
    if env:
        yield Path(env)
    yield ROOT / "baseline" / "_ref"
    yield Path("/root/reference/pkg/src")


def load():
    """The reference ``probestream`` package, or None."""
    if "probestream" in sys.modules:
        return sys.modules["probestream"]
    for c in candidates():
        if (c / "probestream" / "__init__.py").exists():
            sys.path.insert(0, str(c))
            try:
                return importlib.import_module("probestream")
            except Exception:  # pragma: no cover - broken install
                sys.path.remove(str(c))
    return None
