"""The reference package ``mblight``: the setup API this GPU solver plugs into.

The device / scenario / quantum-description objects, the error classes, the
physical constants, the grid sizing, the per-material coefficients, the
relaxation propagator and the stepper constants are all the reference's own
(``mblight``, ``pkg/src/mblight``); this package only adds the GPU solver
behind its solver registry (``core.py:617-641``).

Lookup order: an importable ``mblight`` (installed next to this package, the
normal drop-in situation), else the pinned copy installed into
``<repo>/baseline/_ref`` (``python -m pip install --no-index --no-deps
--target baseline/_ref <reference>/pkg``; ``__graft_entry__.build()`` does
this when the reference sources are mounted).  ``baseline/_ref`` travels with
the repository snapshot to the GPU box, so the box runs the reference's setup
code unmodified, numba included.
"""

from __future__ import annotations

import os
import sys
from importlib import import_module
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
PINNED = REPO / "baseline" / "_ref"


def _load():
    # the reference's numba loops cache their compiled code next to the
    # sources (@njit(cache=True)); keep that cache out of the snapshot
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    try:
        return import_module("mblight")
    except ImportError:
        pass
    if (PINNED / "mblight" / "__init__.py").exists():
        sys.path.insert(0, str(PINNED))
        return import_module("mblight")
    raise ImportError(
        "the reference package mblight is not importable: install it, or run "
        "__graft_entry__.build() with the reference mounted (installs it into baseline/_ref)")


mblight = _load()
core = import_module("mblight.core")
quantum = import_module("mblight.quantum")
solver_fdtd = import_module("mblight.solver_fdtd")
kernels = import_module("mblight._kernels")
