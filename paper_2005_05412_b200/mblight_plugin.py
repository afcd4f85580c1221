"""Plug the GPU solver into the reference package (``mblight``) and its CLI.

    python -m paper_2005_05412_b200.mblight_plugin -d ziolkowski1995 -m gpu-fdtd-reg-cayley -w raw -o out/

The reference CLI resolves solver names through its registry
(``mblight.core.create_solver``, core.py:633-641; called at cli.py:389) but
never imports plugins, so this entry point registers ``gpu-fdtd-reg-cayley``
and ``gpu-fdtd-rk4`` into that registry and then hands over to
``mblight.cli.main`` unchanged.  ``cpu-...`` aliases keep mapping to the
reference solvers (cli.py:59-70); any ``gpu-...`` name passes through to the
registry as-is.
"""

from __future__ import annotations

import sys

from .solver import register_with_reference


def main(argv=None) -> int:
    import mblight  # noqa: PLC0415  (the reference package must be importable)
    from mblight import cli  # noqa: PLC0415

    register_with_reference(mblight)
    return cli.main(argv)


if __name__ == "__main__":
    sys.exit(main())
