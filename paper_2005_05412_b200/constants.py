"""SI constants (CODATA 2018) used by the Maxwell-Bloch setup.

Values are the ones the reference fixes in
``mblight/constants.py:5-10``; the derived ``EPS0`` is formed the same way
(1 / (mu0 c0^2)) so every coefficient computed from it is bit-identical.
"""

import math

HBAR = 1.054571817e-34
PLANCK = 2.0 * math.pi * HBAR
E0 = 1.602176634e-19
C0 = 299792458.0
MU0 = 1.25663706212e-6
EPS0 = 1.0 / (MU0 * C0 * C0)
