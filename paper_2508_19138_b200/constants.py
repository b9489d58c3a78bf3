"""Physical prefactors of the energy convolutions (negfgw/constants.py:16-31).

Natural units, hbar = e = 1, energies in eV."""

from __future__ import annotations

import math

KT_DEFAULT = 0.02585
#: P(E) = C_POLARIZATION * sum_E' G(E') G(E'-E) dE   (constants.py:24)
C_POLARIZATION = -1j / (2.0 * math.pi)
#: Sigma(E) = C_SIGMA * sum_E' G(E-E') W(E') dE    (constants.py:27)
C_SIGMA = 1j / (2.0 * math.pi)
#: per-sample weight of observable integrals   (constants.py:31)
C_OBSERVABLE = 1.0 / (2.0 * math.pi)
