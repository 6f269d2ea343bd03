"""Closed-form Euclidean projection onto the second-order cone.

PAPER.md SM §II-C, Eq.(18) and Fig.3:

    K_soc = {(t, eta) : ||eta||_2 <= t},   r = (r^t, r^eta),  a = ||r^eta||_2
    Pi(r) = (r^t, r^eta)                              if a <= r^t
          = (0, 0)                                    if a <= -r^t
          = ((r^t + a)/2, (r^t + a)/(2a) r^eta)       otherwise

Cases are tested in exactly this order (R13): at a = 0 a point with
t >= 0 is kept and t < 0 maps to the origin, so case 3 never divides by 0.
Pinned by tests/test_oracle_soc.py (worked examples S:260-262, brute force,
Moreau decomposition, idempotence, membership, non-expansiveness).
"""
from __future__ import annotations

import numpy as np


def proj_soc(t: float, y: np.ndarray):
    """Project one point (t, y) onto {||y|| <= t}; returns (t', y')."""
    y = np.asarray(y, float)
    a = float(np.sqrt(np.dot(y, y)))
    if a <= t:
        return float(t), y.copy()
    if a <= -t:
        return 0.0, np.zeros_like(y)
    c = 0.5 * (t + a)
    return c, (c / a) * y


def proj_soc_scale(t: np.ndarray, a: np.ndarray):
    """Vectorised case logic on (t_j, a_j = ||y_j||) for many cones.

    Returns (t'_j, s_j, case_j) with y'_j = s_j * y_j and case in {1, 2, 3}.
    """
    t = np.asarray(t, float)
    a = np.asarray(a, float)
    tp = np.empty_like(t)
    s = np.empty_like(t)
    case = np.empty(t.shape, np.int8)
    c1 = a <= t
    c2 = (~c1) & (a <= -t)
    c3 = ~(c1 | c2)
    tp[c1] = t[c1]; s[c1] = 1.0; case[c1] = 1
    tp[c2] = 0.0; s[c2] = 0.0; case[c2] = 2
    h = 0.5 * (t[c3] + a[c3])
    tp[c3] = h; s[c3] = h / a[c3]; case[c3] = 3
    return tp, s, case
