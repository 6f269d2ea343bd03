"""Test-only helpers: tiny feasible instances and comparison utilities."""
from __future__ import annotations

import json
import os

import numpy as np

from gen.problems import make_unicycle, make_quad, make_franka

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def tiny(kind="uni", T=3, seed=0, r_trust=None, **kw):
    if kind == "uni":
        shape, data = make_unicycle(90, seed, T=T, **kw)
    elif kind == "quad":
        shape, data = make_quad(91, seed, T=T, n_obs=kw.pop("n_obs", 1), **kw)
    else:
        shape, data = make_franka(92, seed, T=T, **kw)
    if r_trust is not None:
        data["r_trust"] = float(r_trust)
    return shape, data


def make_feasible(pb, data, rng, lo=0.02, hi=0.3, scale_bhat=1.0):
    """Rewrite g0 so that (du, k_v, p) = (0, 0, ||b_hat||+) is strictly feasible.

    Used only to build barrier-IP pin instances (feasibility at the start).
    """
    g = -(scale_bhat * np.linalg.norm(pb.bhat, axis=1) + rng.uniform(lo, hi, pb.ng))
    data = dict(data)
    data["g0"] = g
    return data


def relerr(a, b):
    a = np.asarray(a, float); b = np.asarray(b, float)
    d = np.linalg.norm(a - b)
    n = max(np.linalg.norm(b), 1e-300)
    return d / n


def ragged_from_dense(shape, nx, M):
    """Take each cone's ragged support out of a dense [n_g, (T+1) n_x] array."""
    rows = []
    for j in range(shape.n_g):
        k = int(shape.cone_knot[j])
        if shape.cone_kind[j] == 0:
            rows.append(M[j, :(k + 1) * nx])
        else:
            rows.append(M[j, k * nx:(k + 1) * nx])
    return np.concatenate(rows)


def close(x, ref, scale=0.0, tol=1e-9):
    """Normwise parity: ||x - ref|| <= tol (||ref|| + scale).

    `scale` is the norm of the operands an accumulator is built from (e.g.
    ||nu|| for lam_nu = sum(a - nu)), so cancellation does not turn
    round-off into a relative failure (SURVEY §8c parity protocol)."""
    x = np.asarray(x, float); ref = np.asarray(ref, float)
    return np.linalg.norm(x - ref) <= tol * (np.linalg.norm(ref) + scale) + 1e-300


def elementwise(x, ref, floor_frac=1e-3):
    """Element-wise parity metric: max_i |x_i - ref_i| / (|ref_i| + f ||ref||_inf).

    Complements `close` (normwise): an error confined to a small subset of the
    entries (e.g. the control-cone part of nu) is visible here even when it is
    invisible in the norm of the whole array.  The floor f ||ref||_inf keeps
    entries that are zero up to round-off (cancellation) from dividing by ~0."""
    x = np.asarray(x, float).ravel(); ref = np.asarray(ref, float).ravel()
    if ref.size == 0:
        return 0.0
    den = np.abs(ref) + floor_frac * max(np.max(np.abs(ref)), 1e-300)
    return float(np.max(np.abs(x - ref) / den))
