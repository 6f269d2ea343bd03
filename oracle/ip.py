"""Brute-force log-barrier interior point for Problem 2.

    min  sum_k (u_hat_k + du_k)^T R_u (u_hat_k + du_k) + 1/2 k_v^T Q_v k_v
    s.t. g_j + b_j^T du + p_j <= 0               (g^lin,1, reading R1)
         ||A_hat_j k_v + b_hat_j|| <= p_j        j = 1..n_g
         ||F_u du|| <= r_trust

on the dense matrices of oracle.dense.DenseProblem.  Newton's method on
t*f + barrier with feasibility-preserving backtracking, t <- 10 t until the
duality-gap bound m/t < 1e-14 (Boyd & Vandenberghe §11.3).  Tiny instances
only; used as an independent whole-loop pin (SURVEY §8c "Whole loop").
"""
from __future__ import annotations

import numpy as np


def solve_problem2(pb, z0=None, t0=1.0, mu=10.0, gap=1e-14, max_newton=200):
    NU, NK, ng = pb.NU, pb.NK, pb.ng
    n = NU + NK + ng
    Ru2 = 2.0 * pb.Ru
    FtF = pb.F_u.T @ pb.F_u
    r2 = pb.r_trust ** 2

    def split(z):
        return z[:NU], z[NU:NU + NK], z[NU + NK:]

    def feasible(z):
        du, kv, p = split(z)
        if np.any(pb.g0 + pb.b @ du + p >= 0):
            return False
        for j in range(ng):
            y = pb.Ahat[j] @ kv + pb.bhat[j]
            if p[j] <= 0 or p[j] * p[j] - y @ y <= 0:
                return False
        return r2 - du @ FtF @ du > 0

    def phi(z, t):
        du, kv, p = split(z)
        u = pb.u_hat + du
        val = t * (u @ pb.Ru @ u + 0.5 * kv @ pb.Qv @ kv)
        g = np.zeros(n)
        H = np.zeros((n, n))
        g[:NU] = t * Ru2 @ u
        g[NU:NU + NK] = t * pb.Qv @ kv
        H[:NU, :NU] = t * Ru2
        H[NU:NU + NK, NU:NU + NK] = t * pb.Qv
        for j in range(ng):
            l = pb.g0[j] + pb.b[j] @ du + p[j]
            dl = np.zeros(n); dl[:NU] = pb.b[j]; dl[NU + NK + j] = 1.0
            val -= np.log(-l)
            g += dl / (-l)
            H += np.outer(dl, dl) / (l * l)
            y = pb.Ahat[j] @ kv + pb.bhat[j]
            s = p[j] * p[j] - y @ y
            ds = np.zeros(n); ds[NU:NU + NK] = -2.0 * pb.Ahat[j].T @ y; ds[NU + NK + j] = 2.0 * p[j]
            Hs = np.zeros((n, n))
            Hs[NU:NU + NK, NU:NU + NK] = -2.0 * pb.Ahat[j].T @ pb.Ahat[j]
            Hs[NU + NK + j, NU + NK + j] = 2.0
            val -= np.log(s)
            g -= ds / s
            H += np.outer(ds, ds) / (s * s) - Hs / s
        s = r2 - du @ FtF @ du
        ds = np.zeros(n); ds[:NU] = -2.0 * FtF @ du
        Hs = np.zeros((n, n)); Hs[:NU, :NU] = -2.0 * FtF
        val -= np.log(s)
        g -= ds / s
        H += np.outer(ds, ds) / (s * s) - Hs / s
        return val, g, H

    if z0 is None:
        z0 = np.zeros(n)
        for j in range(ng):
            z0[NU + NK + j] = 0.5 * (np.linalg.norm(pb.bhat[j]) - pb.g0[j])  # between the SOC and the row
    z = z0.copy()
    if not feasible(z):
        raise ValueError("barrier start point is not strictly feasible")
    m = 2 * ng + 1
    t = t0
    while True:
        for _ in range(max_newton):
            val, g, H = phi(z, t)
            dz = -np.linalg.solve(H + 1e-300 * np.eye(n), g)
            lam2 = -g @ dz
            if lam2 / 2 <= 1e-13:
                break
            step = 1.0
            while not feasible(z + step * dz):
                step *= 0.5
            while phi(z + step * dz, t)[0] > val - 0.25 * step * lam2:
                step *= 0.5
                if step < 1e-20:
                    break
            z = z + step * dz
        if m / t < gap:
            break
        t *= mu
    du, kv, p = split(z)
    return dict(du=du, kv=kv, p=p, objective=pb.objective(du, kv))
