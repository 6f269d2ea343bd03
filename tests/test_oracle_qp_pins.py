"""Iterate-by-iterate pins of the (14a)/(5b) QP reading R1 (OSQP-form ADMM).

The paper only says "PCG with a Jacobi preconditioner"; DESIGN R1 reads
the QP as the OSQP ADMM iteration (Stellato et al., Algorithm 1).  Round 1 pinned
that reading only at convergence, where a misplaced relaxation or a wrong dual
step still reaches the same optimum.  These pins hold at EVERY iteration and
follow from the structure of the method, not from its formulas:

(P1) x-step = KKT.  x~ solves the quasi-definite system
     [P + sigma I, C^T; C, -I/rho_q] [x~; nu] = [sigma x - q; z - y/rho_q]
     with C = [[B, I], [F_u, 0]] formed LITERALLY from the dense tier (F_u by
     unit responses of the linearised dynamics; b_j = F_u^T grad g_j,
     P:843) -- not from the Riccati sweep that the structured QP uses -- and
     z~ = C x~.
(P2) dual feasibility.  y^{k+1}/rho_q = w - Pi_C(w), w = (relaxed z) + y^k/rho_q,
     so y^{k+1} lies in the normal cone of the constraint set at z^{k+1}:
     rows y_l >= 0, z_l <= -g_l, y_l (z_l + g_l) = 0; ball y_b = mu z_b with
     mu >= 0, mu (||z_b|| - r) = 0.  (Moreau decomposition.)
(P3) averaged operator.  OSQP's ADMM is relaxed Douglas-Rachford on the
     splitting f(x~, z~) = QP cost + I{C x~ = z~}, g(x, z) = I_C(z) with the
     variable s^k = (x^k, z^k + y^k/rho_q) (derivation: ADMM with prox_g first,
     s^k = X^k + U^k, s^{k+1} = s^k + alpha (prox_f(2 prox_g(s^k) - s^k) -
     prox_g(s^k)), Eckstein-Bertsekas); for alpha in (0,2) the map is averaged
     in the metric M = diag(sigma I, rho_q I), hence for a fixed v
       ||s^{k+1} - s^k||_M  is non-increasing,  and
       ||s^k - s*||_M       is non-increasing (Fejer) for the fixed point s*.
(P4) relaxed-DR form.  The same derivation gives, iterate by iterate,
       s^{k+1} - s^k = alpha ( (x~, z~) - prox_g(s^k) ),
       prox_g(s) = (s_x, Pi_C(s_z))   (Pi_C: rows min(., -g), ball radius r),
     which ties the relaxation alpha to BOTH the primal and the dual sequence.

Every pin is also checked to FAIL on plausible mistakes (mutants of the
iteration below): relaxation applied to x only, the dual step taken with the
unrelaxed z~, a dual step of the wrong sign, relaxation in the z-projection but
not in the dual step.
"""
import numpy as np
import pytest

from oracle import dense
from oracle import structured as st
from tests.helpers import tiny, make_feasible


def _instance(kind="uni", T=3, seed=0, r_trust=0.12):
    shape, data = tiny(kind, T=T, seed=seed, r_trust=r_trust)
    pb = dense.DenseProblem(shape, data)
    data = make_feasible(pb, data, np.random.default_rng(seed), lo=0.002, hi=0.05)
    return shape, data, dense.DenseProblem(shape, data)


def _v(pb, seed):
    # v = p~ - lam_p: targets that make rows and the trust region bind
    return np.random.default_rng(100 + seed).uniform(-0.05, 0.3, pb.ng)


def _literal_C(pb):
    C = np.zeros((pb.ng + pb.NX, pb.NU + pb.ng))
    C[:pb.ng, :pb.NU] = pb.b
    C[:pb.ng, pb.NU:] = np.eye(pb.ng)
    C[pb.ng:, :pb.NU] = pb.F_u
    return C


def _Pq(pb, rho, v):
    P = np.zeros((pb.NU + pb.ng, pb.NU + pb.ng))
    P[:pb.NU, :pb.NU] = 2.0 * pb.Ru
    P[pb.NU:, pb.NU:] = rho * np.eye(pb.ng)
    q = np.concatenate([2.0 * pb.Ru @ pb.u_hat, -rho * v])
    return P, q


# ------------------------------------------------------------------ the pins
def pin_kkt(pb, tr, x0, z0, y0, rho, rq, sq, v):
    C = _literal_C(pb)
    P, q = _Pq(pb, rho, v)
    x, z, y = x0, z0, y0
    worst = 0.0
    for r in tr:
        xt, zt = r["xt"], r["zt"]
        nu = rq * (C @ xt - z + y / rq)                      # second block row
        res = (P + sq * np.eye(len(xt))) @ xt + C.T @ nu - (sq * x - q)
        sc = 1.0 + np.linalg.norm(q) + np.linalg.norm(C.T @ nu) + np.linalg.norm(P @ xt)
        worst = max(worst, np.linalg.norm(res) / sc, np.linalg.norm(zt - C @ xt) / (1 + np.linalg.norm(zt)))
        x, z, y = r["x"], r["z"], r["y"]
    return worst


def pin_normal_cone(pb, tr):
    ng = pb.ng
    worst = 0.0
    for r in tr:
        z, y = r["z"], r["y"]
        sc = 1.0 + np.linalg.norm(y) + np.linalg.norm(z)
        zl, yl = z[:ng], y[:ng]
        worst = max(worst, max(0.0, -yl.min(initial=0.0)) / sc,
                    max(0.0, (zl + pb.g0).max(initial=0.0)) / sc,
                    np.abs(yl * (zl + pb.g0)).max(initial=0.0) / sc ** 2)
        zb, yb = z[ng:], y[ng:]
        nz = np.linalg.norm(zb)
        if nz < pb.r_trust * (1 - 1e-9):                      # interior: y_b = 0
            worst = max(worst, np.linalg.norm(yb) / sc)
        else:                                                 # boundary: y_b = mu z_b, mu >= 0
            mu = yb @ zb / nz ** 2
            worst = max(worst, np.linalg.norm(yb - mu * zb) / sc, max(0.0, -mu) * nz / sc,
                        abs(nz - pb.r_trust) / (1 + pb.r_trust))
    return worst


def _proj_C(pb, w):
    # Euclidean projection onto {z_l <= -g} x {||z_b|| <= r} (its definition)
    out = np.minimum(w[:pb.ng], -pb.g0)
    zb = w[pb.ng:]
    nb = np.linalg.norm(zb)
    return np.concatenate([out, zb * (pb.r_trust / nb) if nb > pb.r_trust else zb])


def pin_dr_form(pb, tr, s0, rq, aq):
    nx_ = pb.NU + pb.ng
    s = s0
    worst = 0.0
    for r in tr:
        s1 = _s(r, rq)
        pg = np.concatenate([s[:nx_], _proj_C(pb, s[nx_:])])
        want = s + aq * (np.concatenate([r["xt"], r["zt"]]) - pg)
        worst = max(worst, np.linalg.norm(s1 - want) / (1 + np.linalg.norm(s1)))
        s = s1
    return worst


def _s(r, rq):
    return np.concatenate([r["x"], r["z"] + r["y"] / rq])


def _mnorm(d, nx_, sq, rq):
    return np.sqrt(sq * d[:nx_] @ d[:nx_] + rq * d[nx_:] @ d[nx_:])


def pin_averaged(pb, tr, s0, s_star, sq, rq):
    """Largest relative increase of ||s^{k+1}-s^k||_M and of ||s^k - s*||_M."""
    nx_ = pb.NU + pb.ng
    ss = [s0] + [_s(r, rq) for r in tr]
    d = [_mnorm(ss[k + 1] - ss[k], nx_, sq, rq) for k in range(len(ss) - 1)]
    e = [_mnorm(s - s_star, nx_, sq, rq) for s in ss]
    sc = max(d[0], 1e-300)
    inc_d = max((d[k + 1] - d[k]) / sc for k in range(len(d) - 1))
    inc_e = max((e[k + 1] - e[k]) / max(e[0], 1e-300) for k in range(len(e) - 1))
    return max(inc_d, inc_e)


# ------------------------------------------------------------------ mutants
class _Mutant(dense.DenseQP):
    """DenseQP with one plausible mistake in the iteration (test-only)."""
    kind = "x_only"

    def solve(self, v, iters, trace=None):
        pb = self.pb
        q = np.concatenate([2.0 * pb.Ru @ pb.u_hat, -self.rho * v])
        a, rq = self.alpha_q, self.rho_q
        for _ in range(iters):
            rhs = self.sigma_q * self.x - q + self.C.T @ (rq * self.z - self.y)
            xt = np.linalg.solve(self.Kmat, rhs)
            zt = self.C @ xt
            self.x = a * xt + (1 - a) * self.x
            zh = a * zt + (1 - a) * self.z
            if self.kind == "x_only":            # relaxation on x only
                znew = self.proj(zt + self.y / rq); ynew = self.y + rq * (zt - znew)
            elif self.kind == "dual_unrelaxed":  # dual step with z~ instead of the relaxed z
                znew = self.proj(zh + self.y / rq); ynew = self.y + rq * (zt - znew)
            elif self.kind == "dual_sign":       # dual step of the wrong sign
                znew = self.proj(zh + self.y / rq); ynew = self.y - rq * (zh - znew)
            elif self.kind == "proj_unrelaxed":  # relaxed dual step, unrelaxed projection
                znew = self.proj(zt + self.y / rq); ynew = self.y + rq * (zh - znew)
            self.y, self.z = ynew, znew
            if trace is not None:
                trace.append(dict(xt=xt.copy(), zt=zt.copy(), x=self.x.copy(), z=self.z.copy(),
                                  y=self.y.copy()))
        return self.x[:pb.NU].copy(), self.x[pb.NU:].copy()


RHO, RQ, SQ, AQ = 10.0, 1.0, 1e-6, 1.6


def _ok(pins):
    kkt, ncone, avg, drf = pins
    return kkt <= 1e-10 and ncone <= 1e-10 and avg <= 1e-9 and drf <= 1e-12


def _run_pins(qp_factory, pb, v, warm=40, n=60):
    """Warm the QP up, record n iterations, evaluate the three pins."""
    qp = qp_factory()
    qp.solve(v, warm)
    x0, z0, y0 = _state(qp)
    tr = []
    qp.solve(v, n, trace=tr)
    # fixed point for the Fejer pin: the same (correct) iteration run to convergence
    ref = dense.DenseQP(pb, RHO, RQ, SQ, AQ)
    ref.solve(v, 40000)
    s_star = np.concatenate([ref.x, ref.z + ref.y / RQ])
    s0 = np.concatenate([x0, z0 + y0 / RQ])
    return (pin_kkt(pb, tr, x0, z0, y0, RHO, RQ, SQ, v), pin_normal_cone(pb, tr),
            pin_averaged(pb, tr, s0, s_star, SQ, RQ), pin_dr_form(pb, tr, s0, RQ, AQ))


def _state(qp):
    if isinstance(qp, st.RiccatiQP):
        return (np.concatenate([qp.du.reshape(-1), qp.p]), np.concatenate([qp.zl, qp.zb.reshape(-1)]),
                np.concatenate([qp.yl, qp.yb.reshape(-1)]))
    return qp.x.copy(), qp.z.copy(), qp.y.copy()


CASES = [("uni", 3, 0), ("uni", 4, 1), ("quad", 2, 2)]


@pytest.mark.parametrize("kind,T,seed", CASES)
def test_qp_iterates_pinned_dense(kind, T, seed):
    shape, data, pb = _instance(kind, T, seed)
    v = _v(pb, seed)
    pins = _run_pins(lambda: dense.DenseQP(pb, RHO, RQ, SQ, AQ), pb, v)
    assert _ok(pins), pins


@pytest.mark.parametrize("kind,T,seed", CASES)
def test_qp_iterates_pinned_riccati(kind, T, seed):
    """The structured (Riccati) QP that the GPU parity tests compare against
    satisfies the same pins, with C taken from the dense literal tier."""
    shape, data, pb = _instance(kind, T, seed)
    sp = st.StructuredProblem(shape, data)
    v = _v(pb, seed)
    pins = _run_pins(lambda: st.RiccatiQP(sp, RHO, RQ, SQ, AQ), pb, v)
    assert _ok(pins), pins


def test_qp_pins_bind():
    """The trust region and some rows are active in the pinned iterations (the
    pins are not vacuous)."""
    for kind, T, seed in CASES:
        shape, data, pb = _instance(kind, T, seed)
        qp = dense.DenseQP(pb, RHO, RQ, SQ, AQ)
        qp.solve(_v(pb, seed), 100)
        assert np.linalg.norm(qp.z[pb.ng:]) >= pb.r_trust * (1 - 1e-9)
        assert np.sum(qp.y[:pb.ng] > 1e-8) >= 1


@pytest.mark.parametrize("mut", ["x_only", "dual_unrelaxed", "dual_sign", "proj_unrelaxed"])
def test_qp_pins_catch_mutants(mut):
    """Each plausible mistake breaks at least one pin on at least one case."""
    caught = False
    for kind, T, seed in CASES:
        shape, data, pb = _instance(kind, T, seed)
        v = _v(pb, seed)

        def fac():
            m = _Mutant(pb, RHO, RQ, SQ, AQ)
            m.kind = mut
            return m
        with np.errstate(all="ignore"):
            pins = _run_pins(fac, pb, v)
        if not _ok(pins):
            caught = True
            break
    assert caught, mut
