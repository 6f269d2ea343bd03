"""Host successive-linearisation (SL) outer loop and Monte-Carlo / edge-case
validation around the C ABI.

The paper's NRTO framework is bi-level (Fig. 2): an outer SL loop on
the host linearises the robust trajectory-optimisation problem (Problem 1,
P:113-175) at the current nominal, the inner solver (this library, through
nrto_refresh / nrto_inner_solve) solves the tractable linearised SOCP
(Problem 2), and the host accepts or rejects the step under a trust
region ("linearizes ... packs the SOCP and QP data").  The acceptance
rule and penalty schedule live in the paper's ref. [18]; this module follows
the reconstruction of SPEC S:529-559 with the paper's table values
(P:1291-1310): r_0 = 1.5, r_min = 1e-3, (alpha, beta, eta_1, eta_2) =
(0.8, 1.15, 5, 4), w_p = 100, N_outer = 200, (eps_u, eps_p) = (0.075, 0.01)
(R21-R24).

Model: the planar unicycle of SM §IV (forward Euler, input
saturation) with the disturbance model of Problem 1: x_0 = x_bar_0 + d_bar_0,
x_{k+1} = f(x_k, u_k) + d_k, zeta = [d_bar_0; d_0; ...; d_{T-1}] in the
ellipsoid zeta^T S zeta <= tau (Gamma = I, S block diagonal,
P:1483-1486), affine policy u_k = u_bar_k + K_k d_{k-1}, d_{-1} = d_bar_0
(P:137-144).  Constraints: circular obstacles at every knot, a terminal goal
box (DESIGN R20) and the input bounds |v| <= v_max, |omega| <= omega_max as
control rows (R14).

Validation (§V-A): 1000 disturbances uniform in the interior of the
uncertainty set and 1000 edge cases on its boundary, built as convex
combinations of the worst-case directions of the constraints and renormalised
to the boundary; each is rolled out through the NONLINEAR closed loop with a
fixed seed, and a rollout succeeds iff no constraint is violated by more than
1e-9.

Everything here is host orchestration (numpy); every step of the inner solve
runs in libnrto's kernels.  Tests may inject another inner solver (the oracle)
through `inner=`.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np


# ------------------------------------------------------------------ scenario
@dataclass
class UnicycleScenario:
    """Unicycle robust navigation task (SM §IV, Table)."""
    T: int = 30
    dt: float = 0.1
    tau: float = 0.05                         # tau_0
    x0: tuple = (0.0, 0.0, 0.0)
    goal: tuple = (2.5, 1.5)
    r_goal: float = 0.25
    obstacles: tuple = ()                     # ((cx, cy, r), ...)
    v_max: float = 3.0                        # (v_max, omega_max) = (3, 1.5)
    w_max: float = 1.5
    sigma0: float = 0.02                      # S_0^{-1} = sigma0^2 I  (d_bar_0)
    sigmad: float = 0.01                      # S_d^{-1} = sigmad^2 I  (d_k)
    R_u: float = 0.1                          # R_u = 0.1 I
    W_K: float = 1.0                          # R_K = I
    n_x: int = 3
    n_u: int = 2

    def f(self, x, u):
        """P:1210-1215 forward Euler (u already saturated by the caller)."""
        return np.array([x[0] + u[0] * math.cos(x[2]) * self.dt,
                         x[1] + u[0] * math.sin(x[2]) * self.dt,
                         x[2] + u[1] * self.dt])

    def jac(self, x, u):
        th, v = x[2], u[0]
        A = np.array([[1.0, 0.0, -self.dt * v * math.sin(th)],
                      [0.0, 1.0, self.dt * v * math.cos(th)],
                      [0.0, 0.0, 1.0]])
        B = np.array([[self.dt * math.cos(th), 0.0], [self.dt * math.sin(th), 0.0], [0.0, self.dt]])
        return A, B

    def saturate(self, u):
        return np.array([np.clip(u[0], -self.v_max, self.v_max), np.clip(u[1], -self.w_max, self.w_max)])

    def rollout(self, u, zeta=None):
        """States x_0..x_T for nominal controls u [T, n_u] (zeta = None: no disturbance)."""
        T, nx = self.T, self.n_x
        x = np.zeros((T + 1, nx))
        x[0] = np.asarray(self.x0, float) + (0.0 if zeta is None else zeta[0:nx])
        for k in range(T):
            x[k + 1] = self.f(x[k], self.saturate(u[k]))
            if zeta is not None:
                x[k + 1] += zeta[(k + 1) * nx:(k + 2) * nx]
        return x

    def psi(self):
        """Psi_k with Psi_k^T Psi_k = S_k^{-1}, k = 0..T."""
        P = np.empty((self.T + 1, self.n_x, self.n_x))
        P[0] = self.sigma0 * np.eye(self.n_x)
        P[1:] = self.sigmad * np.eye(self.n_x)
        return P

    # rows: obstacles at knots 1..T, goal box at T (state rows); input bounds (control rows)
    def rows(self):
        knot, kind = [], []
        for k in range(1, self.T + 1):
            for _ in self.obstacles:
                knot.append(k); kind.append(0)
        for _ in range(4):
            knot.append(self.T); kind.append(0)
        for k in range(self.T):
            for _ in range(4):
                knot.append(k); kind.append(1)
        return np.array(knot, np.int32), np.array(kind, np.int8)

    def constraint_values(self, x, u):
        """g_j (state rows at their knots) and h_j (control rows) at (x, u), with
        gradients, in the order of rows()."""
        g, G = [], []
        for k in range(1, self.T + 1):
            for (cx, cy, r) in self.obstacles:
                d = x[k, :2] - np.array([cx, cy])
                nd = max(float(np.linalg.norm(d)), 1e-12)
                g.append(r - nd)
                G.append(np.array([-d[0] / nd, -d[1] / nd, 0.0]))
        for ax in range(2):
            for sgn in (1.0, -1.0):
                g.append(sgn * (x[self.T, ax] - self.goal[ax]) - self.r_goal)
                e = np.zeros(self.n_x); e[ax] = sgn
                G.append(e)
        lim = (self.v_max, self.w_max)
        for k in range(self.T):
            for a in range(2):
                for sgn in (1.0, -1.0):
                    g.append(sgn * u[k, a] - lim[a])
                    e = np.zeros(self.n_x); e[a] = sgn
                    G.append(e)
        return np.array(g), np.array(G)


# ------------------------------------------------------------ linearisation
def linearize(sc: UnicycleScenario, u_hat, r_trust):
    """Problem-2 primitives at the nominal (x_hat, u_hat) (include/nrto.h nrto_data)."""
    x_hat = sc.rollout(u_hat)
    T = sc.T
    A = np.empty((T, sc.n_x, sc.n_x)); B = np.empty((T, sc.n_x, sc.n_u))
    for k in range(T):
        A[k], B[k] = sc.jac(x_hat[k], sc.saturate(u_hat[k]))
    g0, grad = sc.constraint_values(x_hat, u_hat)
    return x_hat, dict(A=A, B=B, grad=grad, g0=g0, Psi=sc.psi(), tau=float(sc.tau),
                       W_K=np.tile(sc.W_K * np.eye(sc.n_u), (T, 1, 1)),
                       R_u=np.tile(sc.R_u * np.eye(sc.n_u), (T, 1, 1)),
                       u_hat=np.array(u_hat, float), r_trust=float(r_trust))


def unvec(kv, T, nu, nx):
    """K_k from the column-major vec(K_k) blocks of k_v."""
    return np.swapaxes(np.asarray(kv).reshape(T, nx, nu), -1, -2)


def robust_terms(sc: UnicycleScenario, data, K):
    """||A_hat_j k_v + b_hat_j|| per row = max_{zeta in U} (closed-loop sensitivity
    of row j)^T zeta (support function): state row at knot k_j:
    block k = sqrt(tau) Psi_k (A_k + B_k K_k)^T c_{j,k+1} (k < k_j), block k_j =
    sqrt(tau) Psi_k grad g_j, with the open-loop costate c_{j,k} = A_k^T c_{j,k+1};
    control row at step k: block k = sqrt(tau) Psi_k K_k^T h'_j (R14)."""
    knot, kind = sc.rows()
    A, Bm, grad, Psi = data["A"], data["B"], data["grad"], data["Psi"]
    st = math.sqrt(data["tau"])
    out = np.zeros(len(knot))
    vecs = []
    for j in range(len(knot)):
        kj = int(knot[j])
        blocks = np.zeros((sc.T + 1, sc.n_x))
        if kind[j] == 0:
            c = grad[j].copy()
            blocks[kj] = st * Psi[kj] @ c
            for k in range(kj - 1, -1, -1):
                blocks[k] = st * Psi[k] @ ((A[k] + Bm[k] @ K[k]).T @ c)
                c = A[k].T @ c
        else:
            blocks[kj] = st * Psi[kj] @ (K[kj].T @ grad[j, :sc.n_u])
        vecs.append(blocks)
        out[j] = float(np.linalg.norm(blocks))
    return out, vecs


# ------------------------------------------------------------- inner solver
class GpuInner:
    """The inner solve through libnrto (C ABI).  One handle, refreshed every SL
    iteration (nrto_refresh); re-created when the penalty changes."""

    def __init__(self, engine="fulladmm", **pkw):
        self.engine, self.pkw = engine, dict(pkw)
        self.solver, self.key = None, None

    def __call__(self, sc, data, params):
        import torch
        from . import nrto
        knot, kind = sc.rows()

        class _Shape:          # nrto.py needs n_x, n_u, T, n_g, cone_knot, cone_kind
            pass
        shp = _Shape()
        shp.n_x, shp.n_u, shp.T, shp.n_g = sc.n_x, sc.n_u, sc.T, len(knot)
        shp.cone_knot, shp.cone_kind = knot, kind
        batch = {k: np.asarray(v, float)[None] if np.ndim(v) else np.array([v], float)
                 for k, v in data.items()}
        dd = nrto.to_tensors(batch, device="cuda")
        key = tuple(sorted(params.items()))
        if self.solver is None or key != self.key:
            if self.solver is not None:
                self.solver.close()
            self.solver = nrto.InnerSolver(shp, dd, **params)
            self.key = key
        else:
            self.solver.refresh(dd)
        eng = nrto.NRTO_FULLADMM if self.engine == "fulladmm" else nrto.NRTO_DR
        out = self.solver.solve(eng, full=True)
        torch.cuda.synchronize()
        return {k: v.cpu().numpy()[0] for k, v in out.items()}

    def close(self):
        if self.solver is not None:
            self.solver.close()
            self.solver = None


# ---------------------------------------------------------------- outer loop
@dataclass
class OuterSettings:
    """P:1291-1310 (FullADMM column where the table gives two values)."""
    max_outer: int = 200
    r0: float = 1.5
    r_min: float = 1e-3
    alpha_tr: float = 0.8
    beta_tr: float = 1.15
    eta1: float = 5.0
    eta2: float = 4.0
    w_p: float = 100.0
    eps_u: float = 0.075
    eps_p: float = 0.01
    rho0: float = 10.0           # FullADMM inner penalty; doubled on persistent slack
    rho_max: float = 180.0
    inner_iters: int = 40        # ADMM iters = 40
    slack_tol: float = 1e-2
    eps_pred: float = 1e-2       # c_eps = 0.01: relative predicted merit decrease read as stationary


def merit(sc, u, K, data, w_p):
    """True cost + w_p * total robust violation at the relinearised nominal
    (SPEC S:553 l1 exact penalty): J = sum u^T R u + sum tr(K^T W K) (Q_u + Q~,
    P:823-840), violation = sum_j max(0, g_j + ||A_hat_j k_v + b_hat_j||)."""
    J = float(sc.R_u * np.sum(u * u) + sc.W_K * np.sum(K * K))
    rob, _ = robust_terms(sc, data, K)
    viol = np.maximum(0.0, data["g0"] + rob)
    return J + w_p * float(viol.sum()), float(viol.max(initial=0.0))


def accept_step(actual, predicted, r, rho, slack, s: OuterSettings):
    """Ratio test: ratio = actual / predicted merit reduction;
    accept iff ratio >= 1/eta_1 (then r <- min(beta r, eta_2 r_0)), else reject
    (r <- max(alpha r, r_min)); persistent slack doubles the penalty up to rho_max."""
    ratio = actual / predicted if predicted > 0 else (1.0 if actual >= 0 else -1.0)
    if predicted > 0 and ratio >= 1.0 / s.eta1:
        ok, r_new = True, min(s.beta_tr * r, s.eta2 * s.r0)
    else:
        ok, r_new = False, max(s.alpha_tr * r, s.r_min)
    rho_new = min(2.0 * rho, s.rho_max) if slack > s.slack_tol else rho
    return ok, r_new, rho_new


@dataclass
class SLResult:
    u: np.ndarray
    K: np.ndarray
    x: np.ndarray
    status: str
    outer_iters: int
    history: list = field(default_factory=list)
    wall_s: float = 0.0
    inner_s: float = 0.0


def run_sl(sc: UnicycleScenario, settings: OuterSettings = None, inner=None, u_init=None):
    """The SL outer loop (Fig. 2): linearise -> inner solve -> candidate rollout
    -> accept / reject -> until ||du||_inf <= eps_u and the max robust
    violation <= eps_p, or max_outer (status "not_converged", never an error)."""
    s = settings or OuterSettings()
    inner = inner or GpuInner()
    T, nu, nx = sc.T, sc.n_u, sc.n_x
    u = np.zeros((T, nu)) if u_init is None else np.array(u_init, float)
    K = np.zeros((T, nu, nx))
    r, rho = s.r0, s.rho0
    t_start = time.perf_counter()
    t_inner = 0.0
    x, data = linearize(sc, u, r)
    m_cur, v_cur = merit(sc, u, K, data, s.w_p)
    hist, status, it = [], "not_converged", 0
    for it in range(1, s.max_outer + 1):
        x, data = linearize(sc, u, r)
        params = dict(rho=rho, max_iter=s.inner_iters, fixed_iters=1)
        t0 = time.perf_counter()
        o = inner(sc, data, params)
        t_inner += time.perf_counter() - t0
        du = np.asarray(o["du"]).reshape(T, nu)
        K_new = unvec(o["kv"], T, nu, nx)
        # model merit: linearised rows g + b^T du + ||A_hat k + b_hat||, from the inner outputs
        rob_lin = -np.asarray(o["margin_lin"]) - o["p"] + o["p_tilde"] - np.asarray(o["margin_cone"])
        J_model = float(sc.R_u * np.sum((u + du) ** 2) + sc.W_K * np.sum(K_new * K_new))
        m_model = J_model + s.w_p * float(np.maximum(0.0, rob_lin).sum())
        u_new = u + du
        _, data_new = linearize(sc, u_new, r)
        m_new, vmax_new = merit(sc, u_new, K_new, data_new, s.w_p)
        slack = float(np.linalg.norm(np.asarray(o["p"]) - np.asarray(o["p_tilde"])))
        pred = m_cur - m_model
        ok, r, rho = accept_step(m_cur - m_new, pred, r, rho, slack, s)
        step = float(np.max(np.abs(du))) if du.size else 0.0
        hist.append(dict(it=it, merit=m_new if ok else m_cur, accepted=ok, r_trust=r, rho=rho,
                         du_inf=step, max_violation=vmax_new if ok else v_cur, slack=slack,
                         predicted=pred))
        if ok:
            u, K, m_cur, v_cur = u_new, K_new, m_new, vmax_new
            if step <= s.eps_u and v_cur <= s.eps_p:
                status = "converged"
                break
        # stationary for the linearisation: the subproblem predicts no further merit
        # decrease at a robustly feasible nominal (the usual SL / SQP stopping test)
        if v_cur <= s.eps_p and pred <= s.eps_pred * max(1.0, abs(m_cur)):
            status = "converged"
            break
        if not ok and r <= s.r_min:
            break
    x = sc.rollout(u)
    return SLResult(u=u, K=K, x=x, status=status, outer_iters=it, history=hist,
                    wall_s=time.perf_counter() - t_start, inner_s=t_inner)


# ---------------------------------------------------------------- validation
def sample_interior(sc: UnicycleScenario, n, seed):
    """n disturbances zeta uniform (by volume) in {zeta^T S zeta <= tau}: zeta =
    Psi^T w with w uniform in the ball of radius sqrt(tau) (Psi^T Psi = S^{-1})."""
    rng = np.random.default_rng(seed)
    nz = (sc.T + 1) * sc.n_x
    w = rng.standard_normal((n, nz))
    w /= np.linalg.norm(w, axis=1, keepdims=True)
    w *= math.sqrt(sc.tau) * rng.uniform(0.0, 1.0, (n, 1)) ** (1.0 / nz)
    return _psiT(sc, w)


def _psiT(sc, w):
    P = sc.psi()
    nx = sc.n_x
    z = np.empty_like(w)
    for k in range(sc.T + 1):
        z[:, k * nx:(k + 1) * nx] = w[:, k * nx:(k + 1) * nx] @ P[k]     # (Psi_k^T w_k)^T
    return z


def sample_edge(sc: UnicycleScenario, data, K, n, seed):
    """n boundary disturbances: random convex combinations of the worst-case
    directions zeta_j* = Psi^T y_j / ||y_j|| sqrt(tau) (y_j = A_hat_j k_v + b_hat_j,
    the maximiser of the support function) of the rows, renormalised to
    zeta^T S zeta = tau."""
    rng = np.random.default_rng(seed)
    rob, vecs = robust_terms(sc, data, K)
    nz = (sc.T + 1) * sc.n_x
    dirs = []
    for j, y in enumerate(vecs):
        ny = np.linalg.norm(y)
        if ny > 0:
            dirs.append((y.reshape(-1) / ny) * math.sqrt(sc.tau))        # w-space maximiser
    if not dirs:
        w = rng.standard_normal((n, nz))
    else:
        D = np.array(dirs)
        lam = rng.dirichlet(np.full(len(D), 0.5), size=n)
        w = lam @ D
    w *= math.sqrt(sc.tau) / np.maximum(np.linalg.norm(w, axis=1, keepdims=True), 1e-300)
    return _psiT(sc, w)


def ellipsoid_value(sc, zeta):
    """zeta^T S zeta for S = blkdiag(S_k), S_k = (Psi_k^T Psi_k)^{-1}."""
    P = sc.psi()
    nx = sc.n_x
    v = 0.0
    for k in range(sc.T + 1):
        w = np.linalg.solve(P[k].T, zeta[..., k * nx:(k + 1) * nx].T).T  # Psi_k^{-T} zeta_k
        v = v + np.sum(w * w, axis=-1)
    return v


def closed_loop(sc, u, K, zeta):
    """Nonlinear rollout under u_k = u_bar_k + K_k d_{k-1} (d_{-1} = d_bar_0)
    with x_{k+1} = f(x_k, sat(u_k)) + d_k; returns (x, u_applied)."""
    T, nx = sc.T, sc.n_x
    x = np.zeros((T + 1, nx))
    ua = np.zeros((T, sc.n_u))
    x[0] = np.asarray(sc.x0, float) + zeta[0:nx]
    for k in range(T):
        d_prev = zeta[k * nx:(k + 1) * nx]
        ua[k] = u[k] + K[k] @ d_prev
        x[k + 1] = sc.f(x[k], sc.saturate(ua[k])) + zeta[(k + 1) * nx:(k + 2) * nx]
    return x, ua


def validate(sc, u, K, n_interior=1000, n_edge=1000, seed=0, tol=1e-9):
    """Fraction of successful closed-loop rollouts over interior + edge samples."""
    _, data = linearize(sc, u, 1.0)
    Z = np.concatenate([sample_interior(sc, n_interior, seed), sample_edge(sc, data, K, n_edge, seed + 1)])
    ok = np.zeros(len(Z), bool)
    worst = np.full(len(Z), -np.inf)
    for i, z in enumerate(Z):
        x, ua = closed_loop(sc, u, K, z)
        g, _ = sc.constraint_values(x, ua)
        worst[i] = g.max(initial=-np.inf)
        ok[i] = worst[i] <= tol
    return {"n_interior": n_interior, "n_edge": n_edge,
            "satisfied_interior": int(ok[:n_interior].sum()), "satisfied_edge": int(ok[n_interior:].sum()),
            "rate": float(ok.mean()), "worst_margin": float(worst.max()), "seed": seed}
