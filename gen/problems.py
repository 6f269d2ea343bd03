"""Synthetic SL-iteration inputs with the shapes of the paper's workloads.

Everything here is *input preparation*: model Jacobians A_k, B_k at a nominal
(x_hat, u_hat) (PAPER.md SM §IV, Table), constraint
gradients / values at the nominal, the uncertainty factor Psi_k with
Psi_k^T Psi_k = S_k^{-1} for S = blkdiag(S_0, S_d, ..., S_d) and Gamma = I
(P:1483-1486), the weights R_u, W_K = R_K^T R_K and r_trust.
None of the method's arithmetic (P:841-869 onwards) lives here.

Instance i of config c is seeded with PCG64(260302642 + 1000*c + i)
(SURVEY.md §8d).  The recipe of every config is stated in DESIGN.md §3.

Row conventions (one SOC cone per row, include/nrto.h):
  kind 0 (state row)   : g_j(x_{k_j}) <= 0,  cone_knot = k_j in 1..T,
                         grad[j] = d g_j / d x_{k_j}  (n_x entries).
  kind 1 (control row) : h_j(u_k) <= 0 linear in u_k, cone_knot = k in 0..T-1,
                         grad[j, :n_u] = h'_j, grad[j, n_u:] = 0.
  g0[j] = g_j(x_hat) or h_j(u_hat).
Rows are emitted grouped: state rows knot-major (k = 1..T), then control rows
step-major (k = 0..T-1).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SEED_BASE = 260302642

CONFIGS = {
    "c1": 1,  # unicycle n_x=3 n_u=2 T=20, 2 circles, single instance, both engines
    "c2": 2,  # quadcopter n_x=12 n_u=4 T=50, 10 spheres + actuator rows, NRTO-DR
    "c3": 3,  # Franka n_x=14 n_u=7 T=100, joint/vel/torque limits + EE sphere, FullADMM
    "c4": 4,  # quadcopter sweep T x obstacles
    "c5": 5,  # batch of Franka c3-shaped instances with per-instance jitter
}


@dataclass
class Shape:
    n_x: int
    n_u: int
    T: int
    cone_knot: np.ndarray  # int32 [n_g]
    cone_kind: np.ndarray  # int8  [n_g]

    @property
    def n_g(self) -> int:
        return int(self.cone_knot.shape[0])

    def key(self):
        return (self.n_x, self.n_u, self.T, self.cone_knot.tobytes(),
                self.cone_kind.tobytes())


# ----------------------------------------------------------------- helpers
def _rng(cfg: int, i: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(SEED_BASE + 1000 * cfg + i))


def _haar(rng: np.random.Generator, n: int) -> np.ndarray:
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    return q * np.sign(np.diag(r))[None, :]


def _psi_blocks(rng, n_x: int, T: int, sigma0: float, sigmad: float) -> np.ndarray:
    """Psi_k = upper Cholesky factor of Sigma_k = S_k^{-1} (input prep).

    Sigma_k = sigma^2 Q diag(e^u) Q^T, u ~ U[-1,1]^n, Q Haar; one Sigma_0 for
    zeta block 0 (d_bar_0) and one shared Sigma_d for blocks 1..T.
    """
    def sig(s):
        Q = _haar(rng, n_x)
        u = rng.uniform(-1.0, 1.0, n_x)
        return (s * s) * (Q * np.exp(u)[None, :]) @ Q.T

    S0, Sd = sig(sigma0), sig(sigmad)
    P0 = np.linalg.cholesky(0.5 * (S0 + S0.T)).T
    Pd = np.linalg.cholesky(0.5 * (Sd + Sd.T)).T
    Psi = np.empty((T + 1, n_x, n_x))
    Psi[0] = P0
    Psi[1:] = Pd
    return Psi


def _fd_jac(f, x, u, h=1e-6):
    n, m = x.size, u.size
    A = np.empty((n, n))
    B = np.empty((n, m))
    for c in range(n):
        e = np.zeros(n); e[c] = h
        A[:, c] = (f(x + e, u) - f(x - e, u)) / (2 * h)
    for c in range(m):
        e = np.zeros(m); e[c] = h
        B[:, c] = (f(x, u + e) - f(x, u - e)) / (2 * h)
    return A, B


# ---------------------------------------------------------------- unicycle
def _unicycle_step(dt):
    def f(x, u):  # P:1210-1215 forward Euler
        return np.array([x[0] + u[0] * math.cos(x[2]) * dt,
                         x[1] + u[0] * math.sin(x[2]) * dt,
                         x[2] + u[1] * dt])
    return f


def make_unicycle(cfg: int, i: int, T: int = 20, n_obs: int = 2, dt: float = 0.1,
                  tau: float = 0.05, sigma0: float = 0.02, sigmad: float = 0.01,
                  r_obs: float = 0.3, r_trust: float = 1.5, r_goal: float = 0.05):
    rng = _rng(cfg, i)
    n_x, n_u = 3, 2
    f = _unicycle_step(dt)
    u_hat = np.stack([np.full(T, 1.0),
                      0.3 * np.sin(2 * math.pi * np.arange(T) / T + rng.uniform(0, 0.3))], 1)
    x = np.zeros((T + 1, n_x))
    for k in range(T):
        x[k + 1] = f(x[k], u_hat[k])
    A = np.empty((T, n_x, n_x)); B = np.empty((T, n_x, n_u))
    for k in range(T):  # analytic Jacobians of P:1212-1214
        th, v = x[k, 2], u_hat[k, 0]
        A[k] = np.array([[1, 0, -dt * v * math.sin(th)], [0, 1, dt * v * math.cos(th)], [0, 0, 1]])
        B[k] = np.array([[dt * math.cos(th), 0], [dt * math.sin(th), 0], [0, dt]])
    # obstacles beside the nominal path (clearance U[0.05,0.25] x scene scale 1)
    centers = []
    for o in range(n_obs):
        k = max(1, min(T, round((o + 1) * T / (n_obs + 1))))
        th = x[k, 2]
        nrm = np.array([-math.sin(th), math.cos(th)]) * (1 if rng.uniform() < 0.5 else -1)
        centers.append(x[k, :2] + nrm * (r_obs + rng.uniform(0.05, 0.25)))
    knot, kind, grad, g0 = [], [], [], []
    for k in range(1, T + 1):
        for c in centers:
            d = x[k, :2] - c
            nd = float(np.linalg.norm(d))
            knot.append(k); kind.append(0)
            grad.append([-d[0] / nd, -d[1] / nd, 0.0]); g0.append(r_obs - nd)
    for ax in range(2):  # terminal goal box |p_T - goal| <= r_goal, goal = nominal end
        for sgn in (1.0, -1.0):
            gr = np.zeros(n_x); gr[ax] = sgn
            knot.append(T); kind.append(0); grad.append(gr); g0.append(-r_goal)
    shape = Shape(n_x, n_u, T, np.array(knot, np.int32), np.array(kind, np.int8))
    data = dict(A=A, B=B, grad=np.array(grad), g0=np.array(g0),
                Psi=_psi_blocks(rng, n_x, T, sigma0, sigmad), tau=float(tau),
                W_K=np.tile(np.eye(n_u), (T, 1, 1)), R_u=np.tile(0.1 * np.eye(n_u), (T, 1, 1)),
                u_hat=u_hat, r_trust=float(r_trust))
    return shape, data


# -------------------------------------------------------------- quadcopter
_QM, _QG, _QJ = 1.0, 9.81, np.array([0.02, 0.02, 0.04])  # Table


def _quad_step(dt):
    def f(x, u):  # P:1221-1237, forward Euler
        p, v, (ph, th, ps), w = x[0:3], x[3:6], x[6:9], x[9:12]
        cph, sph, cth, sth, cps, sps = (math.cos(ph), math.sin(ph), math.cos(th),
                                        math.sin(th), math.cos(ps), math.sin(ps))
        Rz = np.array([[cps, -sps, 0], [sps, cps, 0], [0, 0, 1]])
        Ry = np.array([[cth, 0, sth], [0, 1, 0], [-sth, 0, cth]])
        Rx = np.array([[1, 0, 0], [0, cph, -sph], [0, sph, cph]])
        R = Rz @ Ry @ Rx
        vdot = -_QG * np.array([0, 0, 1.0]) + (u[0] / _QM) * R[:, 2]
        Jw = _QJ * w
        wdot = (u[1:4] - np.cross(w, Jw)) / _QJ
        Tm = np.array([[1, sph * math.tan(th), cph * math.tan(th)],
                       [0, cph, -sph],
                       [0, sph / cth, cph / cth]])
        adot = Tm @ w
        return x + dt * np.concatenate([v, vdot, adot, wdot])
    return f


def make_quad(cfg: int, i: int, T: int = 50, n_obs: int = 10, dt: float = 0.05,
              tau: float = 0.05, sigma0: float = 0.02, sigmad: float = 0.01,
              r_obs: float = 0.5, r_trust: float = 2.5, r_goal: float = 0.1):
    rng = _rng(cfg, i)
    n_x, n_u = 12, 4
    f = _quad_step(dt)
    ph0 = rng.uniform(0, 2 * math.pi, 3)
    kk = np.arange(T)
    u_hat = np.stack([_QM * _QG * (1 + 0.01 * np.sin(2 * math.pi * kk / T + ph0[0])),
                      1e-3 * np.sin(2 * math.pi * kk / T + ph0[1]),
                      1e-3 * np.cos(2 * math.pi * kk / T + ph0[2]),
                      np.zeros(T)], 1)
    x = np.zeros((T + 1, n_x))
    x[0, 3:6] = [1.0, 0.2 * rng.uniform(-1, 1), 0.0]
    for k in range(T):
        x[k + 1] = f(x[k], u_hat[k])
    A = np.empty((T, n_x, n_x)); B = np.empty((T, n_x, n_u))
    for k in range(T):
        A[k], B[k] = _fd_jac(f, x[k], u_hat[k])
    centers = []
    for o in range(n_obs):
        k = max(1, min(T, round((o + 0.5) * T / n_obs)))
        vdir = x[k, 3:6] / (np.linalg.norm(x[k, 3:6]) + 1e-12)
        r = rng.standard_normal(3)
        r -= vdir * (r @ vdir)
        r /= np.linalg.norm(r)
        centers.append(x[k, 0:3] + r * (r_obs + rng.uniform(0.05, 0.25)))
    knot, kind, grad, g0 = [], [], [], []
    for k in range(1, T + 1):
        for c in centers:
            d = x[k, 0:3] - c
            nd = float(np.linalg.norm(d))
            gr = np.zeros(n_x); gr[0:3] = -d / nd
            knot.append(k); kind.append(0); grad.append(gr); g0.append(r_obs - nd)
    for ax in range(3):  # terminal goal box
        for sgn in (1.0, -1.0):
            gr = np.zeros(n_x); gr[ax] = sgn
            knot.append(T); kind.append(0); grad.append(gr); g0.append(-r_goal)
    lo = np.array([0.0, -0.5, -0.5, -0.5]); hi = np.array([15.0, 0.5, 0.5, 0.5])
    for k in range(T):
        for a in range(n_u):
            for sgn in (1.0, -1.0):  # u_a - hi <= 0 ; lo - u_a <= 0
                gr = np.zeros(n_x); gr[a] = sgn
                knot.append(k); kind.append(1); grad.append(gr)
                g0.append(u_hat[k, a] - hi[a] if sgn > 0 else lo[a] - u_hat[k, a])
    shape = Shape(n_x, n_u, T, np.array(knot, np.int32), np.array(kind, np.int8))
    data = dict(A=A, B=B, grad=np.array(grad), g0=np.array(g0),
                Psi=_psi_blocks(rng, n_x, T, sigma0, sigmad), tau=float(tau),
                W_K=np.tile(np.eye(n_u), (T, 1, 1)), R_u=np.tile(0.1 * np.eye(n_u), (T, 1, 1)),
                u_hat=u_hat, r_trust=float(r_trust))
    return shape, data


# ------------------------------------------------------------------ Franka
_FQMIN = np.array([-2.9007, -1.8361, -2.9007, -3.0770, -2.8763, 0.4398, -3.0508])
_FQMAX = np.array([2.9007, 1.8361, 2.9007, -0.1169, 2.8763, 4.6216, 3.0508])
_FDQMAX = np.array([2.62, 2.62, 2.62, 2.62, 5.26, 4.18, 5.26])
_FTAUMAX = np.array([87, 87, 87, 87, 12, 12, 12], float)
_FD, _FI = 0.5, 1.0
# Panda kinematics (Craig modified DH; the paper omits DH values)
_DH_A = np.array([0, 0, 0, 0.0825, -0.0825, 0, 0.088, 0])
_DH_D = np.array([0.333, 0, 0.316, 0, 0.384, 0, 0, 0.107])
_DH_AL = np.array([0, -math.pi / 2, math.pi / 2, math.pi / 2, -math.pi / 2, math.pi / 2,
                   math.pi / 2, 0])


def panda_ee(q: np.ndarray) -> np.ndarray:
    """End-effector position for a batch of configurations q [..., 7]."""
    q = np.asarray(q, float)
    lead = q.shape[:-1]
    M = np.broadcast_to(np.eye(4), lead + (4, 4)).copy()
    th = np.concatenate([q, np.zeros(lead + (1,))], -1)
    for j in range(8):
        ca, sa = math.cos(_DH_AL[j]), math.sin(_DH_AL[j])
        ct, st = np.cos(th[..., j]), np.sin(th[..., j])
        T = np.zeros(lead + (4, 4))
        T[..., 0, 0] = ct; T[..., 0, 1] = -st; T[..., 0, 3] = _DH_A[j]
        T[..., 1, 0] = st * ca; T[..., 1, 1] = ct * ca; T[..., 1, 2] = -sa; T[..., 1, 3] = -sa * _DH_D[j]
        T[..., 2, 0] = st * sa; T[..., 2, 1] = ct * sa; T[..., 2, 2] = ca; T[..., 2, 3] = ca * _DH_D[j]
        T[..., 3, 3] = 1
        M = M @ T
    return M[..., 0:3, 3]


def make_franka(cfg: int, i: int, T: int = 100, dt: float = 0.05, tau: float = 0.01,
                sigma0: float = 0.1, sigmad: float = 0.1, r_obs: float = 0.1,
                r_trust: float = 2.0, r_goal: float = 0.3, jitter: bool = False,
                near: float = 0.97, sway: float = 0.3, jit_q: float = 0.05,
                nnear: int = 4, t_hold: float = 0.5, ru: float = 0.01,
                vfrac: float = 0.985, n_cyc: float = 2.0):
    rng = _rng(cfg, i)
    base = _rng(cfg, 0) if jitter else rng  # c5: shared scene, per-instance jitter
    n_x, n_u = 14, 7
    mid, half = 0.5 * (_FQMIN + _FQMAX), 0.5 * (_FQMAX - _FQMIN)
    qa = mid + 0.8 * half * base.uniform(-1, 1, 7)
    qb = mid + 0.8 * half * base.uniform(-1, 1, 7)
    qa[[0, 2]] = mid[[0, 2]] + 0.2 * half[[0, 2]] * base.uniform(-1, 1, 2)
    # nnear of the joints {2,4,5,6,7} are driven close to a limit (held there from
    # t_hold on) so that their robust position rows bind; joints 1 and 3 sweep
    # back and forth at vfrac of their velocity limit (clipped-sine velocity
    # profile with flat cruise phases) so that robust velocity rows bind; any
    # remaining joint sways on top of its transfer
    near_js = base.choice(np.array([1, 3, 4, 5, 6]), nnear, replace=False)
    cruise_js = np.array([0, 2])
    for jj in near_js:
        qb[jj] = mid[jj] + near * half[jj] * (1 if base.uniform() < 0.5 else -1)
    obs_dir = base.standard_normal(3)
    clear = base.uniform(0.03, 0.08)
    ph = base.uniform(0, 1)
    if jitter:  # c5: x_bar_0 ~ N(0, 0.05^2), endpoint jitter, obstacle +-5 cm
        qa = np.clip(qa + rng.normal(0, jit_q, 7), _FQMIN + 0.02 * half, _FQMAX - 0.02 * half)
        qb = np.clip(qb + rng.normal(0, jit_q, 7), _FQMIN + 0.02 * half, _FQMAX - 0.02 * half)
        # the held joints never end closer to their limit than `near`
        qb[near_js] = np.clip(qb[near_js], mid[near_js] - near * half[near_js],
                              mid[near_js] + near * half[near_js])
    t = np.arange(T + 1) / T
    th = np.full(7, 1.0)
    th[near_js] = t_hold
    s = 0.5 * (1 - np.cos(math.pi * np.minimum(t[:, None] / th[None, :], 1.0)))
    q = qa[None, :] + s * (qb - qa)[None, :]
    # a 4-period sway on the free joints so that velocity / torque rows vary
    amp = sway * np.array([0.15, 0.15, 0.15, 0.15, 0.35, 0.35, 0.35])
    amp[near_js] = 0.0
    amp[cruise_js] = 0.0
    q = q + np.sin(8 * math.pi * t)[:, None] * np.sin(math.pi * t)[:, None] * amp[None, :]
    # cruise joints: dq = vfrac * dq_max * clip(1.6 sin(2 pi (n_cyc t + ph)), -1, 1),
    # position = running sum (semi-implicit Euler), centred on the joint's mid-range
    vel = np.clip(1.6 * np.sin(2 * math.pi * (n_cyc * t[1:] + ph)), -1.0, 1.0)
    for jj in cruise_js:
        qc = np.concatenate([[0.0], np.cumsum(vfrac * _FDQMAX[jj] * vel * dt)])
        q[:, jj] = qa[jj] - 0.5 * (qc.max() + qc.min()) + qc
    dq = np.zeros((T + 1, 7))
    dq[1:] = (q[1:] - q[:-1]) / dt          # semi-implicit Euler
    tauu = _FI * (dq[1:] - dq[:-1]) / dt + _FD * dq[:-1]
    x = np.concatenate([q, dq], 1)
    a = 1.0 - dt * _FD / _FI
    A1 = np.zeros((n_x, n_x)); A1[:7, :7] = np.eye(7); A1[:7, 7:] = dt * a * np.eye(7)
    A1[7:, 7:] = a * np.eye(7)
    B1 = np.zeros((n_x, n_u)); B1[:7] = dt * dt / _FI * np.eye(7); B1[7:] = dt / _FI * np.eye(7)
    A = np.tile(A1, (T, 1, 1)); B = np.tile(B1, (T, 1, 1))
    ee = panda_ee(q)
    kc = T // 2
    od = obs_dir / np.linalg.norm(obs_dir)
    center = ee[kc] + od * (r_obs + clear)
    if jitter:
        center = center + rng.uniform(-0.05, 0.05, 3)
    # the nominal keeps its clearance at EVERY knot (no row violated at the nominal)
    # (and a wider berth away from the encounter knot kc)
    need = r_obs + clear + 0.1 * np.minimum(1.0, np.abs(np.arange(T + 1) - kc) / 20.0)
    for _ in range(2000):
        dist = np.linalg.norm(ee - center[None, :], axis=1)
        kmin = int(np.argmin(dist - need))
        if dist[kmin] >= need[kmin]:
            break
        center = center + 0.002 * (center - ee[kmin]) / max(dist[kmin], 1e-9)
    h = 1e-6
    Jp = np.empty((T + 1, 3, 7))
    for c in range(7):
        e = np.zeros(7); e[c] = h
        Jp[:, :, c] = (panda_ee(q + e) - panda_ee(q - e)) / (2 * h)
    knot, kind, grad, g0 = [], [], [], []
    for k in range(1, T + 1):
        for jn in range(7):
            for sgn in (1.0, -1.0):  # q - qmax <= 0 ; qmin - q <= 0
                gr = np.zeros(n_x); gr[jn] = sgn
                knot.append(k); kind.append(0); grad.append(gr)
                g0.append(q[k, jn] - _FQMAX[jn] if sgn > 0 else _FQMIN[jn] - q[k, jn])
        for jn in range(7):
            for sgn in (1.0, -1.0):
                gr = np.zeros(n_x); gr[7 + jn] = sgn
                knot.append(k); kind.append(0); grad.append(gr)
                g0.append(sgn * dq[k, jn] - _FDQMAX[jn])
        d = ee[k] - center
        nd = float(np.linalg.norm(d))
        gr = np.zeros(n_x); gr[:7] = -(d / nd) @ Jp[k]
        knot.append(k); kind.append(0); grad.append(gr); g0.append(r_obs - nd)
    for ax in range(3):  # terminal end-effector goal box, goal = nominal EE at T
        for sgn in (1.0, -1.0):
            gr = np.zeros(n_x); gr[:7] = sgn * Jp[T, ax]
            knot.append(T); kind.append(0); grad.append(gr); g0.append(-r_goal)
    for k in range(T):
        for jn in range(7):
            for sgn in (1.0, -1.0):
                gr = np.zeros(n_x); gr[jn] = sgn
                knot.append(k); kind.append(1); grad.append(gr)
                g0.append(sgn * tauu[k, jn] - _FTAUMAX[jn])
    shape = Shape(n_x, n_u, T, np.array(knot, np.int32), np.array(kind, np.int8))
    data = dict(A=A, B=B, grad=np.array(grad), g0=np.array(g0),
                Psi=_psi_blocks(base, n_x, T, sigma0, sigmad), tau=float(tau),
                W_K=np.tile(np.eye(n_u), (T, 1, 1)), R_u=np.tile(ru * np.eye(n_u), (T, 1, 1)),
                u_hat=tauu, r_trust=float(r_trust))
    return shape, data


# ------------------------------------------------------------------ public
def make_instance(cfg: str, i: int = 0, **kw):
    """(Shape, data dict) for instance i of config cfg ('c1'..'c5')."""
    c = CONFIGS[cfg]
    if cfg == "c1":
        return make_unicycle(c, i, **kw)
    if cfg == "c2":
        return make_quad(c, i, **kw)
    if cfg == "c3":
        return make_franka(c, i, **kw)
    if cfg == "c4":
        return make_quad(c, i, **kw)
    if cfg == "c5":
        kw.setdefault("jitter", True)
        return make_franka(c, i, **kw)
    raise KeyError(cfg)


def stack_instances(items):
    """Stack [(shape, data)] with identical shapes into one batch dict."""
    shape = items[0][0]
    for s, _ in items[1:]:
        if s.key() != shape.key():
            raise ValueError("instances in a batch must share the cone structure")
    keys = items[0][1].keys()
    batch = {}
    for k in keys:
        vals = [d[k] for _, d in items]
        batch[k] = np.ascontiguousarray(np.stack([np.asarray(v, float) for v in vals]))
    return shape, batch


def make_batch(cfg: str, n: int, start: int = 0, **kw):
    return stack_instances([make_instance(cfg, start + i, **kw) for i in range(n)])


def make_config(cfg: str, **kw):
    return make_instance(cfg, 0, **kw)


def config_shape(cfg: str, **kw) -> Shape:
    return make_instance(cfg, 0, **kw)[0]
