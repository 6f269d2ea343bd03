"""Dense, literal definitions of the NRTO inner solve (tiny instances only).

Every matrix of the paper is formed explicitly, so a reader can check each
line against PAPER.md by eye.  Cost is O(n_g n_z (T n_u n_x)^2): use for
T <= ~6, n_x <= 3.

Notation: zeta = [d_bar_0; d_0; ...; d_{T-1}], x_0 = x_bar_0 + d_bar_0,
x_{k+1} = f + d_k, u_k = u_bar_k + K_k d_{k-1}, d_{-1} = d_bar_0
(P:137-144), k_v = [vec(K_0); ...; vec(K_{T-1})] with column-major vec
(P:178-180).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .soc import proj_soc


# --------------------------------------------------------------- problem data
class DenseProblem:
    """All constants of one SL iteration, formed literally.

    General uncertainty set: zeta = Gamma z, z^T S z <= tau with
    Gamma in R^{(T+1)n_x x n_z} (default I) and S in S^{n_z}_{++} (default the
    block-diagonal S of the generator's Psi_k blocks); Psi^T Psi = S^{-1} and
    A_hat_j = sqrt(tau) Psi Gamma^T [A_bar_j; 0], b_hat_j = sqrt(tau) Psi
    Gamma^T F_zeta^T grad g_j.
    """

    def __init__(self, shape, data, S=None, Gamma=None):
        nx, nu, T = shape.n_x, shape.n_u, shape.T
        ng = shape.n_g
        self.nx, self.nu, self.T, self.ng = nx, nu, T, ng
        self.knot = np.asarray(shape.cone_knot)
        self.kind = np.asarray(shape.cone_kind)
        A, B = np.asarray(data["A"]), np.asarray(data["B"])
        NX = (T + 1) * nx            # dim of stacked x and of zeta
        NU = T * nu
        NK = T * nu * nx             # dim k_v
        G = np.eye(NX) if Gamma is None else np.asarray(Gamma, float)
        nz = G.shape[1]
        self.Gamma = G
        self.NX, self.NU, self.NK, self.nz = NX, NU, NK, nz

        # F_u, F_zeta: delta_x = F_u delta_u + F_zeta zeta for the linearised
        # dynamics dx_{k+1} = A_k dx_k + B_k du_k + d_k, dx_0 = d_bar_0
        # (definition via unit responses; the paper defers F_u to [18]).
        def simulate(du, zeta):
            dx = np.zeros((T + 1, nx))
            dx[0] = zeta[0:nx]
            for k in range(T):
                dx[k + 1] = A[k] @ dx[k] + B[k] @ du[k * nu:(k + 1) * nu] \
                    + zeta[(k + 1) * nx:(k + 2) * nx]
            return dx.reshape(-1)

        self.F_u = np.zeros((NX, NU))
        for c in range(NU):
            e = np.zeros(NU); e[c] = 1.0
            self.F_u[:, c] = simulate(e, np.zeros(NX))
        self.F_z = np.zeros((NX, NX))
        for c in range(NX):
            e = np.zeros(NX); e[c] = 1.0
            self.F_z[:, c] = simulate(np.zeros(NU), e)

        # S and Psi with Psi^T Psi = S^{-1}; default S = blkdiag(S_k)
        # with S_k^{-1} = Psi_k^T Psi_k from the generator's blocks.
        if S is None:
            if Gamma is not None:
                raise ValueError("a general Gamma needs its S")
            S = np.zeros((NX, NX))
            for k in range(T + 1):
                Pk = np.asarray(data["Psi"][k])
                S[k * nx:(k + 1) * nx, k * nx:(k + 1) * nx] = np.linalg.inv(Pk.T @ Pk)
        self.S = S
        Sinv = np.linalg.inv(S)
        self.Psi = np.linalg.cholesky(0.5 * (Sinv + Sinv.T)).T      # upper
        tau = float(data["tau"])
        self.tau = tau
        st = np.sqrt(tau)

        # rows: b_j, A_bar_j, A_hat_j, b_hat_j; control rows (R14)
        self.g0 = np.asarray(data["g0"], float)
        grad = np.asarray(data["grad"], float)
        self.b = np.zeros((ng, NU))
        self.Ahat = np.zeros((ng, nz, NK))
        self.bhat = np.zeros((ng, nz))
        PG = self.Psi @ G.T                                           # Psi Gamma^T
        for j in range(ng):
            k_j = int(self.knot[j])
            if self.kind[j] == 0:
                gfull = np.zeros(NX)
                gfull[k_j * nx:(k_j + 1) * nx] = grad[j]
                self.b[j] = self.F_u.T @ gfull                        # b_j = F_u^T grad g_j
                self.bhat[j] = st * PG @ self.F_z.T @ gfull            # b_hat_j
            else:
                self.b[j, k_j * nu:(k_j + 1) * nu] = grad[j, :nu]      # dh_j/du
            Abar = np.zeros((T * nx, NK))
            for k in range(T):
                bjk = self.b[j, k * nu:(k + 1) * nu]
                Abar[k * nx:(k + 1) * nx, k * nu * nx:(k + 1) * nu * nx] = \
                    np.kron(np.eye(nx), bjk[None, :])                  # I (x) b_{j,k}^T
            self.Ahat[j] = st * PG @ np.vstack([Abar, np.zeros((nx, NK))])

        # cost blocks
        W = np.asarray(data["W_K"], float)
        self.Qv = np.zeros((NK, NK))
        for k in range(T):
            s = slice(k * nu * nx, (k + 1) * nu * nx)
            self.Qv[s, s] = 2.0 * np.kron(np.eye(nx), W[k])
        Ru = np.asarray(data["R_u"], float)
        self.Ru = np.zeros((NU, NU))
        for k in range(T):
            self.Ru[k * nu:(k + 1) * nu, k * nu:(k + 1) * nu] = Ru[k]
        self.u_hat = np.asarray(data["u_hat"], float).reshape(-1)
        self.r_trust = float(data["r_trust"])

    # objective and margins
    def objective(self, du, kv):
        u = self.u_hat + du
        return float(u @ self.Ru @ u + 0.5 * kv @ self.Qv @ kv)

    def cone_margin(self, kv, pt):
        return np.array([pt[j] - np.linalg.norm(self.Ahat[j] @ kv + self.bhat[j])
                         for j in range(self.ng)])

    def lin_margin(self, du, p):
        return -(self.g0 + self.b @ du + p)


# ------------------------------------------------------------ (14a) / (5b) QP
class DenseQP:
    """OSQP-form ADMM for  min Q_u(du) + rho/2 ||p - v||^2
       s.t. g_j + b_j^T du + p_j <= 0,  ||F_u du|| <= r_trust   (reading R1).

    x = (du, p), constraint matrix C = [[B, I], [F_u, 0]], P_qp = blkdiag(2R_u,
    rho I), q_qp = [2 R_u u_hat; -rho v].  The x-step solves the full dense
    (P + sigma I + rho_q C^T C) system.  Warm state persists between calls.
    """

    def __init__(self, pb: DenseProblem, rho, rho_q, sigma_q, alpha_q):
        self.pb = pb
        NU, ng, NX = pb.NU, pb.ng, pb.NX
        self.rho, self.rho_q, self.sigma_q, self.alpha_q = rho, rho_q, sigma_q, alpha_q
        self.C = np.zeros((ng + NX, NU + ng))
        self.C[:ng, :NU] = pb.b
        self.C[:ng, NU:] = np.eye(ng)
        self.C[ng:, :NU] = pb.F_u
        self.P = np.zeros((NU + ng, NU + ng))
        self.P[:NU, :NU] = 2.0 * pb.Ru
        self.P[NU:, NU:] = rho * np.eye(ng)
        self.Kmat = self.P + sigma_q * np.eye(NU + ng) + rho_q * self.C.T @ self.C
        self.Kfac = sla.cho_factor(self.Kmat)          # constant across iterations
        self.x = np.zeros(NU + ng)
        self.z = np.zeros(ng + NX)
        self.y = np.zeros(ng + NX)

    def proj(self, w):
        pb = self.pb
        out = w.copy()
        out[:pb.ng] = np.minimum(w[:pb.ng], -pb.g0)
        zb = w[pb.ng:]
        nb = np.linalg.norm(zb)
        if nb > pb.r_trust:
            out[pb.ng:] = zb * (pb.r_trust / nb)
        return out

    def solve(self, v, iters, trace=None):
        """`trace` (a list) receives per iteration the step-1 solution x~, z~ = C x~
        and the new (x, z, y) -- read only by the iterate pins in the tests."""
        pb = self.pb
        NU = pb.NU
        q = np.concatenate([2.0 * pb.Ru @ pb.u_hat, -self.rho * v])
        a, rq = self.alpha_q, self.rho_q
        for _ in range(iters):
            rhs = self.sigma_q * self.x - q + self.C.T @ (rq * self.z - self.y)
            xt = sla.cho_solve(self.Kfac, rhs)
            zt = self.C @ xt
            self.x = a * xt + (1 - a) * self.x
            zh = a * zt + (1 - a) * self.z
            znew = self.proj(zh + self.y / rq)
            self.y = self.y + rq * (zh - znew)
            self.z = znew
            if trace is not None:
                trace.append(dict(xt=xt.copy(), zt=zt.copy(), x=self.x.copy(),
                                  z=self.z.copy(), y=self.y.copy()))
        return self.x[:NU].copy(), self.x[NU:].copy()


# ------------------------------------------------------------- FullADMM (Alg 1)
def gain_operators(Qv, Ahat, bhat, rho):
    """M, q, calM, calMbar of P:1165-1182 as dense matrices."""
    NK = Qv.shape[0]
    H = Qv + rho * sum((A.T @ A for A in Ahat), np.zeros((NK, NK)))
    M = np.linalg.inv(H)
    q = -rho * M @ sum((A.T @ b for A, b in zip(Ahat, bhat)), np.zeros(NK))
    calM = M @ Qv
    calMbar = [rho * M @ A.T for A in Ahat]
    return M, q, calM, calMbar


def fulladmm(pb: DenseProblem, prm, trace=None):
    """Algorithm 1 with (13), (14a), (14b), (16) literally.

    M, q, calM, calMbar from P:1165-1182 are formed as dense matrices.
    """
    rho = prm["rho"]
    ng, NK, NZ = pb.ng, pb.NK, pb.nz
    M, q, calM, calMbar = gain_operators(pb.Qv, pb.Ahat, pb.bhat, rho)

    kv = np.zeros(NK); lam_nu = np.zeros((ng, NZ)); lam_p = np.zeros(ng)
    p = np.zeros(ng); pt_prev = np.zeros(ng)          # Algorithm 1 line 2 (R10)
    nu = np.zeros((ng, NZ)); pt = np.zeros(ng); du = np.zeros(pb.NU)
    qp = DenseQP(pb, rho, prm["rho_qp"], prm["sigma_qp"], prm["alpha_qp"])
    status, it = 1, 0
    r_p = r_d = np.inf
    for l in range(1, prm["max_iter"] + 1):
        it = l
        for j in range(ng):                                             # (13)
            yj = pb.Ahat[j] @ kv + pb.bhat[j] + lam_nu[j]
            pt[j], nu[j] = proj_soc(p[j] + lam_p[j], yj)
        du, p = qp.solve(pt - lam_p, prm["qp_iters"])                   # (14a)
        kv = q + calM @ kv + sum((calMbar[j] @ nu[j] for j in range(ng)), np.zeros(NK))  # (14b)
        lam_p = lam_p + (p - pt)                                        # (16)
        for j in range(ng):
            lam_nu[j] = lam_nu[j] + (pb.Ahat[j] @ kv + pb.bhat[j] - nu[j])
        r_p = float(np.linalg.norm(p - pt))
        r_d = float(rho * np.linalg.norm(pt - pt_prev))
        pt_prev = pt.copy()
        if trace is not None:
            trace.append(dict(l=l, kv=kv.copy(), pt=pt.copy(), p=p.copy(), du=du.copy(),
                              lam_p=lam_p.copy(), nu=nu.copy(), lam_nu=lam_nu.copy(),
                              r_p=r_p, r_d=r_d))
        if (not prm["fixed_iters"]) and l % prm["check_every"] == 0 \
                and r_p <= prm["eps_p"] and r_d <= prm["eps_d"]:
            status = 0
            break
    return dict(kv=kv, du=du, p=p, p_tilde=pt, lam_p=lam_p, nu=nu, lam_nu=lam_nu,
                iters=it, status=status, r_p=r_p, r_d=r_d,
                objective=pb.objective(du, kv), margin_cone=pb.cone_margin(kv, pt),
                margin_lin=pb.lin_margin(du, p))


# ------------------------------------------------------- DR on (7) / NRTO-ADMM
class DenseDR:
    """Relaxed DR (11a)-(11c) on the standard form (8).

    The affine prox solves the full K_KKT system of P:950-962 densely.
    State xi~ = (chi~, s~) persists across calls (warm start).
    """

    def __init__(self, pb: DenseProblem, rho, alpha, sigma, r_s):
        self.pb = pb
        ng, NK, NX = pb.ng, pb.NK, pb.nz           # cone rows have the n_z of zeta = Gamma z
        self.m = ng * (1 + NX)
        n = NK + ng
        self.rho, self.alpha = rho, alpha
        self.P = np.zeros((n, n))
        self.P[:NK, :NK] = pb.Qv
        self.P[NK:, NK:] = rho * np.eye(ng)
        self.A = np.zeros((self.m, n))
        self.bvec = np.zeros(self.m)
        for j in range(ng):                      # A_j, b_j of P:909-926
            r0 = j * (1 + NX)
            self.A[r0, NK + j] = -1.0
            self.A[r0 + 1:r0 + 1 + NX, :NK] = -pb.Ahat[j]
            self.bvec[r0 + 1:r0 + 1 + NX] = pb.bhat[j]
        self.Rchi = sigma * np.eye(n)
        self.Rs = r_s * np.eye(self.m)
        self.Kkkt = np.block([[self.P + self.Rchi, self.A.T],
                              [self.A, -np.linalg.inv(self.Rs)]])
        self.Kfac = sla.lu_factor(self.Kkkt)           # factor once, reuse solves
        self.chit = np.zeros(n)
        self.st = np.zeros(self.m)

    def proj_K(self, s):
        out = s.copy()
        NX = self.pb.nz
        for j in range(self.pb.ng):
            r0 = j * (1 + NX)
            t, y = proj_soc(s[r0], s[r0 + 1:r0 + 1 + NX])
            out[r0] = t
            out[r0 + 1:r0 + 1 + NX] = y
        return out

    def run(self, qvec, iters, eps_dr, fixed):
        """Returns (chi, s, r_dr, iterations)."""
        n = self.P.shape[0]
        chi = s = None
        r_dr = np.inf
        it = 0
        for l in range(1, iters + 1):
            it = l
            rhs = np.concatenate([self.Rchi @ self.chit - qvec, self.bvec - self.st])
            sol = sla.lu_solve(self.Kfac, rhs)                         # (10)
            chi, yv = sol[:n], sol[n:]
            s = self.st - np.linalg.solve(self.Rs, yv)
            chi_ref = 2 * chi - self.chit                              # (11b)
            s_ref = 2 * s - self.st
            st_new = self.st + self.alpha * (self.proj_K(s_ref) - s)   # (11c)
            self.chit = self.chit + self.alpha * (chi_ref - chi)
            r_dr = float(np.linalg.norm(st_new - self.st))
            self.st = st_new
            if (not fixed) and r_dr <= eps_dr:
                break
        return chi, s, r_dr, it


def nrto_admm_dr(pb: DenseProblem, prm, trace=None):
    """NRTO inner ADMM (5a)-(5c) with (5a) solved by DR on (7)."""
    rho = prm["rho_admm"]
    ng, NK = pb.ng, pb.NK
    dr = DenseDR(pb, rho, prm["alpha_dr"], prm["sigma_dr"], prm["r_s"])
    qp = DenseQP(pb, rho, prm["rho_qp"], prm["sigma_qp"], prm["alpha_qp"])
    p = np.zeros(ng); lam = np.zeros(ng); pt_prev = np.zeros(ng)
    kv = np.zeros(NK); pt = np.zeros(ng); du = np.zeros(pb.NU)
    status, it = 1, 0
    r_p = r_d = np.inf
    dr_iters = 0
    for l in range(1, prm["max_admm_iter"] + 1):
        it = l
        qvec = np.concatenate([np.zeros(NK), -(rho * p + lam)])      # q of (8)
        chi, s, r_dr, ndr = dr.run(qvec, prm["max_dr_iter"], prm["eps_dr"], prm["fixed_iters"])
        dr_iters += ndr
        kv, pt = chi[:NK].copy(), chi[NK:].copy()                    # (5a), R9
        du, p = qp.solve(pt - lam / rho, prm["qp_iters"])            # (5b)
        lam = lam + rho * (p - pt)                                   # (5c), R4
        r_p = float(np.linalg.norm(p - pt))
        r_d = float(rho * np.linalg.norm(pt - pt_prev))
        pt_prev = pt.copy()
        if trace is not None:
            trace.append(dict(l=l, kv=kv.copy(), pt=pt.copy(), p=p.copy(), du=du.copy(),
                              lam=lam.copy(), st=dr.st.copy(), chit=dr.chit.copy(),
                              r_p=r_p, r_d=r_d, r_dr=r_dr))
        if (not prm["fixed_iters"]) and l % prm["check_every"] == 0 \
                and r_p <= prm["eps_p"] and r_d <= prm["eps_d"]:
            status = 0
            break
    return dict(kv=kv, du=du, p=p, p_tilde=pt, lam_p=lam, iters=it, status=status,
                r_p=r_p, r_d=r_d, dr_iters=dr_iters, st=dr.st, chit=dr.chit,
                objective=pb.objective(du, kv), margin_cone=pb.cone_margin(kv, pt),
                margin_lin=pb.lin_margin(du, p))
