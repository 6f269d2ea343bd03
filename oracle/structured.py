"""Structured oracle: the same algorithms as oracle.dense on ragged per-block data.

Workload assumption: Gamma = I, S = blkdiag(S_0, ..., S_T), so Psi
is block diagonal and Psi_k^T Psi_k = S_k^{-1}.  Then, per SM §I:

  * zeta block k is d_{k-1} (k = 0..T, d_{-1} = d_bar_0) and K_k multiplies it;
  * b_j = F_u^T grad g_j splits into blocks b_{j,k} = B_k^T c_{j,k+1} (k < k_j),
    where c_{j,k} = Phi(k_j, k)^T grad g_j is block k of F_zeta^T grad g_j
    (c_{j,k_j} = grad g_j, c_{j,k} = A_k^T c_{j,k+1}), zero for k >= k_j;
  * block k of A_hat_j k_v = sqrt(tau) Psi_k (I (x) b_{j,k}^T) vec(K_k)
                           = sqrt(tau) Psi_k K_k^T b_{j,k}
    and block k of b_hat_j = sqrt(tau) Psi_k c_{j,k};  blocks k > k_j are 0.
  * control rows (reading R14): b_{j,k} = h'_j at their own step k only, b_hat = 0.

So cone j is stored raggedly: state rows hold blocks 0..k_j ((k_j+1) n_x
doubles), control rows hold block k (n_x doubles).  `ragged_layout` gives
the offsets (include/nrto.h, nrto_layout).  Nothing else is restructured:
each algorithm step below is the same step as in oracle.dense, in the same
order, evaluated block by block.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .soc import proj_soc_scale


def ragged_layout(shape):
    """Offsets of each cone's row in the flat ragged arrays (length E)."""
    knot = np.asarray(shape.cone_knot, np.int64)
    kind = np.asarray(shape.cone_kind)
    L = np.where(kind == 0, (knot + 1) * shape.n_x, shape.n_x)
    off = np.zeros(shape.n_g + 1, np.int64)
    off[1:] = np.cumsum(L)
    return off


def vec_cm(K):
    """Column-major vec of a (.., n_u, n_x) matrix stack."""
    K = np.asarray(K)
    return np.swapaxes(K, -1, -2).reshape(K.shape[:-2] + (-1,))


def unvec_cm(v, nu, nx):
    v = np.asarray(v)
    return np.swapaxes(v.reshape(v.shape[:-1] + (nx, nu)), -1, -2)


class StructuredProblem:
    """Per-SL-iteration constants on the ragged structure (setup S0)."""

    def __init__(self, shape, data):
        nx, nu, T, ng = shape.n_x, shape.n_u, shape.T, shape.n_g
        self.nx, self.nu, self.T, self.ng = nx, nu, T, ng
        self.NK = T * nu * nx
        self.knot = np.asarray(shape.cone_knot, np.int64)
        self.kind = np.asarray(shape.cone_kind, np.int64)
        self.A = np.asarray(data["A"], float)
        self.B = np.asarray(data["B"], float)
        self.grad = np.asarray(data["grad"], float)
        self.g0 = np.asarray(data["g0"], float)
        self.Psi = np.asarray(data["Psi"], float)
        self.tau = float(data["tau"])
        self.st = np.sqrt(self.tau)
        self.W = np.asarray(data["W_K"], float)
        self.Ru = np.asarray(data["R_u"], float)
        self.u_hat = np.asarray(data["u_hat"], float)
        self.r_trust = float(data["r_trust"])
        self.off = ragged_layout(shape)
        self.E = int(self.off[-1])
        state = self.kind == 0

        # cones having a block at k, and where that block sits in the ragged row
        self.at = []
        self.pos = []
        for k in range(T + 1):
            js = np.nonzero((state & (self.knot >= k)) | (~state & (self.knot == k)))[0]
            self.at.append(js)
            self.pos.append(self.off[js] + np.where(state[js], k, 0) * nx)
        # costate sweeps: c_{j,k}, b_{j,k}, b_hat_{j,k}, per cone
        self.b_at = [np.zeros((len(self.at[k]), nu)) for k in range(T)]
        self.bh_at = [np.zeros((len(self.at[k]), nx)) for k in range(T + 1)]
        where = [dict((int(j), r) for r, j in enumerate(self.at[k])) for k in range(T + 1)]
        for j in range(ng):
            kj = int(self.knot[j])
            if state[j]:
                c = self.grad[j].copy()                     # c_{j,k_j} = grad g_j
                self.bh_at[kj][where[kj][j]] = self.st * self.Psi[kj] @ c
                for k in range(kj - 1, -1, -1):
                    self.b_at[k][where[k][j]] = self.B[k].T @ c  # b_{j,k} = B_k^T c_{j,k+1}
                    c = self.A[k].T @ c                      # c_{j,k} = A_k^T c_{j,k+1}
                    self.bh_at[k][where[k][j]] = self.st * self.Psi[k] @ c
            else:
                self.b_at[kj][where[kj][j]] = self.grad[j, :nu]
        # linear rows of g^lin,1 (R1): state rows act through x_{k_j}, control rows through u_k
        self.state_at = [np.nonzero(state & (self.knot == k))[0] for k in range(T + 1)]
        self.ctrl_at = [np.nonzero(~state & (self.knot == k))[0] for k in range(T)]

    # ---- A_hat / A_hat^T in block form ---------------------------------------
    def fwd(self, kv, with_bhat=True):
        """a_j = A_hat_j k_v (+ b_hat_j) as a flat ragged array (length E)."""
        K = unvec_cm(kv.reshape(self.T, -1), self.nu, self.nx)        # [T, nu, nx]
        out = np.zeros(self.E)
        idx = np.arange(self.nx)
        for k in range(self.T + 1):
            if len(self.at[k]) == 0:
                continue
            blk = np.zeros((len(self.at[k]), self.nx))
            if k < self.T:
                # sqrt(tau) Psi_k K_k^T b_{j,k}, written row-wise
                blk += self.st * (self.b_at[k] @ K[k]) @ self.Psi[k].T
            if with_bhat:
                blk += self.bh_at[k]
            out[self.pos[k][:, None] + idx[None, :]] = blk
        return out

    def adj(self, e):
        """sum_j A_hat_j^T e_j for a flat ragged e; returns k_v-shaped vector."""
        G = np.zeros((self.T, self.nu, self.nx))
        idx = np.arange(self.nx)
        for k in range(self.T):
            if len(self.at[k]) == 0:
                continue
            Ek = e[self.pos[k][:, None] + idx[None, :]]                  # rows e_{j,k}
            # block k = sqrt(tau) sum_j (I (x) b_{j,k}) Psi_k^T e_{j,k}
            #         = vec( sqrt(tau) sum_j b_{j,k} (Psi_k^T e_{j,k})^T )
            G[k] = self.st * self.b_at[k].T @ (Ek @ self.Psi[k])
        return vec_cm(G).reshape(-1)

    def bhat_flat(self):
        return self.fwd(np.zeros(self.NK), with_bhat=True)

    def gram_blocks(self, coef, shift):
        """Diagonal blocks of Q_v + shift*I + coef * sum_j A_hat_j^T A_hat_j.

        Formed by explicit summation over the rows of every A_hat_j block
        (P:1167); block (k,k) only, since A_hat_j is block diagonal in k.
        """
        nx, nu = self.nx, self.nu
        H = np.empty((self.T, nu * nx, nu * nx))
        I = np.eye(nx)
        for k in range(self.T):
            bk = self.b_at[k]
            Abar = np.einsum("ab,jm->jabm", I, bk).reshape(len(bk), nx, nx * nu)  # I (x) b^T
            G = (self.st * np.einsum("ab,jbc->jac", self.Psi[k], Abar)).reshape(-1, nx * nu)
            H[k] = 2.0 * np.kron(I, self.W[k]) + shift * np.eye(nx * nu) + coef * (G.T @ G)
        return H

    # ---- reported quantities -----------------------------------
    def cone_norms(self, a):
        return np.sqrt(np.add.reduceat(a * a, self.off[:-1]))

    def objective(self, du, kv):
        u = self.u_hat + du.reshape(self.T, self.nu)
        J = float(np.einsum("ki,kij,kj->", u, self.Ru, u))
        K = unvec_cm(kv.reshape(self.T, -1), self.nu, self.nx)
        J += float(sum(np.sum(K[k] * (self.W[k] @ K[k])) for k in range(self.T)))
        return J

    def row_dot(self, du, dx):
        """(B du)_j: grad_j^T dx_{k_j} for state rows, h'_j^T du_k for control rows."""
        out = np.empty(self.ng)
        st = self.kind == 0
        out[st] = np.einsum("ji,ji->j", self.grad[st], dx[self.knot[st]])
        ct = ~st
        out[ct] = np.einsum("ji,ji->j", self.grad[ct, :self.nu], du[self.knot[ct]])
        return out

    def lin_margin(self, du, p):
        dx = self.rollout(du)
        return -(self.g0 + self.row_dot(du.reshape(self.T, self.nu), dx) + p)

    def rollout(self, du):
        du = du.reshape(self.T, self.nu)
        dx = np.zeros((self.T + 1, self.nx))
        for k in range(self.T):
            dx[k + 1] = self.A[k] @ dx[k] + self.B[k] @ du[k]
        return dx


class RiccatiQP:
    """(14a)/(5b) QP by OSQP-form ADMM (reading R1) with a Riccati x-step.

    Same iteration as oracle.dense.DenseQP.  Eliminating p from the x-step
    system leaves (R~ + F_u^T Q~ F_u) du = r_u + F_u^T r_x with
      R~_k = 2 R_u,k + sigma I + c sum_{ctrl j@k} h'_j h'_j^T,
      Q~_k = rho_q I + c sum_{state j@k} grad_j grad_j^T   (k = 1..T),
      c = rho_q (rho+sigma)/(rho+sigma+rho_q),
    an LQR normal matrix, solved by a backward Riccati sweep and a
    forward rollout.  Products with B and F_u go through the dynamics.
    """

    def __init__(self, sp: StructuredProblem, rho, rho_q, sigma_q, alpha_q):
        self.sp = sp
        T, nx, nu, ng = sp.T, sp.nx, sp.nu, sp.ng
        self.rho, self.rq, self.sq, self.aq = rho, rho_q, sigma_q, alpha_q
        self.den = rho + sigma_q + rho_q
        self.beta = rho_q / self.den
        c = rho_q * (rho + sigma_q) / self.den
        Qt = np.zeros((T + 1, nx, nx))
        for k in range(1, T + 1):
            G = sp.grad[sp.state_at[k]]
            Qt[k] = rho_q * np.eye(nx) + c * G.T @ G
        Rt = np.zeros((T, nu, nu))
        for k in range(T):
            H = sp.grad[sp.ctrl_at[k], :nu]
            Rt[k] = 2.0 * sp.Ru[k] + sigma_q * np.eye(nu) + c * H.T @ H
        self.Kf = np.zeros((T, nu, nx))
        self.Hc = []
        P = Qt[T]
        for k in range(T - 1, -1, -1):
            A, B = sp.A[k], sp.B[k]
            Huu = Rt[k] + B.T @ P @ B
            Hux = B.T @ P @ A
            cf = sla.cho_factor(Huu, lower=True)
            self.Kf[k] = sla.cho_solve(cf, Hux)
            self.Hc.insert(0, cf)
            P = Qt[k] + A.T @ P @ A - Hux.T @ self.Kf[k]
        self.du = np.zeros((T, nu)); self.p = np.zeros(ng)
        self.zl = np.zeros(ng); self.zb = np.zeros((T + 1, nx))
        self.yl = np.zeros(ng); self.yb = np.zeros((T + 1, nx))

    def lqr(self, ru, rx):
        sp = self.sp
        T = sp.T
        kff = np.zeros((T, sp.nu))
        s = rx[T].copy()
        for k in range(T - 1, -1, -1):
            gu = ru[k] + sp.B[k].T @ s
            kff[k] = sla.cho_solve(self.Hc[k], gu)
            s = rx[k] + sp.A[k].T @ s - self.Kf[k].T @ gu
        du = np.zeros((T, sp.nu)); dx = np.zeros((T + 1, sp.nx))
        for k in range(T):
            du[k] = kff[k] - self.Kf[k] @ dx[k]
            dx[k + 1] = sp.A[k] @ dx[k] + sp.B[k] @ du[k]
        return du, dx

    def solve(self, v, iters, trace=None):
        """`trace` (a list) receives per iteration x~ = (du~, p~'), z~ = (B du~ + p~',
        dx~) and the new (x, z, y), flattened in DenseQP's order (x = (du, p),
        z = (z_lin, z_ball)) -- read only by the iterate pins in the tests."""
        sp = self.sp
        T = sp.T
        st = sp.kind == 0
        rq, sq, aq = self.rq, self.sq, self.aq
        for _ in range(iters):
            rp = sq * self.p + self.rho * v + rq * self.zl - self.yl
            w = rq * self.zl - self.yl - self.beta * rp
            rx = rq * self.zb - self.yb
            np.add.at(rx, sp.knot[st], sp.grad[st] * w[st, None])
            ru = sq * self.du - 2.0 * np.einsum("kij,kj->ki", sp.Ru, sp.u_hat)
            np.add.at(ru, sp.knot[~st], sp.grad[~st, :sp.nu] * w[~st, None])
            rx[0] = 0.0
            dut, dxt = self.lqr(ru, rx)
            Bdu = sp.row_dot(dut, dxt)
            pt = (rp - rq * Bdu) / self.den
            ztl = Bdu + pt
            self.du = aq * dut + (1 - aq) * self.du
            self.p = aq * pt + (1 - aq) * self.p
            zhl = aq * ztl + (1 - aq) * self.zl
            zhb = aq * dxt + (1 - aq) * self.zb
            znl = np.minimum(zhl + self.yl / rq, -sp.g0)
            wb = zhb + self.yb / rq
            nb = np.linalg.norm(wb)
            znb = wb * (sp.r_trust / nb) if nb > sp.r_trust else wb
            self.yl = self.yl + rq * (zhl - znl)
            self.yb = self.yb + rq * (zhb - znb)
            self.zl, self.zb = znl, znb
            if trace is not None:
                trace.append(dict(xt=np.concatenate([dut.reshape(-1), pt]),
                                  zt=np.concatenate([ztl, dxt.reshape(-1)]),
                                  x=np.concatenate([self.du.reshape(-1), self.p]),
                                  z=np.concatenate([self.zl, self.zb.reshape(-1)]),
                                  y=np.concatenate([self.yl, self.yb.reshape(-1)])))
        return self.du.reshape(-1).copy(), self.p.copy()


# --------------------------------------------------------------- FullADMM
def fulladmm(sp: StructuredProblem, prm, trace=None, hist=False):
    """Algorithm 1: (13) -> (14a) -> (14b) -> (16) -> r_p, r_d."""
    rho = prm["rho"]
    T, nu, nx, ng = sp.T, sp.nu, sp.nx, sp.ng
    H = sp.gram_blocks(rho, 0.0)                       # M^{-1} = Q_v + rho sum A^T A
    cf = [sla.cho_factor(H[k], lower=True) for k in range(T)]
    bh = sp.bhat_flat()
    Qv = lambda kv: vec_cm(2.0 * np.einsum("kab,kbc->kac", sp.W,
                                           unvec_cm(kv.reshape(T, -1), nu, nx))).reshape(-1)
    kv = np.zeros(sp.NK); lam_nu = np.zeros(sp.E); lam_p = np.zeros(ng)
    p = np.zeros(ng); pt_prev = np.zeros(ng)
    nu_v = np.zeros(sp.E); pt = np.zeros(ng); du = np.zeros(T * nu)
    qp = RiccatiQP(sp, rho, prm["rho_qp"], prm["sigma_qp"], prm["alpha_qp"])
    status, it = 1, 0
    r_p = r_d = np.inf
    H_hist = []
    cases = []
    for l in range(1, prm["max_iter"] + 1):
        it = l
        y = sp.fwd(kv) + lam_nu                                      # (13)
        a = sp.cone_norms(y)
        pt, s, case = proj_soc_scale(p + lam_p, a)
        nu_v = y * np.repeat(s, np.diff(sp.off))
        cases.append(np.bincount(case, minlength=4)[1:])
        du, p = qp.solve(pt - lam_p, prm["qp_iters"])                 # (14a)
        rhs = Qv(kv) + rho * sp.adj(nu_v - bh)                        # (14b): M(Q_v k + rho sum A^T(nu-b_hat))
        kv = np.concatenate([sla.cho_solve(cf[k], rhs[k * nu * nx:(k + 1) * nu * nx])
                             for k in range(T)])
        lam_p = lam_p + (p - pt)                                      # (16)
        lam_nu = lam_nu + (sp.fwd(kv) - nu_v)
        r_p = float(np.linalg.norm(p - pt))
        r_d = float(rho * np.linalg.norm(pt - pt_prev))
        pt_prev = pt.copy()
        H_hist.append((r_p, r_d, 0.0))
        if trace is not None:
            trace.append(dict(l=l, kv=kv.copy(), pt=pt.copy(), p=p.copy(), du=du.copy(),
                              lam_p=lam_p.copy(), nu=nu_v.copy(), lam_nu=lam_nu.copy(),
                              r_p=r_p, r_d=r_d))
        if (not prm["fixed_iters"]) and l % prm["check_every"] == 0 \
                and r_p <= prm["eps_p"] and r_d <= prm["eps_d"]:
            status = 0
            break
    a_fin = sp.cone_norms(sp.fwd(kv))
    return dict(kv=kv, du=du, p=p, p_tilde=pt, lam_p=lam_p, nu=nu_v, lam_nu=lam_nu,
                iters=it, status=status, r_p=r_p, r_d=r_d,
                objective=sp.objective(du, kv), margin_cone=pt - a_fin,
                margin_lin=sp.lin_margin(du, p), hist=np.array(H_hist),
                cases=np.array(cases))


# ----------------------------------------------------- NRTO-ADMM with DR
def nrto_admm_dr(sp: StructuredProblem, prm, trace=None):
    """(5a)-(5c); (5a) by relaxed DR (11a)-(11c).

    The affine prox (10) is solved through its Schur complement: with
    R_chi = sigma I and R_s = r_s I the K_KKT system of P:950-962 reduces to
      (Q_v + sigma I + r_s sum A_hat^T A_hat) k = sigma k~ + r_s sum A_hat^T(eta~ - b_hat)
      (rho + sigma + r_s) pi_j = sigma pi~_j + rho p_j + lambda_j + r_s t~_j
    and s = b - A chi = (pi, A_hat k + b_hat) (pinned against the
    dense K_KKT solve in tests/test_oracle_structured.py).
    """
    rho, alpha, sig, rs = prm["rho_admm"], prm["alpha_dr"], prm["sigma_dr"], prm["r_s"]
    T, nu, nx, ng = sp.T, sp.nu, sp.nx, sp.ng
    H = sp.gram_blocks(rs, sig)
    cf = [sla.cho_factor(H[k], lower=True) for k in range(T)]
    bh = sp.bhat_flat()
    seg = np.diff(sp.off)
    kt = np.zeros(sp.NK); pit = np.zeros(ng)          # chi~ = (k~, pi~)
    tt = np.zeros(ng); et = np.zeros(sp.E)            # s~ = (t~, eta~)
    p = np.zeros(ng); lam = np.zeros(ng); pt_prev = np.zeros(ng)
    kv = np.zeros(sp.NK); pi = np.zeros(ng); du = np.zeros(T * nu)
    qp = RiccatiQP(sp, rho, prm["rho_qp"], prm["sigma_qp"], prm["alpha_qp"])
    status, it, dr_total = 1, 0, 0
    r_p = r_d = r_dr = np.inf
    for l in range(1, prm["max_admm_iter"] + 1):
        it = l
        for m in range(1, prm["max_dr_iter"] + 1):
            dr_total += 1
            rhs = sig * kt + rs * sp.adj(et - bh)                        # (10) via Schur
            kv = np.concatenate([sla.cho_solve(cf[k], rhs[k * nu * nx:(k + 1) * nu * nx])
                                 for k in range(T)])
            pi = (sig * pit + rho * p + lam + rs * tt) / (rho + sig + rs)
            a = sp.fwd(kv)                                               # s = (pi, a)
            tr = 2 * pi - tt                                             # (11b)
            er = 2 * a - et
            tpi, sc, _ = proj_soc_scale(tr, sp.cone_norms(er))
            tt_new = tt + alpha * (tpi - pi)                             # (11c)
            et_new = et + alpha * (er * np.repeat(sc, seg) - a)
            kt = kt + alpha * (kv - kt)
            pit = pit + alpha * (pi - pit)
            r_dr = float(np.sqrt(np.sum((tt_new - tt) ** 2) + np.sum((et_new - et) ** 2)))
            tt, et = tt_new, et_new
            if (not prm["fixed_iters"]) and r_dr <= prm["eps_dr"]:
                break
        pt = pi.copy()                                                   # R9
        du, p = qp.solve(pt - lam / rho, prm["qp_iters"])               # (5b)
        lam = lam + rho * (p - pt)                                       # (5c)
        r_p = float(np.linalg.norm(p - pt))
        r_d = float(rho * np.linalg.norm(pt - pt_prev))
        pt_prev = pt.copy()
        if trace is not None:
            trace.append(dict(l=l, kv=kv.copy(), pt=pt.copy(), p=p.copy(), du=du.copy(),
                              lam=lam.copy(), tt=tt.copy(), et=et.copy(), kt=kt.copy(),
                              pit=pit.copy(), r_p=r_p, r_d=r_d, r_dr=r_dr))
        if (not prm["fixed_iters"]) and l % prm["check_every"] == 0 \
                and r_p <= prm["eps_p"] and r_d <= prm["eps_d"]:
            status = 0
            break
    a_fin = sp.cone_norms(sp.fwd(kv))
    return dict(kv=kv, du=du, p=p, p_tilde=pt, lam_p=lam, iters=it, status=status,
                r_p=r_p, r_d=r_d, r_dr=r_dr, dr_iters=dr_total, tt=tt, et=et, kt=kt, pit=pit,
                objective=sp.objective(du, kv), margin_cone=pt - a_fin,
                margin_lin=sp.lin_margin(du, p))
