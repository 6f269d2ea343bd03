"""Inner-solver hyper-parameters (oracle side).

Defaults follow the paper's tables where it gives a value and DESIGN.md's
readings (R2-R11, R18) where it does not:
  rho = 10           FullADMM penalty
  rho_admm = 40      NRTO-ADMM penalty (DR)      P:1304 (R3)
  alpha_dr = 0.9     DR relaxation in (0,1)      P:322 (R7)
  sigma_dr = 1e-6    R_chi = sigma I             P:341 (R7)
  r_s = 1            R_s = r_s I                 P:341 (R7)
  eps_p = eps_d = 1e-3                           P:1345, P:1439 (R6)
  eps_dr = 1e-4      absolute ||s~^l - s~^(l-1)||  P:1339 (R8)
  max_iter 40 (50 for Franka c3/c5)              P:1345, P:1439 (R18)
  max_admm_iter 40, max_dr_iter 100
  (14a) QP (R1): OSQP-form ADMM, rho_qp=1, sigma_qp=1e-6, alpha_qp=1.6,
  qp_iters=10 warm-started.
"""
from __future__ import annotations

DEFAULTS = dict(
    rho=10.0, rho_admm=40.0, alpha_dr=0.9, sigma_dr=1e-6, r_s=1.0,
    eps_p=1e-3, eps_d=1e-3, eps_dr=1e-4,
    rho_qp=1.0, sigma_qp=1e-6, alpha_qp=1.6,
    max_iter=40, max_admm_iter=40, max_dr_iter=100, qp_iters=10,
    check_every=1, fixed_iters=0,
)


def make_params(**kw):
    p = dict(DEFAULTS)
    for k, v in kw.items():
        if k not in p:
            raise KeyError(k)
        p[k] = v
    return p
