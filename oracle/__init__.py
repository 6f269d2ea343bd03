"""CPU ORACLE for the NRTO inner solve -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import or execute anything under `oracle/`.
The product path (paper_2603_02642_b200/, libnrto.so) never imports it and
shares no code with it; the two meet only on the arrays produced by `gen/`.

Tiers
-----
* `oracle.soc`        closed-form SOC projection, SM Eq.(18).
* `oracle.dense`      literal dense definitions for tiny instances: F_u, F_zeta,
                      Psi (Psi^T Psi = S^-1), A_hat_j, b_hat_j, Q_v
                      (P:835-839), M, q, calM, calMbar, K_KKT
                      (P:950-962), Algorithm 1, relaxed DR,
                      NRTO-ADMM (5a-c).  Any S, Gamma=I.
* `oracle.structured` the same algorithms on the ragged per-timestep structure
                      (Gamma = I, S block diagonal), fast enough
                      for the c1-c3 configs; pinned to `oracle.dense` on tiny
                      cases.
* `oracle.ip`         brute-force log-barrier interior point for Problem 2
                      (P:184-206), the whole-loop pin.

All arithmetic is float64 (the paper states no precision; R17).
Functions without an independent pin say "parity unpinned" in their
docstring; see DESIGN.md §4 for the list.
"""
