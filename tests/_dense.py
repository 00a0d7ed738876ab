"""Test-only dense linear algebra restating the paper's *definitions* (not the oracle's
algorithms): the stacked Jacobian of Eq. linearized_residual, its normal equations
(P:160-184), the explicit Schur complement and a brute-force least-squares solve.
Built from the oracle's per-observation Jacobians, which are themselves pinned to central finite
differences and golden projection values (tests/test_oracle_model.py)."""
import numpy as np


def stacked(o):
    """Scaled J = [J_p S_p | J_l S_l] (2 n_obs x (9 n_p + 3 n_l)), r, D^2 (CSR row order)."""
    r, Jc, Jl = o.linearization()
    sp, Dp2, sl, Dl2 = o.scaling()
    n_obs, n_p, n_l = o.n_obs, o.n_p, o.n_l
    lm = np.repeat(np.arange(n_l), np.diff(o.lm_ptr))
    cam = o.csr_cam
    N = 9 * n_p + 3 * n_l
    J = np.zeros((2 * n_obs, N))
    rows = np.arange(2 * n_obs).reshape(n_obs, 2)
    for q in range(9):
        J[rows, (9 * cam + q)[:, None]] = Jc[:, :, q] * sp[9 * cam + q][:, None]
    for q in range(3):
        J[rows, (9 * n_p + 3 * lm + q)[:, None]] = Jl[:, :, q] * sl[3 * lm + q][:, None]
    return J, r.reshape(-1), np.concatenate([Dp2, Dl2])


def schur(J, r, D2, lam, n_p):
    """Damped explicit SC (P:197-198 with P:277): returns H~, b~ and the blocks for back-sub."""
    Np = 9 * n_p
    H = J.T @ J + lam * np.diag(D2)
    b = J.T @ r
    Hpp, Hpl, Hll = H[:Np, :Np], H[:Np, Np:], H[Np:, Np:]
    bp, bl = b[:Np], b[Np:]
    X = np.linalg.solve(Hll, np.concatenate([Hpl.T, bl[:, None]], 1))
    Ht = Hpp - Hpl @ X[:, :-1]
    bt = bp - Hpl @ X[:, -1]
    return Ht, bt, Hll, Hpl, bl


def brute_force_step(J, r, D2, lam):
    """argmin |[r;0] + [J; sqrt(lam) D] dx|^2 (Eq. linearized_residual) by dense least squares."""
    A = np.vstack([J, np.sqrt(lam) * np.diag(np.sqrt(D2))])
    rhs = -np.concatenate([r, np.zeros(J.shape[1])])
    dx, *_ = np.linalg.lstsq(A, rhs, rcond=None)
    return dx


def relf(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
