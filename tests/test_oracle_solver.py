"""Pins for the oracle's marginalization, damping, reduced system, PCG, back-substitution and LM
against what the paper and the mathematics fix (P:92-119 QR identities, P:243-277 SC equivalence,
P:305-320 damping, P:148-155 brute-force least squares, P:502 positive definiteness)."""
import numpy as np
import pytest

import oracle
from paper_2103_01843_b200 import synth

from _dense import brute_force_step, relf, schur, stacked


def _small(seed, **kw):
    return synth.make_random_small(seed, **kw)


def test_block_shape_and_layout():
    """(2k+3) x (9k+4) per landmark (k=2 -> 7 x 22); Fig. 2b layout."""
    p = _small(0, n_p=4, n_l=8, kmin=2, kmax=4)
    o = oracle.Oracle(p)
    o.linearize()
    r, Jc, Jl = o.linearization()
    sp, _, sl, _ = o.scaling()
    for j in range(o.n_l):
        k = o.track_length(j)
        B = o.block(j)
        assert B.shape == (2 * k + 3, 9 * k + 4)
        if k == 2:
            assert B.shape == (7, 22)
        o0 = o.lm_ptr[j]
        for i in range(k):
            cam = o.csr_cam[o0 + i]
            np.testing.assert_allclose(B[2 * i:2 * i + 2, 9 * i:9 * i + 9], Jc[o0 + i] * sp[9 * cam:9 * cam + 9])
            np.testing.assert_allclose(B[2 * i:2 * i + 2, 9 * k:9 * k + 3], Jl[o0 + i] * sl[3 * j:3 * j + 3])
            np.testing.assert_allclose(B[2 * i:2 * i + 2, 9 * k + 3], r[o0 + i])
        assert not B[2 * k:].any()


def test_column_scaling_definition():
    """s = 1/(1 + |c|) over full-Jacobian columns (C7; norm 3 -> 0.25); D^2 = clamp(|c|^2 s^2)."""
    p = _small(1)
    o = oracle.Oracle(p)
    o.linearize()
    r, Jc, Jl = o.linearization()
    sp, Dp2, sl, Dl2 = o.scaling()
    lm = np.repeat(np.arange(o.n_l), np.diff(o.lm_ptr))
    cn = np.zeros(9 * o.n_p)
    np.add.at(cn, (9 * o.csr_cam[:, None] + np.arange(9)).ravel(), (Jc ** 2).sum(1).ravel())
    ln = np.zeros(3 * o.n_l)
    np.add.at(ln, (3 * lm[:, None] + np.arange(3)).ravel(), (Jl ** 2).sum(1).ravel())
    np.testing.assert_allclose(sp, 1 / (1 + np.sqrt(cn)), rtol=1e-13)
    np.testing.assert_allclose(sl, 1 / (1 + np.sqrt(ln)), rtol=1e-13)
    np.testing.assert_allclose(Dp2, np.clip(cn * sp ** 2, 1e-6, 1e32), rtol=1e-13)
    np.testing.assert_allclose(Dl2, np.clip(ln * sl ** 2, 1e-6, 1e32), rtol=1e-13)


@pytest.mark.parametrize("seed", range(6))
def test_qr_identities(seed):
    """Q2^T J_l = 0, Q orthogonal => block Gram matrix B^T B preserved (column
    norms and |r|^2 = |Q1^T r|^2 + |Q2^T r|^2), R1^T R1 = J_l^T J_l, 6k-6 rotations."""
    p = _small(seed, n_p=6, n_l=10, kmin=2, kmax=6)
    o = oracle.Oracle(p)
    o.linearize()
    before = [o.block(j) for j in range(o.n_l)]
    o.marginalize()
    for j in range(o.n_l):
        k = o.track_length(j)
        B0, B = before[j], o.block(j)
        Jl0 = B0[:2 * k, 9 * k:9 * k + 3]
        assert np.all(B[3:2 * k, 9 * k:9 * k + 3] == 0.0)
        R1 = B[:3, 9 * k:9 * k + 3]
        assert np.allclose(np.tril(R1, -1), 0)
        np.testing.assert_allclose(R1.T @ R1, Jl0.T @ Jl0, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(B.T @ B, B0.T @ B0, rtol=1e-11, atol=1e-12)
        np.testing.assert_allclose(np.sum(B[:3, -1] ** 2) + np.sum(B[3:2 * k, -1] ** 2),
                                   np.sum(B0[:2 * k, -1] ** 2), rtol=1e-12)


@pytest.mark.parametrize("lam", [0.0, 1e-4, 1.0, 1e3])
def test_damping(lam):
    """Damping: R^1^T R^1 = J_l^T J_l + lam D_l^2; equals a from-scratch orthogonal
    factorization of the damped stack (Gram matrix of [B; sqrt(lam) D_l rows]); undo restores the
    marginalized block (Fig. 3c); lam = 0 stores identity rotations."""
    p = _small(7, n_p=5, n_l=10)
    o = oracle.Oracle(p)
    o.linearize()
    lin = [o.block(j) for j in range(o.n_l)]
    _, _, _, Dl2 = o.scaling()
    o.marginalize()
    marg = [o.block(j) for j in range(o.n_l)]
    o.damp(lam)
    for j in range(o.n_l):
        k = o.track_length(j)
        B = o.block(j)
        Jl0 = lin[j][:2 * k, 9 * k:9 * k + 3]
        R1 = B[:3, 9 * k:9 * k + 3]
        Dl = np.diag(Dl2[3 * j:3 * j + 3])
        np.testing.assert_allclose(R1.T @ R1, Jl0.T @ Jl0 + lam * Dl, rtol=1e-11, atol=1e-13)
        assert np.all(B[3:, 9 * k:9 * k + 3] == 0.0)
        stack = lin[j].copy()
        stack[2 * k:, 9 * k:9 * k + 3] = np.sqrt(lam) * np.sqrt(Dl)
        np.testing.assert_allclose(B.T @ B, stack.T @ stack, rtol=1e-10, atol=1e-12)
        if lam == 0.0:
            np.testing.assert_array_equal(o.givens_of(j), np.tile([1.0, 0.0], (6, 1)))
    o.undamp()
    for j in range(o.n_l):
        B = o.block(j)
        assert np.abs(B - marg[j]).max() <= 1e-12 * max(1.0, np.abs(marg[j]).max())
    # re-damping after undo equals direct damping
    o.damp(lam)
    d1 = [o.block(j) for j in range(o.n_l)]
    o.damp(2 * lam + 1)
    o.damp(lam)
    for j in range(o.n_l):
        np.testing.assert_allclose(o.block(j), d1[j], rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("seed,lam", [(10, 1e-4), (11, 0.0), (12, 1.0), (13, 1e-2)])
def test_reduced_system_equals_schur_complement(seed, lam):
    """The paper's central claim (damped P:277): sum A^T A + lam D_p^2 equals the explicit
    damped Schur complement H_pp - H_pl (H_ll)^-1 H_lp, and sum A^T q equals b_p - H_pl H_ll^-1 b_l.
    The SC here is formed in numpy from the normal equations; no QR involved."""
    p = _small(seed, n_p=6, n_l=25, kmin=2, kmax=6)
    o = oracle.Oracle(p)
    o.linearize()
    o.marginalize()
    o.damp(lam)
    H, b = o.reduced_dense()
    J, r, D2 = stacked(o)
    Ht, bt, *_ = schur(J, r, D2, lam, o.n_p)
    assert relf(H, Ht) < 1e-10
    assert relf(b, bt) < 1e-10
    assert np.allclose(H, H.T, rtol=0, atol=1e-12 * np.abs(H).max())
    # implicit product (Eq. cg_mult) equals the dense matrix; symmetry u^T H v = v^T H u
    rng = np.random.default_rng(seed)
    u, v = rng.normal(size=(2, 9 * o.n_p))
    np.testing.assert_allclose(o.matvec(v), H @ v, rtol=1e-11, atol=1e-12 * np.abs(H).max())
    assert abs(u @ o.matvec(v) - v @ o.matvec(u)) < 1e-10 * np.abs(H).max() * 9 * o.n_p
    # rhs from the preconditioner pass equals the dense rhs
    assert o.precond_rhs() == 0
    np.testing.assert_allclose(o.rhs(), b, rtol=1e-12, atol=1e-12 * np.abs(b).max())
    # positive definite by construction
    if lam > 0:
        assert np.linalg.eigvalsh(H).min() > 0


@pytest.mark.parametrize("seed,lam", [(20, 1e-4), (21, 1e-2)])
def test_pcg_backsub_and_brute_force_step(seed, lam):
    """PCG at tol 1e-12 equals the dense solve of H~ dp = -b~; NM back-substitution equals SC
    back-substitution; and (dp, dl) equals the brute-force dense least-squares minimizer
    of Eq. linearized_residual.  The model decrease (C10) equals |r|^2 - |r + J dx|^2."""
    p = _small(seed, n_p=6, n_l=30, kmin=2, kmax=6)
    o = oracle.Oracle(p)
    o.linearize()
    o.marginalize()
    o.damp(lam)
    H, b = o.reduced_dense()
    assert o.precond_rhs() == 0
    it, reason, rel = o.pcg(tol=1e-12, max_iters=2000)
    assert reason == 0 and it > 0
    dp = o.dp()
    dp_exact = np.linalg.solve(H, -b)
    assert relf(dp, dp_exact) < 1e-9
    o.backsub()
    dl = o.dl()
    J, r, D2 = stacked(o)
    Ht, bt, Hll, Hpl, bl = schur(J, r, D2, lam, o.n_p)
    dl_sc = -np.linalg.solve(Hll, bl + Hpl.T @ dp)
    assert relf(dl, dl_sc) < 1e-9
    dx = brute_force_step(J, r, D2, lam)
    assert relf(dp, dx[:9 * o.n_p]) < 1e-8
    assert relf(dl, dx[9 * o.n_p:]) < 1e-8
    # C10 model decrease, with the inexact dp of a loose PCG too
    for tol in (1e-12, 1e-1):
        o.pcg(tol=tol, max_iters=500)
        o.backsub()
        dxx = np.concatenate([o.dp(), o.dl()])
        direct = r @ r - np.sum((r + J @ dxx) ** 2)
        np.testing.assert_allclose(o.model_decrease(), direct, rtol=1e-9)


@pytest.mark.parametrize("seed,lam", [(14, 1e-4), (15, 1.0)])
def test_block_jacobi_blocks_are_the_diagonal_of_the_reduced_system(seed, lam):
    """The preconditioner is block Jacobi on H~ ("block-diagonal of H~pp", C12): each
    9 x 9 block P_i of orc_precond_rhs (reconstructed from its stored Cholesky factor) equals the
    diagonal block of the dense H~ of orc_reduced_dense, whose diagonal includes lambda D_p^2, and
    the dense H~ itself is pinned to the explicit Schur complement above.  The first PCG iterate
    is alpha M^-1 (-b~) with M = blockdiag(H~): a point-Jacobi or unpreconditioned
    PCG fails both checks."""
    p = _small(seed, n_p=6, n_l=30, kmin=2, kmax=6)
    o = oracle.Oracle(p)
    o.linearize()
    o.marginalize()
    o.damp(lam)
    H, b = o.reduced_dense()
    assert o.precond_rhs() == 0
    P = o.precond_blocks()
    for i in range(o.n_p):
        Hi = H[9 * i:9 * i + 9, 9 * i:9 * i + 9]
        np.testing.assert_allclose(P[i], Hi, rtol=1e-12, atol=1e-13 * np.abs(Hi).max())
        assert np.abs(Hi - np.diag(np.diag(Hi))).max() > 1e-3 * np.abs(Hi).max()  # genuinely 9 x 9
    M = np.zeros_like(H)
    for i in range(o.n_p):
        M[9 * i:9 * i + 9, 9 * i:9 * i + 9] = H[9 * i:9 * i + 9, 9 * i:9 * i + 9]
    z = np.linalg.solve(M, -b)
    alpha = (-b @ z) / (z @ H @ z)
    it, reason, _ = o.pcg(tol=0.0, max_iters=1)
    assert it == 1 and reason == 1
    assert relf(o.dp(), alpha * z) < 1e-11


def test_pcg_degenerate_and_limits():
    p = _small(30, n_p=5, n_l=12)
    o = oracle.Oracle(p)
    o.linearize()
    o.marginalize()
    o.damp(1e-3)
    assert o.precond_rhs() == 0
    it, reason, _ = o.pcg(tol=1e-30, max_iters=3)
    assert it == 3 and reason == 1
    # huge lambda: H~ ~ lam D_p^2 -> preconditioner exact, converges in 1 iteration
    o.damp(1e12)
    assert o.precond_rhs() == 0
    it, reason, _ = o.pcg(tol=1e-6, max_iters=50)
    assert it == 1 and reason == 0


def _dense_lm_reference(p, iters, lam0=1e-4):
    """A plain numpy LM loop: dense least squares of Eq. linearized_residual per iteration, the
    direct model decrease |r|^2 - |r + J dx|^2, and the C9 lambda rule.  Uses only the oracle's
    pinned per-observation model (projection / Jacobians)."""
    cams, pts = p["cameras_init"].copy(), p["points_init"].copy()
    oc, op, uv = p["obs_cam"], p["obs_pt"], p["obs_uv"]
    n_p, n_l = len(cams), len(pts)

    def lin(cams, pts):
        n = len(oc)
        r = np.zeros(2 * n)
        J = np.zeros((2 * n, 9 * n_p + 3 * n_l))
        for i in range(n):
            ri, Jc, Jl = oracle.residual_jacobian(cams[oc[i]], pts[op[i]], uv[i])
            r[2 * i:2 * i + 2] = ri
            J[2 * i:2 * i + 2, 9 * oc[i]:9 * oc[i] + 9] = Jc
            J[2 * i:2 * i + 2, 9 * n_p + 3 * op[i]:9 * n_p + 3 * op[i] + 3] = Jl
        return r, J

    def cost(cams, pts):
        s = 0.0
        for i in range(len(oc)):
            q, pz = oracle.project(cams[oc[i]], pts[op[i]])
            if pz >= 0:
                return np.inf
            s += np.sum((q - uv[i]) ** 2)
        return s

    lam, nu = lam0, 2.0
    E = cost(cams, pts)
    r, J = lin(cams, pts)
    out = []
    for _ in range(iters):
        c2 = np.sum(J * J, 0)
        s = 1 / (1 + np.sqrt(c2))
        Js = J * s
        D2 = np.clip(c2 * s * s, 1e-6, 1e32)
        dz = brute_force_step(Js, r, D2, lam)
        dx = s * dz
        model = r @ r - np.sum((r + Js @ dz) ** 2)
        c_t = cams + dx[:9 * n_p].reshape(n_p, 9)
        p_t = pts + dx[9 * n_p:].reshape(n_l, 3)
        Et = cost(c_t, p_t)
        rho = (E - Et) / model
        if model > 0 and np.isfinite(Et) and rho > 1e-3:
            cams, pts, E = c_t, p_t, Et
            lam *= max(1 / 3, 1 - (2 * rho - 1) ** 3)
            nu = 2.0
            r, J = lin(cams, pts)
        else:
            lam *= nu
            nu *= 2
        lam = min(max(lam, 1e-16), 1e16)
        out.append(E)
    return np.array(out)


def test_lm_matches_dense_reference_config1():
    """5 LM iterations on config 1 (BASELINE configs[0]): the oracle with PCG at 1e-12 reproduces
    the dense brute-force LM trajectory; accepted costs strictly decrease; never indefinite."""
    p = synth.make_problem(1)
    o = oracle.Oracle(p)
    costs, prev = [], o.cost()
    for _ in range(5):
        rep = o.lm_step(pcg_tol=1e-12, pcg_max_iters=2000)
        assert rep["pcg_reason"] != 2
        if rep["accepted"]:
            assert rep["cost_after"] < prev
        prev = rep["cost_after"]
        costs.append(rep["cost_after"])
    ref = _dense_lm_reference(p, 5)
    np.testing.assert_allclose(costs, ref, rtol=1e-9)


def test_lm_backtracking_reuses_linearization():
    """A rejected step re-damps the same linearization: forcing huge first steps by a
    tiny lambda on a noisy problem must still leave the cost non-increasing."""
    p = _small(40, n_p=5, n_l=20, cam_noise=0.05, pt_noise=0.3)
    o = oracle.Oracle(p)
    o.set_lm(1e-12)
    prev = o.cost()
    for _ in range(8):
        rep = o.lm_step()
        assert rep["cost_after"] <= prev
        prev = rep["cost_after"]


def test_streaming_mode_equals_arena_mode():
    """The streaming mode (SURVEY §8c "Oracle capacity": blocks recomputed, O3-O5, wherever they are
    read) runs the same per-landmark arithmetic as the block arena: identical blocks and rotations,
    the same products / preconditioner / b~ / PCG / back-substitution up to FP64 summation order,
    the same LM trajectory; the batched products equal single products."""
    p = _small(50, n_p=7, n_l=40, kmin=2, kmax=7)
    a = oracle.Oracle(p)
    b = oracle.Oracle(p)
    b.set_streaming(True)
    for o in (a, b):
        o.linearize()
        o.marginalize()
        o.damp(3e-3)
    for j in range(a.n_l):
        np.testing.assert_array_equal(a.block(j), b.block(j))
        np.testing.assert_array_equal(a.givens_of(j), b.givens_of(j))
    rng = np.random.default_rng(1)
    V = rng.normal(size=(3, 9 * a.n_p))
    for v in V:
        np.testing.assert_allclose(b.matvec(v), a.matvec(v), rtol=1e-12, atol=1e-12 * np.abs(a.matvec(v)).max())
    np.testing.assert_allclose(a.products(V), np.stack([a.matvec(v) for v in V]), rtol=1e-12,
                               atol=1e-12 * np.abs(a.matvec(V[0])).max())
    assert a.precond_rhs() == 0 and b.precond_rhs() == 0
    np.testing.assert_allclose(b.precond_blocks(), a.precond_blocks(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(b.rhs(), a.rhs(), rtol=1e-12, atol=1e-13 * np.abs(a.rhs()).max())
    ia, _, _ = a.pcg(1e-8, 200)
    ib, _, _ = b.pcg(1e-8, 200)
    assert ia == ib
    assert relf(b.dp(), a.dp()) < 1e-10
    a.backsub()
    b.backsub()
    assert relf(b.dl(), a.dl()) < 1e-10
    for o in (a, b):
        o.set_state(p["cameras_init"], p["points_init"])
        o.set_lm(1e-4, 2.0)
    for _ in range(4):
        # (PCG run to the fixed point: the iteration count at a loose tolerance depends on the
        #  summation order of the two modes' products on this ill-conditioned tiny problem)
        ra, rb = a.lm_step(pcg_tol=1e-13, pcg_max_iters=5000), b.lm_step(pcg_tol=1e-13, pcg_max_iters=5000)
        assert ra["accepted"] == rb["accepted"]
        np.testing.assert_allclose(rb["cost_after"], ra["cost_after"], rtol=1e-11)
