"""GPU parity on the degenerate and extreme inputs of the method (SURVEY §8c protocol, same bars):
the smallest problem (one landmark, k = 2, two cameras), a camera without observations (its
block of H~ is lambda D^2 with D^2 clamped to diag_min, C8), a problem made only of k = 2 tracks
(every landmark on the smallest small-k path), a track at the maximum length KMAX (huge path,
two-pass / fused product), and a problem without observations."""
import numpy as np
import pytest

import oracle
from _lm import lm_parity
from paper_2103_01843_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

KMAX = 3072  # rba_internal.cuh


def relf(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _solver(p, **kw):
    from paper_2103_01843_b200.rba import Solver
    return Solver(p, **kw)


def _pair(p, lam):
    s = _solver(p)
    s.linearize()
    s.marginalize(lam)
    o = oracle.Oracle(p)
    o.linearize()
    o.marginalize()
    o.damp(lam)
    return s, o


def _mv(s, v):
    return s.matvec(torch.tensor(v, dtype=torch.float32, device="cuda")).double().cpu().numpy()


def _dense_H(s, n):
    return np.stack([_mv(s, np.eye(n)[i]) for i in range(n)], 1)


def _lm(p, iters=5, ref="after"):
    """Costs after each LM iteration within 1e-4 of the oracle's, relative to the cost after the
    iteration (ref="after", the §8c bar) or to the initial cost (ref="start": an underdetermined
    problem whose cost falls to the FP32 rounding floor of its residuals, where a relative bar on
    the remainder would compare rounding noise)."""
    s, o = _solver(p), oracle.Oracle(p)
    e0 = o.cost()
    for i in range(iters):
        (rg, ro, _), = lm_parity(s, o, 1, bar=np.inf)  # §8c replay at the tolerance edge (tests/_lm.py)
        den = ro["cost_after"] if ref == "after" else e0
        assert abs(rg["cost_after"] - ro["cost_after"]) <= 1e-4 * den, (i, rg, ro)


@pytest.mark.parametrize("lam", [0.0, 1e-4])
def test_single_landmark_two_cameras(lam):
    p = synth.make_tracks(61, [2], n_p=2)
    s, o = _pair(p, lam)
    if lam > 0:  # at lambda = 0 a single landmark leaves H~ singular (gauge); the product still agrees
        H, b = o.reduced_dense()
        assert relf(_dense_H(s, 18), H) <= 1e-4
        s.pcg()
        assert relf(s.rhs(), b) <= 1e-4
    else:
        v = np.random.default_rng(0).normal(size=18)
        assert relf(_mv(s, v), o.matvec(v)) <= 1e-4
    _lm(p, ref="start")  # 4 residuals, 21 unknowns: the cost goes to ~0


def test_camera_without_observations():
    base = synth.make_tracks(62, list(np.random.default_rng(62).integers(2, 7, 60)), n_p=12)
    p = dict(base)
    extra = base["cameras_init"][:1].copy()
    p["cameras_init"] = np.concatenate([base["cameras_init"], extra])
    p["cameras_true"] = np.concatenate([base["cameras_true"], extra])
    lam = 1e-3
    s, o = _pair(p, lam)
    H, b = o.reduced_dense()
    Hg = _dense_H(s, 9 * 13)
    assert relf(Hg, H) <= 1e-4
    blk = Hg[-9:, -9:]  # lambda * clamp(0) = lambda * diag_min on the diagonal, zero elsewhere
    np.testing.assert_allclose(np.diag(blk), lam * 1e-6, rtol=1e-6)
    assert np.all(Hg[-9:, :-9] == 0) and np.all(Hg[:-9, -9:] == 0)
    s.pcg()
    assert relf(s.rhs(), b) <= 1e-4
    s.backsub()
    dp, _ = s.step()
    assert np.all(dp[-9:] == 0)
    _lm(p)


def test_only_k2_tracks():
    p = synth.make_tracks(63, [2] * 3000, n_p=24)
    s, o = _pair(p, 1e-4)
    H, b = o.reduced_dense()
    assert relf(_dense_H(s, 9 * 24), H) <= 1e-4
    for j in range(0, 3000, 499):
        Bg, Bo = s.block(j), o.block(j)
        assert relf(Bg.T @ Bg, Bo.T @ Bo) <= 1e-4
    _lm(p, 3)


def test_track_at_kmax():
    """k = KMAX: marginalization with multi-block threads, the huge-track product and the
    preconditioner's second pass, against the oracle's probes."""
    ks = [KMAX] + list(np.random.default_rng(64).integers(2, 9, 80))
    p = synth.make_tracks(64, ks, n_p=KMAX)
    s, o = _pair(p, 1e-3)
    rng = np.random.default_rng(1)
    for _ in range(2):
        v = rng.normal(size=9 * KMAX)
        assert relf(_mv(s, v), o.matvec(v)) <= 1e-4
    s.pcg()
    assert o.precond_rhs() == 0
    assert relf(s.rhs(), o.rhs()) <= 1e-4
    Bg = s.block(0)
    assert Bg.shape == (2 * KMAX + 3, 9 * KMAX + 4)
    Bo = o.block(0)
    # the top 3 rows hold R^1 and Q^1^T J_p: rotation-invariant checks on rows 0..2 and the norms
    assert relf(np.linalg.norm(Bg[3:, :9 * KMAX]), np.linalg.norm(Bo[3:, :9 * KMAX])) <= 1e-5
    assert relf(Bg[:3, :9 * KMAX].T @ Bg[:3, 9 * KMAX:9 * KMAX + 3], Bo[:3, :9 * KMAX].T @ Bo[:3, 9 * KMAX:9 * KMAX + 3]) <= 1e-4


def test_track_at_kmax_redamp():
    """Re-damping (K3) of a k = KMAX block (multi-block threads): marginalized at 1e-3,
    re-damped to 0.7, against the oracle damped at 0.7 from scratch (R^1^T R^1, Gram probes of the
    reduced rows, the product and b~)."""
    ks = [KMAX] + list(np.random.default_rng(66).integers(2, 9, 80))
    p = synth.make_tracks(66, ks, n_p=KMAX)
    s = _solver(p)
    s.linearize()
    s.marginalize(1e-3)
    s.marginalize(0.7)
    o = oracle.Oracle(p)
    o.linearize()
    o.marginalize()
    o.damp(0.7)
    Bg, Bo = s.block(0), o.block(0)
    k = KMAX
    R1g, R1o = Bg[:3, 9 * k:9 * k + 3], Bo[:3, 9 * k:9 * k + 3]
    assert relf(R1g.T @ R1g, R1o.T @ R1o) <= 1e-4
    rng = np.random.default_rng(2)
    for _ in range(2):
        z = rng.normal(size=9 * k + 1)
        Ag = np.concatenate([Bg[3:, :9 * k], Bg[3:, -1:]], 1)
        Ao = np.concatenate([Bo[3:, :9 * k], Bo[3:, -1:]], 1)
        assert relf(Ag.T @ (Ag @ z), Ao.T @ (Ao @ z)) <= 1e-4
    for _ in range(2):
        v = rng.normal(size=9 * KMAX)
        assert relf(_mv(s, v), o.matvec(v)) <= 1e-4
    s.pcg()
    assert o.precond_rhs() == 0
    assert relf(s.rhs(), o.rhs()) <= 1e-4


def test_no_observations():
    """No landmarks: E = 0, the reduced system is lambda D^2 alone (b~ = 0), and an LM step leaves
    the state unchanged without error."""
    p = synth.make_tracks(65, [2], n_p=3)
    p = dict(p, points_init=p["points_init"][:0], points_true=p["points_true"][:0],
             obs_cam=p["obs_cam"][:0], obs_pt=p["obs_pt"][:0], obs_uv=p["obs_uv"][:0])
    s = _solver(p)
    r = s.lm_step()
    assert r["cost"] == 0.0 and r["cost_after"] == 0.0
    cams, pts = s.state()
    assert np.array_equal(cams, p["cameras_init"]) and pts.shape == (0, 3)
