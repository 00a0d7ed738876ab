"""Pins for the oracle's camera model (O1): golden projection values, an independent
rotation routine (scipy), central finite differences for the analytic Jacobians,
Givens golden values and the statistical size of E at the true state."""
import os

import numpy as np
import pytest

import oracle
from paper_2103_01843_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    out = []
    for line in open(os.path.join(GOLD, name)):
        line = line.split("#")[0].strip()
        if line:
            out.append([float(x) for x in line.split()])
    return np.array(out)


def test_projection_golden():
    for row in _rows("projection.txt"):
        cam, X, uv = row[:9], row[9:12], row[12:14]
        got, pz = oracle.project(cam, X)
        assert pz < 0
        np.testing.assert_allclose(got, uv, rtol=0, atol=1e-12)


def test_projection_vs_scipy_rotation():
    """P = R(w) X + t with R from scipy's rotvec (a library routine, not the oracle's Rodrigues)."""
    from scipy.spatial.transform import Rotation
    rng = np.random.default_rng(1)
    for _ in range(200):
        w = rng.normal(0, 1.0, 3)
        if rng.random() < 0.2:
            w *= 1e-9  # small-angle series branch (C22)
        t = rng.normal(0, 1, 3)
        f, k1, k2 = rng.uniform(100, 1000), rng.normal(0, 0.1), rng.normal(0, 0.01)
        X = rng.normal(0, 1, 3)
        P = Rotation.from_rotvec(w).as_matrix() @ X + t
        if P[2] > -0.5:
            X = X - (P[2] + 1.0) * Rotation.from_rotvec(w).as_matrix()[2]
            P = Rotation.from_rotvec(w).as_matrix() @ X + t
        p = -P[:2] / P[2]
        n = p @ p
        expect = f * (1 + k1 * n + k2 * n * n) * p
        got, pz = oracle.project(np.r_[w, t, f, k1, k2], X)
        np.testing.assert_allclose(pz, P[2], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(got, expect, rtol=1e-11, atol=1e-9)


def test_jacobians_central_fd():
    """1000 random configurations, central differences h=1e-6 in FP64, 1e-5 relative."""
    rng = np.random.default_rng(2)
    worst = 0.0
    for _ in range(1000):
        cam = np.r_[rng.normal(0, 0.8, 3), rng.normal(0, 1, 3), rng.uniform(200, 1200),
                    rng.normal(0, 0.05), rng.normal(0, 0.01)]
        if rng.random() < 0.1:
            cam[:3] *= 1e-10
        X = rng.normal(0, 1, 3)
        _, pz = oracle.project(cam, X)
        if pz > -0.5:
            continue
        u = rng.normal(0, 100, 2)
        r, Jc, Jl = oracle.residual_jacobian(cam, X, u)
        h = 1e-6
        Jc_fd = np.zeros((2, 9))
        Jl_fd = np.zeros((2, 3))
        for q in range(9):
            e = np.zeros(9)
            e[q] = h * max(1.0, abs(cam[q]))
            Jc_fd[:, q] = (oracle.residual_jacobian(cam + e, X, u)[0]
                           - oracle.residual_jacobian(cam - e, X, u)[0]) / (2 * e[q])
        for q in range(3):
            e = np.zeros(3)
            e[q] = h
            Jl_fd[:, q] = (oracle.residual_jacobian(cam, X + e, u)[0]
                           - oracle.residual_jacobian(cam, X - e, u)[0]) / (2 * h)
        scale = max(np.abs(Jc).max(), np.abs(Jl).max())
        err = max(np.abs(Jc - Jc_fd).max(), np.abs(Jl - Jl_fd).max()) / scale
        worst = max(worst, err)
        # residual = projection - observation (S:129 sign convention)
        uv, _ = oracle.project(cam, X)
        np.testing.assert_allclose(r, uv - u, atol=1e-9)
    assert worst < 1e-5, worst


def test_givens_golden():
    for a, b, c, s, rho in _rows("givens.txt"):
        got = oracle.givens(a, b)
        np.testing.assert_allclose(got, (c, s, rho), atol=1e-15)
    rng = np.random.default_rng(3)
    for _ in range(100):
        a, b = rng.normal(size=2)
        c, s, rho = oracle.givens(a, b)
        assert abs(c * c + s * s - 1) < 1e-15                        # P:571 orthogonality
        assert abs(-s * a + c * b) < 1e-15                           # target zeroed (C5)
        assert abs(c * a + s * b - rho) < 1e-14


def test_cost_at_truth_is_noise_level():
    """E = sum |r|^2 (no 1/2 -- C3).  At the true state the residual is the N(0,1) pixel
    noise, so E / (2 n_obs) is chi^2/dof ~ 1 with std 1/sqrt(n_obs)."""
    for cfg in (1, 2):
        p = synth.make_problem(cfg)
        o = oracle.Oracle(p, cams=p["cameras_true"], pts=p["points_true"])
        n = len(p["obs_cam"])
        ratio = o.cost() / (2 * n)
        assert abs(ratio - 1) < 6 / np.sqrt(n), ratio


def test_cost_behind_camera_is_inf():
    p = synth.make_random_small(5)
    pts = p["points_init"].copy()
    cam0 = p["cameras_init"][p["obs_cam"][0]]
    j = p["obs_pt"][0]
    # move landmark j behind camera obs_cam[0]: X' such that P_z > 0
    from scipy.spatial.transform import Rotation
    R = Rotation.from_rotvec(cam0[:3]).as_matrix()
    pts[j] = R.T @ (np.array([0, 0, 5.0]) - cam0[3:6])
    o = oracle.Oracle(p, pts=pts)
    assert o.cost() == np.inf


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_generator_shapes(cfg):
    """Generated workloads have the shapes of the paper's BAL rows / BASELINE configs (§8d-2)."""
    if cfg >= 3:
        pytest.skip("large generator configs are exercised by bench/gpu tests")
    p = synth.make_problem(cfg)
    st = synth.stats(p)
    assert st["n_p"] == synth.CONFIGS[cfg]["n_p"] and st["n_l"] == synth.CONFIGS[cfg]["n_l"]
    if cfg == 1:
        assert 3 <= st["k_mean"] <= 8 and 900 <= st["n_obs"] <= 1300
    if cfg == 2:
        assert abs(st["k_mean"] - 3.46) < 0.1 and abs(st["n_obs"] - 225_000) < 5000
    # unique (cam, pt) pairs and k >= 2
    key = p["obs_pt"].astype(np.int64) * 100000 + p["obs_cam"]
    assert np.unique(key).size == key.size
    assert np.bincount(p["obs_pt"]).min() >= 2
    assert synth.digest(p) == synth.digest(synth.make_problem(cfg))  # seeded, deterministic
