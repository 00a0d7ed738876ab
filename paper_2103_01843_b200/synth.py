"""Seeded synthetic bundle-adjustment problems shaped like the paper's BAL workloads.

This module is the ONLY code shared by the CUDA path and the FP64 oracle, and it holds
none of the method's arithmetic (no Jacobians, no QR, no solver).  It only *synthesizes
inputs*: true cameras and points, observations = forward projection of the true state plus
pixel noise, and a perturbed initial state.  The forward projection used to synthesize the
observations is written here independently (rotation matrices, not angle-axis Rodrigues),
so neither side of the parity comparison supplies the other's inputs.

Configurations follow BASELINE.json `configs` and the readings in SURVEY.md §8d-2 / §8c
(C18-C21), recorded in DESIGN.md §3:

* cfg 1: 16 cameras on a circle of radius 10 looking at the origin, 200 landmarks uniform in
  [-2,2]^3, each seen by a random 3..8-subset of cameras, f=500, k1=k2=0.
* cfg 2..5: "street" geometry (noisy ground-plane trajectory, optical axis +y); track lengths
  per config (geometric / log-normal / mixed); f~U(400,1200), k1~N(0,1e-2), k2~N(0,1e-4).
* all: pixel noise N(0,1); initial angle-axis += N(0,0.01), t += N(0,0.05), X += N(0,0.05)
  (second argument of N is a standard deviation, C20/C21).

Camera parameter order is BAL's: [w0 w1 w2 t0 t1 t2 f k1 k2]; projection convention
p = -P_xy/P_z (visible iff P_z < 0), pi = f (1 + k1|p|^2 + k2|p|^4) p  (PAPER.md P:463,
"Snavely projection model").
"""
from __future__ import annotations

import hashlib
import math

import numpy as np

# (n_p, n_l) per config, BASELINE.json configs[0..4]
CONFIGS = {
    1: dict(n_p=16, n_l=200, lm_iters=5),
    2: dict(n_p=257, n_l=65_000, lm_iters=20),
    3: dict(n_p=356, n_l=226_000, lm_iters=10),
    4: dict(n_p=1778, n_l=993_000, lm_iters=10),
    5: dict(n_p=13682, n_l=4_460_000, lm_iters=10),
}


# ----------------------------------------------------------------------------- rotations
def _skew(w):
    z = np.zeros(w.shape[:-1])
    return np.stack([
        np.stack([z, -w[..., 2], w[..., 1]], -1),
        np.stack([w[..., 2], z, -w[..., 0]], -1),
        np.stack([-w[..., 1], w[..., 0], z], -1)], -2)


def rotvec_to_matrix(w):
    """Exponential map (Rodrigues), vectorized; used only to synthesize noise rotations."""
    w = np.asarray(w, dtype=np.float64)
    th = np.linalg.norm(w, axis=-1)[..., None, None]
    K = _skew(w)
    small = th < 1e-12
    ths = np.where(small, 1.0, th)
    a = np.where(small, 1.0, np.sin(ths) / ths)
    b = np.where(small, 0.5, (1.0 - np.cos(ths)) / (ths * ths))
    return np.eye(3) + a * K + b * (K @ K)


def matrix_to_rotvec(R):
    """Logarithm map of rotation matrices (angles < pi - 1e-3 here), vectorized."""
    # via a unit quaternion (Shepperd's branch on the largest diagonal term), robust up to pi
    R = np.asarray(R, dtype=np.float64).reshape(-1, 3, 3)
    m = R
    tr = m[:, 0, 0] + m[:, 1, 1] + m[:, 2, 2]
    cand = np.stack([tr, m[:, 0, 0], m[:, 1, 1], m[:, 2, 2]], 1)
    sel = np.argmax(cand, 1)
    q = np.zeros((R.shape[0], 4))  # (w, x, y, z)
    for b in range(4):
        i = sel == b
        if not i.any():
            continue
        mm = m[i]
        if b == 0:
            s = 2.0 * np.sqrt(1.0 + cand[i, 0])
            q[i] = np.stack([0.25 * s, (mm[:, 2, 1] - mm[:, 1, 2]) / s,
                             (mm[:, 0, 2] - mm[:, 2, 0]) / s, (mm[:, 1, 0] - mm[:, 0, 1]) / s], 1)
        elif b == 1:
            s = 2.0 * np.sqrt(1.0 + mm[:, 0, 0] - mm[:, 1, 1] - mm[:, 2, 2])
            q[i] = np.stack([(mm[:, 2, 1] - mm[:, 1, 2]) / s, 0.25 * s,
                             (mm[:, 0, 1] + mm[:, 1, 0]) / s, (mm[:, 0, 2] + mm[:, 2, 0]) / s], 1)
        elif b == 2:
            s = 2.0 * np.sqrt(1.0 + mm[:, 1, 1] - mm[:, 0, 0] - mm[:, 2, 2])
            q[i] = np.stack([(mm[:, 0, 2] - mm[:, 2, 0]) / s, (mm[:, 0, 1] + mm[:, 1, 0]) / s,
                             0.25 * s, (mm[:, 1, 2] + mm[:, 2, 1]) / s], 1)
        else:
            s = 2.0 * np.sqrt(1.0 + mm[:, 2, 2] - mm[:, 0, 0] - mm[:, 1, 1])
            q[i] = np.stack([(mm[:, 1, 0] - mm[:, 0, 1]) / s, (mm[:, 0, 2] + mm[:, 2, 0]) / s,
                             (mm[:, 1, 2] + mm[:, 2, 1]) / s, 0.25 * s], 1)
    q[q[:, 0] < 0] *= -1.0
    vn = np.linalg.norm(q[:, 1:], axis=1)
    th = 2.0 * np.arctan2(vn, q[:, 0])
    scale = np.where(vn < 1e-12, 2.0, th / np.where(vn < 1e-12, 1.0, vn))
    return q[:, 1:] * scale[:, None]


# ----------------------------------------------------------------------------- projection
def _project_true(Rs, ts, intr, cam_idx, X):
    """Forward model for synthesis only: P = R X + t, p = -P_xy/P_z, pi = f d p."""
    P = np.einsum("nij,nj->ni", Rs[cam_idx], X) + ts[cam_idx]
    p = -P[:, :2] / P[:, 2:3]
    n = np.sum(p * p, axis=1)
    f, k1, k2 = intr[cam_idx, 0], intr[cam_idx, 1], intr[cam_idx, 2]
    d = 1.0 + k1 * n + k2 * n * n
    return (f * d)[:, None] * p, P[:, 2], np.sqrt(n)


# ----------------------------------------------------------------------------- track lengths
def _track_lengths(cfg, n_l, n_p, rng):
    if cfg == 1:
        return rng.integers(3, 9, size=n_l)
    if cfg == 2:  # 2 + Geom(p=0.406) on {0,1,...}: mean ~3.46
        k = 2 + (rng.geometric(0.406, size=n_l) - 1)
        kmax = 42
    elif cfg == 3:  # lognormal (C19): 2 + floor(exp(mu + sigma Z)), <= 200
        k = _lognormal_k(rng, n_l, 0.7675, 1.130, 200)
        kmax = 200
    elif cfg == 4:  # C18: 0.5% log-uniform[50,400], rest 2 + Geom(p=0.3115)
        k = 2 + (rng.geometric(0.3115, size=n_l) - 1)
        nlong = int(round(0.005 * n_l))
        idx = rng.choice(n_l, size=nlong, replace=False)
        k[idx] = np.round(np.exp(rng.uniform(math.log(50), math.log(400), size=nlong))).astype(np.int64)
        kmax = 400
    elif cfg == 5:  # C19: lognormal (0.2179, 1.690), <= 1748
        k = _lognormal_k(rng, n_l, 0.2179, 1.690, 1748)
        kmax = 1748
    else:
        raise ValueError(cfg)
    return np.minimum(np.minimum(k, kmax), n_p).astype(np.int64)


def _lognormal_k(rng, n, mu, sigma, kmax):
    k = 2 + np.floor(np.exp(mu + sigma * rng.standard_normal(n))).astype(np.int64)
    bad = k > kmax
    while bad.any():  # resample (truncate by rejection)
        k[bad] = 2 + np.floor(np.exp(mu + sigma * rng.standard_normal(int(bad.sum())))).astype(np.int64)
        bad = k > kmax
    return k


# ----------------------------------------------------------------------------- geometry
def _circle_cameras(n_p):
    Rs, ts = [], []
    for i in range(n_p):
        a = 2.0 * math.pi * i / n_p
        C = 10.0 * np.array([math.cos(a), math.sin(a), 0.0])
        z = C / np.linalg.norm(C)               # camera looks down -z, i.e. at the origin
        x = np.cross([0.0, 0.0, 1.0], z)
        x /= np.linalg.norm(x)
        y = np.cross(z, x)
        R = np.stack([x, y, z])
        Rs.append(R)
        ts.append(-R @ C)
    return np.array(Rs), np.array(ts)


def _street_cameras(n_p, rng):
    C = np.stack([np.arange(n_p) * 1.0 + rng.normal(0, 0.1, n_p),
                  rng.normal(0, 0.5, n_p),
                  1.6 + rng.normal(0, 0.05, n_p)], 1)
    # optical axis (camera -z) = +y world; image x = world +x; image y = world +z
    Rbase = np.array([[1.0, 0, 0], [0, 0, 1.0], [0, -1.0, 0]])
    noise = rng.normal(0, math.radians(2.0), size=(n_p, 3))  # yaw/pitch/roll-sized noise
    Rs = rotvec_to_matrix(noise) @ Rbase
    ts = -np.einsum("nij,nj->ni", Rs, C)
    return Rs, ts, C


def _perturb_poses(Rs, ts, intr, rng, rot_sigma, pos_sigma):
    """Reading C21: a pose is perturbed as a rigid body -- orientation by a random rotation with
    per-axis std `rot_sigma` rad, camera centre by N(0, pos_sigma) per axis -- and re-expressed
    in BAL parameters (angle-axis w, t = -R C).  Perturbing (w, t) additively instead would swing
    far-from-origin street cameras by metres (0.01 rad x 1 km), putting points behind cameras."""
    n_p = Rs.shape[0]
    C = -np.einsum("nji,nj->ni", Rs, ts)            # C = -R^T t
    R2 = rotvec_to_matrix(rng.normal(0, rot_sigma, size=(n_p, 3))) @ Rs
    C2 = C + rng.normal(0, pos_sigma, size=(n_p, 3))
    t2 = -np.einsum("nij,nj->ni", R2, C2)
    return np.concatenate([matrix_to_rotvec(R2), t2, intr], 1)


def make_problem(cfg: int, seed: int | None = None) -> dict:
    """Build configuration `cfg` (1..5) with seed (default: the config id)."""
    spec = CONFIGS[cfg]
    n_p, n_l = spec["n_p"], spec["n_l"]
    rng = np.random.default_rng(cfg if seed is None else seed)
    k = _track_lengths(cfg, n_l, n_p, rng)
    ptr = np.zeros(n_l + 1, np.int64)
    np.cumsum(k, out=ptr[1:])
    n_obs = int(ptr[-1])
    lm_of_obs = np.repeat(np.arange(n_l), k)
    pos_in_track = np.arange(n_obs) - ptr[lm_of_obs]

    if cfg == 1:
        Rs, ts = _circle_cameras(n_p)
        intr = np.tile([500.0, 0.0, 0.0], (n_p, 1))
        obs_cam = np.empty(n_obs, np.int64)
        for j in range(n_l):
            obs_cam[ptr[j]:ptr[j + 1]] = np.sort(rng.choice(n_p, size=k[j], replace=False))
        X = rng.uniform(-2.0, 2.0, size=(n_l, 3))
    else:
        Rs, ts, C = _street_cameras(n_p, rng)
        intr = np.stack([rng.uniform(400, 1200, n_p), rng.normal(0, 1e-2, n_p),
                         rng.normal(0, 1e-4, n_p)], 1)
        start = rng.integers(0, n_p - k + 1)
        obs_cam = start[lm_of_obs] + pos_in_track
        # window statistics of camera centres along x
        cx = C[:, 0]
        csum = np.concatenate([[0.0], np.cumsum(cx)])
        xbar = (csum[start + k] - csum[start]) / k
        xlo = cx[start]
        xhi = cx[start + k - 1]
        extent = np.abs(xhi - xlo)
        X = np.empty((n_l, 3))
        todo = np.arange(n_l)
        for _ in range(200):
            m = todo.size
            if m == 0:
                break
            d = np.maximum(8.0, 0.7 * extent[todo]) + rng.uniform(0, 20, m)
            X[todo] = np.stack([xbar[todo] + rng.uniform(-2, 2, m), d, rng.uniform(0, 8, m)], 1)
            sel = np.isin(lm_of_obs, todo)
            oc = obs_cam[sel]
            ol = lm_of_obs[sel]
            _, Pz, pn = _project_true(Rs, ts, intr, oc, X[ol])
            bad_obs = (Pz >= -1.0) | (pn >= 1.2)
            bad_lm = np.unique(ol[bad_obs])
            todo = bad_lm
        if todo.size:
            raise RuntimeError(f"generator: {todo.size} landmarks could not be placed")

    uv_true, Pz, _ = _project_true(Rs, ts, intr, obs_cam, X[lm_of_obs])
    assert np.all(Pz < 0)
    obs_uv = uv_true + rng.normal(0.0, 1.0, size=(n_obs, 2))

    cams_true = np.concatenate([matrix_to_rotvec(Rs), ts, intr], 1)
    cams_init = _perturb_poses(Rs, ts, intr, rng, 0.01, 0.05)
    pts_init = X + rng.normal(0, 0.05, size=(n_l, 3))
    return dict(
        cfg=cfg, seed=cfg if seed is None else seed,
        cameras_true=cams_true, points_true=X,
        cameras_init=cams_init, points_init=pts_init,
        obs_cam=obs_cam.astype(np.int32), obs_pt=lm_of_obs.astype(np.int32),
        obs_uv=obs_uv, lm_iters=spec["lm_iters"])


def make_random_small(seed: int, n_p: int = 4, n_l: int = 12, kmin: int = 2, kmax: int = 6,
                      cam_noise: float = 0.01, pt_noise: float = 0.05) -> dict:
    """Tiny random problems (circle geometry, random intrinsics incl. distortion) for oracle
    self-checks and GPU edge cases.  Same dict layout as make_problem."""
    rng = np.random.default_rng(seed)
    Rs, ts = _circle_cameras(n_p)
    Rs = rotvec_to_matrix(rng.normal(0, 0.05, (n_p, 3))) @ Rs
    intr = np.stack([rng.uniform(300, 800, n_p), rng.normal(0, 0.05, n_p),
                     rng.normal(0, 0.01, n_p)], 1)
    kmax = min(kmax, n_p)
    k = rng.integers(kmin, kmax + 1, size=n_l)
    obs_cam, obs_pt = [], []
    for j in range(n_l):
        obs_cam.append(np.sort(rng.choice(n_p, size=k[j], replace=False)))
        obs_pt.append(np.full(k[j], j))
    obs_cam = np.concatenate(obs_cam)
    obs_pt = np.concatenate(obs_pt)
    X = rng.uniform(-2.0, 2.0, size=(n_l, 3))
    uv, Pz, _ = _project_true(Rs, ts, intr, obs_cam, X[obs_pt])
    assert np.all(Pz < 0)
    cams_true = np.concatenate([matrix_to_rotvec(Rs), ts, intr], 1)
    cams_init = _perturb_poses(Rs, ts, intr, rng, cam_noise, 5 * cam_noise)
    return dict(cfg=0, seed=seed, cameras_true=cams_true, points_true=X,
                cameras_init=cams_init, points_init=X + rng.normal(0, pt_noise, X.shape),
                obs_cam=obs_cam.astype(np.int32), obs_pt=obs_pt.astype(np.int32),
                obs_uv=uv + rng.normal(0, 1.0, uv.shape), lm_iters=5)


def subsample_landmarks(prob: dict, every: int, offset: int = 0) -> dict:
    """Deterministic landmark subsample (every `every`-th landmark) with dense reindexing;
    used only for bounded CPU-baseline samples."""
    n_l = prob["points_init"].shape[0]
    keep = np.arange(offset, n_l, every)
    newid = -np.ones(n_l, np.int64)
    newid[keep] = np.arange(keep.size)
    sel = newid[prob["obs_pt"]] >= 0
    out = dict(prob)
    out["points_true"] = prob["points_true"][keep]
    out["points_init"] = prob["points_init"][keep]
    out["obs_cam"] = prob["obs_cam"][sel]
    out["obs_pt"] = newid[prob["obs_pt"][sel]].astype(np.int32)
    out["obs_uv"] = prob["obs_uv"][sel]
    return out


def stats(prob: dict) -> dict:
    k = np.bincount(prob["obs_pt"], minlength=prob["points_init"].shape[0]).astype(np.float64)
    return dict(n_p=int(prob["cameras_init"].shape[0]), n_l=int(k.size), n_obs=int(k.sum()),
                k_mean=float(k.mean()), k_std=float(k.std()), k_max=int(k.max()),
                sum_k2=float((k * k).sum()),
                block_bytes=int(((2 * k + 3) * (9 * k + 4)).sum() * 4),
                r2_bytes=int((72 * k * k).sum()))


def digest(prob: dict) -> str:
    h = hashlib.sha256()
    for key in ("cameras_init", "points_init", "obs_cam", "obs_pt", "obs_uv"):
        h.update(np.ascontiguousarray(prob[key]).tobytes())
    return h.hexdigest()


def make_tracks(seed: int, ks, n_p: int | None = None, pt_noise: float = 0.05, cam_noise: float = 0.01) -> dict:
    """Circle-geometry problem with prescribed track lengths `ks` (edge cases: k = 2, bucket
    boundaries 4/5, 8/9, 16/17, 32/33, long tracks).  Cameras on a circle of radius 10 looking at
    the origin (like cfg 1) with random intrinsics; landmark j seen by a random ks[j]-subset."""
    ks = np.asarray(ks, np.int64)
    n_p = int(max(ks.max(), 16) if n_p is None else n_p)
    rng = np.random.default_rng(seed)
    Rs, ts = _circle_cameras(n_p)
    intr = np.stack([rng.uniform(300, 800, n_p), rng.normal(0, 0.02, n_p), rng.normal(0, 0.005, n_p)], 1)
    obs_cam = np.concatenate([np.sort(rng.choice(n_p, size=k, replace=False)) for k in ks])
    obs_pt = np.repeat(np.arange(ks.size), ks)
    X = rng.uniform(-2.0, 2.0, size=(ks.size, 3))
    uv, Pz, _ = _project_true(Rs, ts, intr, obs_cam, X[obs_pt])
    assert np.all(Pz < 0)
    cams_true = np.concatenate([matrix_to_rotvec(Rs), ts, intr], 1)
    cams_init = _perturb_poses(Rs, ts, intr, rng, cam_noise, 5 * cam_noise)
    return dict(cfg=0, seed=seed, cameras_true=cams_true, points_true=X, cameras_init=cams_init,
                points_init=X + rng.normal(0, pt_noise, X.shape), obs_cam=obs_cam.astype(np.int32),
                obs_pt=obs_pt.astype(np.int32), obs_uv=uv + rng.normal(0, 1.0, uv.shape), lm_iters=5)
