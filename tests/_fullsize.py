"""Helpers of the full-size GPU parity tests (data selection and rotation-invariant comparisons;
no arithmetic of the method)."""
import numpy as np

LAM = 1e-4  # lambda0: the damping the bench's first marginalization folds in


def relf(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _sample_landmarks(k, n, seed):
    """n random landmarks, the 3 longest tracks and one landmark per kernel-bucket boundary."""
    rng = np.random.default_rng(seed)
    idx = set(rng.choice(len(k), size=min(n, len(k)), replace=False).tolist())
    idx |= set(np.argsort(k)[-3:].tolist())
    for kb in (2, 3, 4, 5, 8, 9, 16, 17, 32, 33, 64, 65, 128, 129, 256, 257, 512, 513):
        hit = np.flatnonzero(k == kb)
        if hit.size:
            idx.add(int(hit[0]))
    return sorted(idx)


def _sub_problem(p, lms):
    """The landmarks `lms` (re-indexed 0..m-1) with all their observations and ALL cameras."""
    lms = np.asarray(lms)
    sel = np.isin(p["obs_pt"], lms)
    remap = np.full(p["points_init"].shape[0], -1, np.int64)
    remap[lms] = np.arange(lms.size)
    return dict(cameras_init=p["cameras_init"], points_init=p["points_init"][lms],
                obs_cam=p["obs_cam"][sel], obs_pt=remap[p["obs_pt"][sel]].astype(np.int32),
                obs_uv=p["obs_uv"][sel])


def _reduced(B, k):
    return B[3:, :9 * k], B[3:, -1]


def _cmp_block(Bg, Bo, k, spg=None, spo=None, rng=None):
    """Rotation-invariant comparison (reading C16) of one landmark block: R1^T R1 and the Gram of
    the reduced rows (A | q) (Gram probes for k > 64), pose columns unscaled first when spg / spo
    (each side's own S_p) are given.  Returns (|dG|^2, |G|^2) of the reduced rows for the
    sample-level bar; asserts a loose per-block bound (1e-2: FP32 error of a single block grows
    with the conditioning of its J_l, e.g. two-view tracks with a short baseline)."""
    assert np.all(Bg[3:, 9 * k:9 * k + 3] == 0.0)
    R1g, R1o = Bg[:3, 9 * k:9 * k + 3], Bo[:3, 9 * k:9 * k + 3]
    assert relf(R1g.T @ R1g, R1o.T @ R1o) <= 1e-2
    Ag, qg = _reduced(Bg, k)
    Ao, qo = _reduced(Bo, k)
    if spg is not None:
        Ag, Ao = Ag / spg[None, :], Ao / spo[None, :]
    Mg, Mo = np.concatenate([Ag, qg[:, None]], 1), np.concatenate([Ao, qo[:, None]], 1)
    if k <= 64:
        dg, go = Mg.T @ Mg - Mo.T @ Mo, Mo.T @ Mo
    else:  # Gram probes (the 9k x 9k Gram of a long track is large)
        Z = rng.normal(size=(9 * k + 1, 3))
        go = Mo.T @ (Mo @ Z)
        dg = Mg.T @ (Mg @ Z) - go
    e2, n2 = float((dg ** 2).sum()), float((go ** 2).sum())
    assert e2 <= 1e-4 * n2, (k, np.sqrt(e2 / n2))
    return e2, n2


def _blocks_bar(errs):
    """Sample-level bar: relative Frobenius error of the sampled blocks' reduced Grams <= 1e-4
    (the north_star's reduced-system bar applied to the sum of squares over the sample)."""
    e2 = sum(e for e, _ in errs)
    n2 = sum(n for _, n in errs)
    assert np.sqrt(e2 / n2) <= 1e-4, np.sqrt(e2 / n2)


def _lm_sp(sp, cams):
    return np.concatenate([sp[9 * c:9 * c + 9] for c in cams])


def oracle_reduced_dense(o, lam):
    """H~ = sum_j A_j^T A_j + lam D_p^2 and b~ = sum_j A_j^T q_j (Eq. cg_mult; the
    definition), assembled with numpy BLAS from the oracle's marginalized + damped landmark blocks
    (a read-only view of its block arena), landmarks of equal track length batched.  The oracle's
    own orc_reduced_dense is the same sum, pinned on small problems against the explicit Schur
    complement, but too slow for configs 3-4."""
    N = 9 * o.n_p
    H = np.zeros((N, N))
    b = np.zeros(N)
    arena, off = o.block_arena()
    lp, cc = o.lm_ptr, o.csr_cam
    k_all = np.diff(lp)
    for k in np.unique(k_all):
        k = int(k)
        js = np.flatnonzero(k_all == k)
        R, W = 2 * k + 3, 9 * k + 4
        for c0 in range(0, js.size, max(1, (1 << 27) // (R * W))):  # chunks of <= 1 GB
            jj = js[c0:c0 + max(1, (1 << 27) // (R * W))]
            X = arena[off[jj][:, None] + np.arange(R * W)[None, :]].reshape(jj.size, R, W)
            A, q = np.ascontiguousarray(X[:, 3:, :9 * k]), np.ascontiguousarray(X[:, 3:, -1])
            G = np.matmul(A.transpose(0, 2, 1), A)  # (contiguous operands: one BLAS call per landmark)
            g = np.matmul(A.transpose(0, 2, 1), q[:, :, None])[:, :, 0]
            cams = cc[lp[jj][:, None] + np.arange(k)[None, :]]
            for n in range(jj.size):
                c = cams[n]
                if c[-1] - c[0] == k - 1:  # consecutive cameras (the street geometry): a dense slice
                    s0 = 9 * int(c[0])
                    H[s0:s0 + 9 * k, s0:s0 + 9 * k] += G[n]
                    b[s0:s0 + 9 * k] += g[n]
                else:
                    idx = (9 * c[:, None] + np.arange(9)).ravel()
                    H[np.ix_(idx, idx)] += G[n]
                    b[idx] += g[n]
    H[np.diag_indices(N)] += lam * o.scaling()[1]
    return H, b
