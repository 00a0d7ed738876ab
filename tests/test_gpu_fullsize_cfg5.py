"""GPU parity at BASELINE.json's full size for config 5 (final13682-shaped: 13682 cameras, 4.46M
landmarks, 30M observations, k up to 1727; 131.7 GB of FP32 landmark blocks on one GPU), in the
launch configuration bench.py times.  See test_gpu_fullsize.py for the method: the FP64 oracle
cannot hold the 263 GB of FP64 blocks, so it computes E and every scaling / damping entry of the
full problem (orc_scaling, no blocks) and, on sub-problems it can hold, sampled landmark blocks
and sampled H~ columns, compared camera-unscaled (Q^_2 depends only on the landmark's own
(J_l S_l, D_l), so S_p^-1 A_j^T A_j S_p^-1 and a camera's unscaled Schur column do not depend on
landmarks outside the sub-problem).  The LM steps are checked through the oracle's E
at the GPU's states."""
import numpy as np
import pytest

import oracle
from paper_2103_01843_b200 import synth
from _fullsize import LAM, _blocks_bar, _cmp_block, _lm_sp, _sample_landmarks, _sub_problem, relf

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cfg5():
    from paper_2103_01843_b200.rba import Solver
    p = synth.make_problem(5)
    s = Solver(p)
    s.linearize()
    s.marginalize(LAM)
    yield p, s
    s.close()


def test_cfg5_linearize_full(cfg5):
    """E and every scaling / damping entry of the full 30M-observation problem."""
    p, s = cfg5
    o = oracle.Oracle(p)
    o.linearize_scaling()
    assert abs(s.cost() - o.cost()) <= 1e-5 * o.cost()
    for g, r in zip(s.scaling(), o.scaling()):
        assert relf(g, r) <= 1e-4


def test_cfg5_blocks_sampled(cfg5):
    p, s = cfg5
    k = np.bincount(p["obs_pt"])
    lms = _sample_landmarks(k, 40, 5)
    sub = _sub_problem(p, lms)
    o = oracle.Oracle(sub)
    o.linearize()
    o.marginalize()
    o.damp(LAM)
    spg, spo = s.scaling()[0], o.scaling()[0]
    rng = np.random.default_rng(7)
    errs = []
    for jj, j in enumerate(lms):
        cams = np.sort(p["obs_cam"][p["obs_pt"] == j])
        errs.append(_cmp_block(s.block(j), o.block(jj), int(k[j]), _lm_sp(spg, cams), _lm_sp(spo, cams), rng))
    _blocks_bar(errs)


def test_cfg5_reduced_columns_sampled(cfg5):
    """Unscaled columns S^-1 (H~ - lam D_p^2) S^-1 e_i of the reduced camera system for sampled
    cameras, against an oracle sub-problem holding every landmark of that camera."""
    p, s = cfg5
    N = 9 * p["cameras_init"].shape[0]
    spg, Dpg = s.scaling()[:2]
    rng = np.random.default_rng(11)
    for cam in rng.choice(p["cameras_init"].shape[0], size=3, replace=False):
        i = 9 * int(cam) + int(rng.integers(9))
        lms = np.unique(p["obs_pt"][p["obs_cam"] == cam])
        o = oracle.Oracle(_sub_problem(p, lms))
        o.linearize()
        o.marginalize()
        o.damp(LAM)
        spo, Dpo = o.scaling()[:2]
        e = np.zeros(N)
        e[i] = 1.0 / spg[i]
        g = s.matvec(torch.tensor(e, dtype=torch.float32, device="cuda")).double().cpu().numpy()
        g = (g - LAM * Dpg * e) / spg
        e[i] = 1.0 / spo[i]
        r = (o.matvec(e) - LAM * Dpo * e) / spo
        assert relf(g, r) <= 1e-4, (cam, i)
        del o


def test_cfg5_lm_costs(cfg5):
    """Two LM iterations at full size: never indefinite, and the cost the GPU reports after each
    decision equals the oracle's E (Eq. ba_energy) at the GPU's state; accepted steps decrease E."""
    p, s = cfg5
    o = oracle.Oracle(p)
    for i in range(2):
        r = s.lm_step()
        assert r["pcg_reason"] != 2
        cams, pts = s.state()
        o.set_state(cams, pts)
        assert abs(r["cost_after"] - o.cost()) <= 1e-4 * o.cost(), (i, r)
        if r["accepted"]:
            assert r["cost_after"] < r["cost"]
