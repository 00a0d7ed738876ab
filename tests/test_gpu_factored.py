"""GPU parity of the factored landmark storage (Householder vectors, compact-WY
T, the 6 damping Givens and the scaled J_p instead of the dense (2k+3) x (9k+4) block
"never ... store ... Q").  The reduced camera system it applies is the same matrix (exact algebra),
so the bars are the north_star's: H~ <= 1e-4 relative Frobenius, b~ <= 1e-4, PCG solution <= 1e-3,
cost after each of 5 LM iterations <= 1e-4, against the FP64 oracle on the same inputs."""
import numpy as np
import pytest

import oracle
from _lm import lm_parity
from paper_2103_01843_b200 import synth
from paper_2103_01843_b200.rba import RBA_STORAGE_DENSE, RBA_STORAGE_FACTORED

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def relf(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _solver(p, **kw):
    from paper_2103_01843_b200.rba import Solver
    return Solver(p, storage=RBA_STORAGE_FACTORED, **kw)


def _oracle(p, lam):
    o = oracle.Oracle(p)
    o.linearize()
    o.marginalize()
    o.damp(lam)
    return o


def _mv(s, v):
    return s.matvec(torch.tensor(v, dtype=torch.float32, device="cuda")).double().cpu().numpy()


@pytest.mark.parametrize("lam", [0.0, 1e-4, 1.0])
def test_factored_reduced_system_config1(lam):
    p = synth.make_problem(1)
    s = _solver(p)
    s.linearize()
    s.marginalize(lam)
    o = _oracle(p, lam)
    H, b = o.reduced_dense()
    N = 9 * o.n_p
    Hg = np.stack([_mv(s, np.eye(N)[i]) for i in range(N)], 1)
    assert relf(Hg, H) <= 1e-4
    s.pcg()
    assert relf(s.rhs(), b) <= 1e-4


def test_factored_redamp():
    """lambda changes at an unchanged linearization only re-damp (O(1) per landmark)."""
    p = synth.make_tracks(31, [2, 3, 5, 9, 17, 40, 120], n_p=150)
    s = _solver(p)
    s.linearize()
    s.marginalize(1e-3)
    s.marginalize(0.5)
    o = _oracle(p, 0.5)
    rng = np.random.default_rng(1)
    for _ in range(3):
        v = rng.normal(size=9 * o.n_p)
        assert relf(_mv(s, v), o.matvec(v)) <= 1e-4


def test_factored_all_buckets_and_huge():
    """Every group size (k = 2, 3-4, 5-8, 9-16, > 16) and long tracks up to k = 700."""
    rng = np.random.default_rng(5)
    ks = list(rng.integers(2, 40, 300)) + [64, 129, 300, 700]
    p = synth.make_tracks(37, ks, n_p=800)
    s = _solver(p)
    s.linearize()
    s.marginalize(1e-3)
    o = _oracle(p, 1e-3)
    for _ in range(3):
        v = rng.normal(size=9 * o.n_p)
        assert relf(_mv(s, v), o.matvec(v)) <= 1e-4
    s.pcg()
    assert o.precond_rhs() == 0
    assert relf(s.rhs(), o.rhs()) <= 1e-4


@pytest.mark.parametrize("cfg", [1, 2])
def test_factored_pcg_backsub_and_lm(cfg):
    p = synth.make_problem(cfg)
    s = _solver(p)
    s.linearize()
    s.marginalize(1e-4)
    o = _oracle(p, 1e-4)
    st = s.pcg()
    assert o.precond_rhs() == 0
    it, reason, _ = o.pcg(1e-2, 500)
    if st["iters"] == it:
        s.backsub()
        o.backsub()
        dp, dl = s.step()
        assert relf(dp, o.dp()) <= 1e-3
        assert relf(dl, o.dl()) <= 1e-3
    s.close()
    s = _solver(p)
    o = oracle.Oracle(p)
    lm_parity(s, o, 5)


def test_factored_matches_dense_at_config3():
    """Full-size config 3: the factored and the dense GPU products agree (same operator)."""
    from paper_2103_01843_b200.rba import Solver
    p = synth.make_problem(3)
    a = Solver(p, storage=RBA_STORAGE_DENSE)
    b = Solver(p, storage=RBA_STORAGE_FACTORED)
    for s in (a, b):
        s.linearize()
        s.marginalize(1e-4)
    rng = np.random.default_rng(2)
    for _ in range(3):
        v = rng.normal(size=9 * p["cameras_init"].shape[0])
        assert relf(_mv(b, v), _mv(a, v)) <= 1e-4
    la, lb = a.arena_bytes()[0], b.arena_bytes()[0]
    assert lb < la / 5
