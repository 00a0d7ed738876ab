"""BAL ingest and the paper's preprocessing (NEXT row f1), host code of librba (no GPU):
parse / write round trip, counts from the paper's problem-size table, error reporting with line
numbers, gauge normalization (median centre, MAD 100, residuals unchanged), seeded perturbation,
and the z-filter with landmark removal (hand-traced cases)."""
import numpy as np
import pytest

import oracle
from paper_2103_01843_b200 import rba, synth


def bal_text(p):
    """Format a problem dict as BAL text (test helper)."""
    lines = [f"{p['cameras_init'].shape[0]} {p['points_init'].shape[0]} {len(p['obs_cam'])}"]
    for c, j, (u, v) in zip(p["obs_cam"], p["obs_pt"], p["obs_uv"]):
        lines.append(f"{int(c)} {int(j)} {float(u)!r} {float(v)!r}")
    lines += [repr(float(x)) for x in p["cameras_init"].ravel()]
    lines += [repr(float(x)) for x in p["points_init"].ravel()]
    return "\n".join(lines) + "\n"


def test_parse_values_and_round_trip(tmp_path):
    p = synth.make_random_small(1, n_p=4, n_l=9)
    b = rba.BalProblem.parse(bal_text(p))
    q = b.as_problem()
    for key in ("cameras_init", "points_init", "obs_cam", "obs_pt", "obs_uv"):
        np.testing.assert_array_equal(q[key], p[key])
    f = tmp_path / "p.txt"
    b.write(str(f))
    q2 = rba.BalProblem.read(str(f)).as_problem()
    for key in q:
        np.testing.assert_array_equal(q2[key], q[key])


@pytest.mark.parametrize("n_p,n_l,n_obs", [(49, 7766, 31812), (16, 22106, 83718)])
def test_counts_from_paper_table(n_p, n_l, n_obs):
    """Problem sizes of the paper's appendix table (ladybug49, dubrovnik16)."""
    rng = np.random.default_rng(n_p)
    p = dict(cameras_init=rng.normal(size=(n_p, 9)), points_init=rng.normal(size=(n_l, 3)),
             obs_cam=rng.integers(0, n_p, n_obs).astype(np.int32), obs_pt=rng.integers(0, n_l, n_obs).astype(np.int32),
             obs_uv=rng.normal(size=(n_obs, 2)))
    q = rba.BalProblem.parse(bal_text(p)).as_problem()
    assert q["cameras_init"].shape == (n_p, 9) and q["points_init"].shape == (n_l, 3) and q["obs_cam"].shape == (n_obs,)


@pytest.mark.parametrize("text,line", [
    ("x 1 1\n", 1),
    ("1 1 1\n0 3 1.0 2.0\n", 2),            # landmark index out of range
    ("1 1 2\n0 0 1.0 2.0\n0 0 1.0\n", 4),   # truncated observation
    ("1 1 1\n0 0 1 2\n" + "0 " * 8 + "\n", 4),  # truncated camera block (ends at line 4)
])
def test_parse_errors_name_the_line(text, line):
    with pytest.raises(rba.RBAError) as e:
        rba.BalProblem.parse(text)
    assert e.value.status == rba.RBA_ERR_BAD_PROBLEM
    assert f"line {line}" in str(e.value)


def _one_camera(points):
    cams = np.array([[0, 0, 0, 0, 0, -500.0, 500, 0, 0]])
    n = len(points)
    return dict(cameras_init=cams, points_init=np.asarray(points, float), obs_cam=np.zeros(n, np.int32),
                obs_pt=np.arange(n, dtype=np.int32), obs_uv=np.zeros((n, 2)))


def test_normalize_hand_case():
    """{(0,0,0),(2,0,0),(4,0,0)}: median (2,0,0), L1 deviations 2,0,2 -> MAD 2 -> scale 50."""
    b = rba.BalProblem.parse(bal_text(_one_camera([[0, 0, 0], [2, 0, 0], [4, 0, 0]])))
    b.normalize(100.0)
    np.testing.assert_allclose(b.as_problem()["points_init"], [[-100, 0, 0], [0, 0, 0], [100, 0, 0]], atol=1e-12)


def test_normalize_keeps_residuals_and_is_idempotent():
    p = synth.make_random_small(2, n_p=5, n_l=30)
    b = rba.BalProblem.parse(bal_text(p))
    b.normalize(100.0)
    q = b.as_problem()
    med = np.median(q["points_init"], 0)
    np.testing.assert_allclose(med, 0, atol=1e-9)
    np.testing.assert_allclose(np.median(np.abs(q["points_init"] - med).sum(1)), 100.0, rtol=1e-12)
    for i in range(len(p["obs_cam"])):   # reprojection (oracle's camera model) unchanged
        c, j = p["obs_cam"][i], p["obs_pt"][i]
        uv0, _ = oracle.project(p["cameras_init"][c], p["points_init"][j])
        uv1, _ = oracle.project(q["cameras_init"][c], q["points_init"][j])
        np.testing.assert_allclose(uv1, uv0, rtol=0, atol=1e-9)
    b.normalize(100.0)
    q2 = b.as_problem()
    np.testing.assert_allclose(q2["points_init"], q["points_init"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(q2["cameras_init"], q["cameras_init"], rtol=0, atol=1e-9)
    with pytest.raises(rba.RBAError):
        rba.BalProblem.parse(bal_text(_one_camera([[1, 1, 1], [1, 1, 1], [1, 1, 1]]))).normalize(100.0)


def test_perturb_seeded():
    p = synth.make_random_small(3, n_p=6, n_l=40)
    t = bal_text(p)
    a = rba.BalProblem.parse(t).perturb(0, 0, 0, 7).as_problem()
    for key in a:
        np.testing.assert_array_equal(a[key], p[key])
    x = rba.BalProblem.parse(t).perturb(0.01, 0.05, 0.05, 7).as_problem()
    y = rba.BalProblem.parse(t).perturb(0.01, 0.05, 0.05, 7).as_problem()
    z = rba.BalProblem.parse(t).perturb(0.01, 0.05, 0.05, 8).as_problem()
    for key in x:
        np.testing.assert_array_equal(x[key], y[key])
    assert np.any(x["points_init"] != z["points_init"])
    # noise statistics on many points: N(0, sigma^2) per coordinate
    big = _one_camera(np.zeros((20000, 3)))
    d = rba.BalProblem.parse(bal_text(big)).perturb(0, 0, 0.5, 11).as_problem()["points_init"].ravel()
    assert abs(d.mean()) < 0.02 and abs(d.std() - 0.5) < 0.01


def test_filter_hand_cases():
    # camera at the origin looking down -z: a point is in front iff z < 0 (depth -P_z = -z)
    cams = np.array([[0, 0, 0, 0, 0, 0, 500, 0, 0], [0, 0, 0, 0, 0, 0.5, 500, 0, 0.0]])
    pts = np.array([[0, 0, -5.0], [0, 0, -0.2], [1, 1, -3.0]])
    # lm0: two valid obs; lm1: obs of cam 1 has depth -(-0.2+0.5) < 0 -> 1 left -> removed; lm2: valid
    p = dict(cameras_init=cams, points_init=pts, obs_cam=np.array([0, 1, 0, 1, 0, 1], np.int32),
             obs_pt=np.array([0, 0, 1, 1, 2, 2], np.int32), obs_uv=np.arange(12.0).reshape(6, 2))
    b = rba.BalProblem.parse(bal_text(p))
    ro, rp = b.filter(1e-8)
    q = b.as_problem()
    assert (ro, rp) == (2, 1)
    np.testing.assert_array_equal(q["points_init"], pts[[0, 2]])
    np.testing.assert_array_equal(q["obs_pt"], [0, 0, 1, 1])
    np.testing.assert_array_equal(q["obs_uv"], p["obs_uv"][[0, 1, 4, 5]])
    # all valid -> unchanged
    s = synth.make_random_small(4)
    b = rba.BalProblem.parse(bal_text(s))
    assert b.filter(1e-8) == (0, 0)
    np.testing.assert_array_equal(b.as_problem()["obs_cam"], s["obs_cam"])


def test_parse_is_bounded_by_len():
    """rba_bal_parse reads at most `len` bytes: a buffer that is not NUL-terminated (here followed
    by more digits in memory) parses exactly as its first `len` bytes (strtod overran)."""
    import ctypes as C
    text = b"1 2 2\n0 0 1.5 2.5\n0 1 3.5 4.5\n" + b"\n".join(b"0.25" for _ in range(9)) + b"\n1 2 3\n4 5 6"
    tail = b"789123"  # would extend the last number to 6789123 if the parser ran past len
    raw = C.create_string_buffer(text + tail, len(text) + len(tail))
    b = rba.rba_bal()
    assert rba.lib().rba_bal_parse(C.cast(raw, C.c_char_p), len(text), C.byref(b)) == rba.RBA_OK
    p = rba.BalProblem(b).as_problem()
    assert p["points_init"][1, 2] == 6.0
    assert np.allclose(p["obs_uv"], [[1.5, 2.5], [3.5, 4.5]])


def test_read_gzip(tmp_path):
    """rba_bal_read takes gzip-compressed BAL files (the distribution format) as well as plain text."""
    import gzip
    p = synth.make_random_small(3, n_p=4, n_l=6)
    plain = tmp_path / "p.txt"
    b = rba.BalProblem.parse(bal_text(p))
    b.write(str(plain))
    gz = tmp_path / "p.txt.gz"
    gz.write_bytes(gzip.compress(plain.read_bytes()))
    a, z = rba.BalProblem.read(str(plain)).as_problem(), rba.BalProblem.read(str(gz)).as_problem()
    for key in a:
        assert np.array_equal(a[key], z[key]), key
