"""CPU-side checks of the C ABI (no compute calls without a GPU): every symbol declared in
include/rba.h is exported by librba.so, the host planner (LPT landmark sharding) is a
deterministic balanced partition, and host-side validation rejects bad problems with the documented
status codes before touching the device."""
import os
import re

import numpy as np
import pytest

from paper_2103_01843_b200 import rba, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "rba.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rba_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    names = _header_functions()
    assert len(names) >= 20
    lib = rba.lib()
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(rba.EXPORTED) == names


def test_default_options():
    o = rba.rba_default_options()
    assert (o.lambda0, o.pcg_rel_tol, o.pcg_max_iters, o.min_rel_decrease) == (1e-4, 1e-2, 500, 1e-3)
    assert (o.diag_min, o.diag_max, o.world, o.rank) == (1e-6, 1e32, 1, 0)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_plan_shards_lpt(world):
    rng = np.random.default_rng(world)
    k = np.concatenate([rng.integers(2, 9, 5000), rng.integers(50, 400, 40)]).astype(np.int32)
    o1 = rba.rba_plan_shards(k, world)
    o2 = rba.rba_plan_shards(k, world)
    np.testing.assert_array_equal(o1, o2)  # deterministic: every rank computes the same partition
    assert o1.min() >= 0 and o1.max() < world
    if world == 1:
        assert not o1.any()
        return
    b = (2 * k.astype(np.int64) + 3) * (9 * k + 4)
    load = np.bincount(o1, weights=b, minlength=world)
    # LPT bound: max load <= mean + largest item
    assert load.max() <= b.sum() / world + b.max()


def _prob():
    return synth.make_random_small(3, n_p=4, n_l=6)


@pytest.mark.parametrize("mutate,status", [
    (lambda p: p.update(obs_pt=np.where(p["obs_pt"] == 0, 1, p["obs_pt"]).astype(np.int32)), rba.RBA_ERR_BAD_PROBLEM),
    (lambda p: p["obs_cam"].__setitem__(0, 99), rba.RBA_ERR_BAD_PROBLEM),
    (lambda p: p["cameras_init"].__setitem__((1, 6), -5.0), rba.RBA_ERR_BAD_PROBLEM),
    (lambda p: p["points_init"].__setitem__((2, 1), np.nan), rba.RBA_ERR_BAD_PROBLEM),
    (lambda p: p.update(obs_cam=np.r_[p["obs_cam"], p["obs_cam"][:1]].astype(np.int32),
                        obs_pt=np.r_[p["obs_pt"], p["obs_pt"][:1]].astype(np.int32),
                        obs_uv=np.r_[p["obs_uv"], p["obs_uv"][:1]]), rba.RBA_ERR_BAD_PROBLEM),
])
def test_create_rejects_bad_problems(mutate, status):
    """k < 2, index out of range, f <= 0, non-finite, duplicate (cam, pt) -> BAD_PROBLEM."""
    p = _prob()
    p = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in p.items()}
    mutate(p)
    with pytest.raises(rba.RBAError) as ei:
        rba.rba_create(p["cameras_init"], p["points_init"], p["obs_cam"], p["obs_pt"], p["obs_uv"])
    assert ei.value.status == status


def _one_track(k):
    """One landmark seen by k distinct cameras (the track-length limits)."""
    rng = np.random.default_rng(k)
    cams = np.zeros((k, 9))
    cams[:, 3:6] = rng.normal(0, 1, (k, 3))
    cams[:, 5] = 10.0
    cams[:, 6] = 500.0
    return (cams, np.zeros((1, 3)), np.arange(k, dtype=np.int32), np.zeros(k, np.int32),
            rng.normal(0, 1, (k, 2)))


@pytest.mark.parametrize("k,precision", [(3073, 0), (1025, 1)])
def test_create_rejects_tracks_beyond_kmax(k, precision):
    """Track lengths above KMAX (3072) / KMAX64 (1024, sqrt-BA-64) are BAD_PROBLEM, checked on the
    host before any device work."""
    o = rba.rba_default_options()
    o.precision = precision
    with pytest.raises(rba.RBAError) as ei:
        rba.rba_create(*_one_track(k), o)
    assert ei.value.status == rba.RBA_ERR_BAD_PROBLEM
    assert str(k) in str(ei.value)


def test_create_rejects_bad_options():
    p = _prob()
    o = rba.rba_default_options()
    o.world, o.rank = 2, 5
    with pytest.raises(rba.RBAError) as ei:
        rba.rba_create(p["cameras_init"], p["points_init"], p["obs_cam"], p["obs_pt"], p["obs_uv"], o)
    assert ei.value.status == rba.RBA_ERR_INVALID_ARG


def test_layout_constants_match_paper_block_size():
    """The arena stores the logical (2k+3) x (9k+4) block per landmark: R2 = 2k x 9k
    (packed without padding for k <= 32; 4-row tiles for k > 32, so odd k pads 2 zero rows), R1
    (3 x 9k) + TL ((2k+3) x 4) + G (12) in the side region (16-byte alignment padding)."""
    pad4 = lambda x: (x + 3) // 4 * 4
    for k in list(range(2, 40)) + [64, 100, 257, 400, 512]:
        r2 = 18 * k * k if k <= 32 else 36 * k * ((k + 1) // 2)
        side = pad4(27 * k) + 4 * (2 * k + 3) + 12
        logical = (2 * k + 3) * (9 * k + 4) + 12
        extra = r2 + side - logical
        assert 0 <= extra <= 3 + (18 * k if (k > 32 and k % 2) else 0)


def test_null_context_and_bad_arguments_are_rejected_without_a_gpu():
    """Every entry point added for the device-side LM loop, the replay rule and the measurement
    hooks validates its arguments on the host: a null context / null output is INVALID_ARG."""
    import ctypes as C
    L = rba.lib()
    d, i64, n = C.c_double(), C.c_int64(), C.c_int()
    assert L.rba_lm_step(None, None) == rba.RBA_ERR_INVALID_ARG
    assert L.rba_lm_solve(None, 5, 1e-6, None, C.byref(n)) == rba.RBA_ERR_INVALID_ARG
    assert L.rba_set_lm(None, 1e-4, 2.0) == rba.RBA_ERR_INVALID_ARG
    assert L.rba_get_lm(None, C.byref(d), C.byref(d), C.byref(i64)) == rba.RBA_ERR_INVALID_ARG
    assert L.rba_set_pcg_limits(None, 1e-2, 500) == rba.RBA_ERR_INVALID_ARG
    assert L.rba_device_bytes(None, C.byref(i64)) == rba.RBA_ERR_INVALID_ARG
    assert L.rba_plan_bytes(None, C.byref(d), C.byref(d)) == rba.RBA_ERR_INVALID_ARG
    assert L.rba_get_info(None, C.byref(rba.rba_info())) == rba.RBA_ERR_INVALID_ARG
    assert L.rba_checksums(None, (C.c_uint64 * 4)()) == rba.RBA_ERR_INVALID_ARG
    assert L.rba_get_precond(None, None) == rba.RBA_ERR_INVALID_ARG


def test_deterministic_option_validated_on_the_host():
    """deterministic = 1 only for dense FP32 sqrt-BA (rba.h), rejected before any device work."""
    p = _prob()
    for field, value in (("storage", 1), ("precision", 1), ("solver", 1)):
        o = rba.rba_default_options()
        o.deterministic = 1
        setattr(o, field, value)
        with pytest.raises(rba.RBAError) as ei:
            rba.rba_create(p["cameras_init"], p["points_init"], p["obs_cam"], p["obs_pt"], p["obs_uv"], o)
        assert ei.value.status == rba.RBA_ERR_INVALID_ARG
