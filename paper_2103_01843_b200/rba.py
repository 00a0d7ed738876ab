"""Thin ctypes binding of librba.so (include/rba.h); argument marshalling only.

Function names mirror the C ABI.  Every step of the method runs in librba's CUDA kernels; this
module never computes any part of it and there is no CPU fallback: if the extension is missing,
importing fails loudly.  PyTorch is used for device memory (the caching allocator is passed in
as rba_options.alloc/free), the CUDA stream, and -- in bench.py -- the process group that
broadcasts the NCCL unique id.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RBA_LIB") or os.path.join(_HERE, "librba.so")  # RBA_LIB: build variants (tools/)

RBA_OK, RBA_ERR_INVALID_ARG, RBA_ERR_BAD_PROBLEM, RBA_ERR_STATE, RBA_ERR_OOM, RBA_ERR_CUDA, RBA_ERR_NCCL = range(7)
STATUS_NAMES = ["OK", "INVALID_ARG", "BAD_PROBLEM", "STATE", "OOM", "CUDA", "NCCL"]
KERNELS = {"linearize": 0, "marginalize": 1, "damp": 2, "precond": 3, "matvec": 4, "pcg": 5, "backsub": 6,
           "cost": 7}

_ALLOC_T = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
_FREE_T = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class rba_options(C.Structure):
    _fields_ = [("device", C.c_int), ("stream", C.c_void_p), ("world", C.c_int), ("rank", C.c_int),
                ("nccl_unique_id", C.c_void_p), ("lambda0", C.c_double), ("pcg_rel_tol", C.c_double),
                ("pcg_max_iters", C.c_int), ("min_rel_decrease", C.c_double), ("diag_min", C.c_double),
                ("diag_max", C.c_double), ("alloc", _ALLOC_T), ("free", _FREE_T), ("alloc_ctx", C.c_void_p),
                ("huber_delta", C.c_double), ("solver", C.c_int), ("storage", C.c_int), ("precision", C.c_int),
                ("deterministic", C.c_int)]
RBA_PRECISION_FP32, RBA_PRECISION_FP64 = 0, 1
RBA_STORAGE_DENSE, RBA_STORAGE_FACTORED = 0, 1
RBA_SOLVER_SQRTBA, RBA_SOLVER_EXPLICIT_SC32, RBA_SOLVER_EXPLICIT_SC64 = 0, 1, 2


class rba_info(C.Structure):
    _fields_ = [("lm_graph", C.c_int), ("pcg_graph", C.c_int), ("nccl", C.c_int), ("deterministic", C.c_int),
                ("n_landmarks", C.c_int64), ("n_observations", C.c_int64)]


class rba_pcg_stats(C.Structure):
    _fields_ = [("iters", C.c_int), ("reason", C.c_int), ("rel_residual", C.c_double)]


class rba_lm_report(C.Structure):
    _fields_ = [("iter", C.c_int64), ("accepted", C.c_int), ("pcg_iters", C.c_int), ("pcg_reason", C.c_int),
                ("cost", C.c_double), ("cost_trial", C.c_double), ("cost_after", C.c_double),
                ("model", C.c_double), ("rho", C.c_double), ("lambda_", C.c_double), ("lambda_next", C.c_double),
                ("relinearized", C.c_int), ("status", C.c_int), ("t_linearize_ms", C.c_double),
                ("t_marginalize_ms", C.c_double), ("t_precond_ms", C.c_double), ("t_pcg_ms", C.c_double),
                ("t_trial_ms", C.c_double), ("t_total_ms", C.c_double), ("device_bytes", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class rba_bal(C.Structure):
    _fields_ = [("n_cams", C.c_int64), ("n_points", C.c_int64), ("n_obs", C.c_int64),
                ("cameras", C.POINTER(C.c_double)), ("points", C.POINTER(C.c_double)),
                ("obs_uv", C.POINTER(C.c_double)), ("obs_cam", C.POINTER(C.c_int32)),
                ("obs_pt", C.POINTER(C.c_int32))]


class RBAError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"librba {STATUS_NAMES[status] if 0 <= status < 7 else status}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"librba.so not built ({LIB_PATH}); run __graft_entry__.build()")
    lib = C.CDLL(LIB_PATH)
    P, I64, D, I = C.c_void_p, C.c_int64, C.c_double, C.c_int
    sig = {
        "rba_default_options": (None, [C.POINTER(rba_options)]),
        "rba_create": (I, [P, I64, P, I64, P, P, P, I64, C.POINTER(rba_options), C.POINTER(C.c_void_p)]),
        "rba_destroy": (I, [P]),
        "rba_linearize": (I, [P]),
        "rba_marginalize_qr": (I, [P, D]),
        "rba_pcg_solve": (I, [P, C.POINTER(rba_pcg_stats)]),
        "rba_backsubstitute": (I, [P]),
        "rba_cost": (I, [P, I, C.POINTER(C.c_double)]),
        "rba_lm_step": (I, [P, C.POINTER(rba_lm_report)]),
        "rba_lm_solve": (I, [P, I, D, P, C.POINTER(I)]),
        "rba_set_lm": (I, [P, D, D]),
        "rba_get_lm": (I, [P, C.POINTER(D), C.POINTER(D), C.POINTER(I64)]),
        "rba_set_pcg_limits": (I, [P, D, I]),
        "rba_device_bytes": (I, [P, C.POINTER(I64)]),
        "rba_plan_bytes": (I, [P, C.POINTER(D), C.POINTER(D)]),
        "rba_get_info": (I, [P, C.POINTER(rba_info)]),
        "rba_checksums": (I, [P, C.POINTER(C.c_uint64)]),
        "rba_get_state": (I, [P, P, P]),
        "rba_set_state": (I, [P, P, P]),
        "rba_reset_lm": (I, [P]),
        "rba_matvec": (I, [P, P, P]),
        "rba_get_rhs": (I, [P, P]),
        "rba_get_precond": (I, [P, P]),
        "rba_get_step": (I, [P, P, P]),
        "rba_get_scaling": (I, [P, P, P, P, P]),
        "rba_export_block": (I, [P, I64, P, I64, C.POINTER(I64), C.POINTER(I64)]),
        "rba_arena_bytes": (I, [P, C.POINTER(I64), C.POINTER(I64)]),
        "rba_kernel_launches": (I, [P, C.POINTER(I64)]),
        "rba_profile": (I, [P, I]),
        "rba_profile_get": (I, [P, I, C.POINTER(D), C.POINTER(I64), C.POINTER(D)]),
        "rba_plan_shards": (I, [P, I64, I, P]),
        "rba_nccl_unique_id": (I, [P]),
        "rba_last_error": (C.c_char_p, []),
        "rba_bal_parse": (I, [C.c_char_p, C.c_size_t, C.POINTER(rba_bal)]),
        "rba_bal_read": (I, [C.c_char_p, C.POINTER(rba_bal)]),
        "rba_bal_write": (I, [C.c_char_p, C.POINTER(rba_bal)]),
        "rba_bal_normalize": (I, [C.POINTER(rba_bal), D]),
        "rba_bal_perturb": (I, [C.POINTER(rba_bal), D, D, D, C.c_uint64]),
        "rba_bal_filter": (I, [C.POINTER(rba_bal), D, C.POINTER(I64), C.POINTER(I64)]),
        "rba_bal_free": (None, [C.POINTER(rba_bal)]),
        "rba_bal_last_error": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()
EXPORTED = ["rba_default_options", "rba_create", "rba_destroy", "rba_linearize", "rba_marginalize_qr",
            "rba_pcg_solve", "rba_backsubstitute", "rba_cost", "rba_lm_step", "rba_lm_solve", "rba_get_state",
            "rba_set_state", "rba_reset_lm", "rba_set_lm", "rba_get_lm", "rba_set_pcg_limits", "rba_device_bytes", "rba_plan_bytes", "rba_get_info", "rba_checksums",
            "rba_matvec", "rba_get_rhs", "rba_get_precond", "rba_get_step", "rba_get_scaling", "rba_export_block", "rba_arena_bytes",
            "rba_kernel_launches", "rba_profile", "rba_profile_get", "rba_plan_shards", "rba_nccl_unique_id",
            "rba_last_error", "rba_bal_parse", "rba_bal_read", "rba_bal_write", "rba_bal_normalize",
            "rba_bal_perturb", "rba_bal_filter", "rba_bal_free", "rba_bal_last_error"]


def lib():
    return _lib


def _check(status):
    if status != RBA_OK:
        raise RBAError(status, _lib.rba_last_error().decode())


def _p(a):
    return C.c_void_p(a.ctypes.data) if isinstance(a, np.ndarray) else C.c_void_p(a)


# ------------------------------------------------------------------------- ABI-named wrappers
def rba_default_options() -> rba_options:
    o = rba_options()
    _lib.rba_default_options(C.byref(o))
    return o


def rba_create(cameras, points, obs_cam, obs_pt, obs_uv, opt: rba_options | None = None):
    cameras = np.ascontiguousarray(cameras, np.float64)
    points = np.ascontiguousarray(points, np.float64)
    obs_cam = np.ascontiguousarray(obs_cam, np.int32)
    obs_pt = np.ascontiguousarray(obs_pt, np.int32)
    obs_uv = np.ascontiguousarray(obs_uv, np.float64)
    h = C.c_void_p()
    _check(_lib.rba_create(_p(cameras), cameras.shape[0], _p(points), points.shape[0], _p(obs_cam), _p(obs_pt),
                           _p(obs_uv), obs_cam.shape[0], C.byref(opt) if opt is not None else None, C.byref(h)))
    return h


def rba_destroy(h):
    _check(_lib.rba_destroy(h))


def rba_linearize(h):
    _check(_lib.rba_linearize(h))


def rba_marginalize_qr(h, lam):
    _check(_lib.rba_marginalize_qr(h, float(lam)))


def rba_pcg_solve(h) -> dict:
    st = rba_pcg_stats()
    _check(_lib.rba_pcg_solve(h, C.byref(st)))
    return {"iters": st.iters, "reason": st.reason, "rel_residual": st.rel_residual}


def rba_backsubstitute(h):
    _check(_lib.rba_backsubstitute(h))


def rba_cost(h, at_trial=False) -> float:
    v = C.c_double()
    _check(_lib.rba_cost(h, int(bool(at_trial)), C.byref(v)))
    return v.value


def rba_lm_step(h) -> dict:
    r = rba_lm_report()
    _check(_lib.rba_lm_step(h, C.byref(r)))
    return r.as_dict()


def rba_lm_solve(h, max_iters: int, ftol: float = 1e-6) -> list:
    reps = (rba_lm_report * max(1, int(max_iters)))()
    n = C.c_int()
    _check(_lib.rba_lm_solve(h, int(max_iters), float(ftol), reps, C.byref(n)))
    return [reps[i].as_dict() for i in range(n.value)]


def rba_set_lm(h, lam, nu=2.0):
    _check(_lib.rba_set_lm(h, float(lam), float(nu)))


def rba_get_lm(h):
    lam, nu, it = C.c_double(), C.c_double(), C.c_int64()
    _check(_lib.rba_get_lm(h, C.byref(lam), C.byref(nu), C.byref(it)))
    return lam.value, nu.value, it.value


def rba_set_pcg_limits(h, rel_tol, max_iters):
    _check(_lib.rba_set_pcg_limits(h, float(rel_tol), int(max_iters)))


def rba_device_bytes(h) -> int:
    n = C.c_int64()
    _check(_lib.rba_device_bytes(h, C.byref(n)))
    return n.value


def rba_plan_bytes(h):
    a, b = C.c_double(), C.c_double()
    _check(_lib.rba_plan_bytes(h, C.byref(a), C.byref(b)))
    return a.value, b.value


def rba_get_info(h) -> dict:
    i = rba_info()
    _check(_lib.rba_get_info(h, C.byref(i)))
    return {k: getattr(i, k) for k, _ in i._fields_}


def rba_checksums(h) -> list:
    out = (C.c_uint64 * 4)()
    _check(_lib.rba_checksums(h, out))
    return list(out)


def rba_get_state(h, n_cams, n_points, out=None):
    """out: optional (cams (n_cams, 9), pts (n_points, 3)) C-contiguous float64 arrays to fill
    (e.g. views of pinned host memory)."""
    if out is None:
        cams, pts = np.zeros((n_cams, 9)), np.zeros((n_points, 3))
    else:
        cams, pts = out
        assert cams.dtype == pts.dtype == np.float64 and cams.flags.c_contiguous and pts.flags.c_contiguous
        assert cams.shape == (n_cams, 9) and pts.shape == (n_points, 3)
    _check(_lib.rba_get_state(h, _p(cams), _p(pts)))
    return cams, pts


def rba_set_state(h, cameras, points):
    cameras = np.ascontiguousarray(cameras, np.float64)
    points = np.ascontiguousarray(points, np.float64)
    _check(_lib.rba_set_state(h, _p(cameras), _p(points)))


def rba_reset_lm(h):
    _check(_lib.rba_reset_lm(h))


def rba_matvec(h, v_dev_ptr: int, out_dev_ptr: int):
    _check(_lib.rba_matvec(h, C.c_void_p(v_dev_ptr), C.c_void_p(out_dev_ptr)))


def rba_get_rhs(h, n_cams):
    b = np.zeros(9 * n_cams)
    _check(_lib.rba_get_rhs(h, _p(b)))
    return b


def rba_get_precond(h, n_cams):
    out = np.zeros((n_cams, 54))
    _check(_lib.rba_get_precond(h, _p(out)))
    return out


def rba_get_step(h, n_cams, n_points):
    dp, dl = np.zeros(9 * n_cams), np.zeros(3 * n_points)
    _check(_lib.rba_get_step(h, _p(dp), _p(dl)))
    return dp, dl


def rba_get_scaling(h, n_cams, n_points):
    sp, Dp2, sl, Dl2 = np.zeros(9 * n_cams), np.zeros(9 * n_cams), np.zeros(3 * n_points), np.zeros(3 * n_points)
    _check(_lib.rba_get_scaling(h, _p(sp), _p(Dp2), _p(sl), _p(Dl2)))
    return sp, Dp2, sl, Dl2


def rba_export_block(h, landmark):
    r, c = C.c_int64(), C.c_int64()
    _lib.rba_export_block(h, int(landmark), _p(np.zeros(1)), 0, C.byref(r), C.byref(c))  # shape query
    if r.value <= 0:
        _check(_lib.rba_export_block(h, int(landmark), _p(np.zeros(1)), 0, C.byref(r), C.byref(c)))
    buf = np.zeros((r.value, c.value))
    _check(_lib.rba_export_block(h, int(landmark), _p(buf), buf.size, C.byref(r), C.byref(c)))
    return buf


def rba_arena_bytes(h):
    a, b = C.c_int64(), C.c_int64()
    _check(_lib.rba_arena_bytes(h, C.byref(a), C.byref(b)))
    return a.value, b.value


def rba_kernel_launches(h) -> int:
    n = C.c_int64()
    _check(_lib.rba_kernel_launches(h, C.byref(n)))
    return n.value


def rba_profile(h, enable: bool):
    _check(_lib.rba_profile(h, int(bool(enable))))


def rba_profile_get(h, kernel):
    kid = KERNELS[kernel] if isinstance(kernel, str) else int(kernel)
    ms, n, by = C.c_double(), C.c_int64(), C.c_double()
    _check(_lib.rba_profile_get(h, kid, C.byref(ms), C.byref(n), C.byref(by)))
    return ms.value, n.value, by.value


def rba_plan_shards(k, world):
    k = np.ascontiguousarray(k, np.int32)
    owner = np.zeros(k.shape[0], np.int32)
    _check(_lib.rba_plan_shards(_p(k), k.shape[0], int(world), _p(owner)))
    return owner


def rba_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.rba_nccl_unique_id(buf))
    return buf.raw


def rba_last_error() -> str:
    return _lib.rba_last_error().decode()


# ------------------------------------------------------------------------- BAL ingest (f1)
def _bal_check(status):
    if status != RBA_OK:
        raise RBAError(status, _lib.rba_bal_last_error().decode())


class BalProblem:
    """A BAL problem owned by librba (host memory); every operation runs in librba's C++."""

    def __init__(self, b: rba_bal):
        self.b = b

    @classmethod
    def parse(cls, text: str | bytes):
        data = text.encode() if isinstance(text, str) else text
        b = rba_bal()
        _bal_check(_lib.rba_bal_parse(data, len(data), C.byref(b)))
        return cls(b)

    @classmethod
    def read(cls, path: str):
        b = rba_bal()
        _bal_check(_lib.rba_bal_read(os.fsencode(path), C.byref(b)))
        return cls(b)

    def write(self, path: str):
        _bal_check(_lib.rba_bal_write(os.fsencode(path), C.byref(self.b)))

    def normalize(self, target_mad: float = 100.0):
        _bal_check(_lib.rba_bal_normalize(C.byref(self.b), float(target_mad)))
        return self

    def perturb(self, sigma_rot: float, sigma_centre: float, sigma_point: float, seed: int):
        _bal_check(_lib.rba_bal_perturb(C.byref(self.b), float(sigma_rot), float(sigma_centre), float(sigma_point),
                                        int(seed) & 0xFFFFFFFFFFFFFFFF))
        return self

    def filter(self, z_min: float = 1e-8):
        ro, rp = C.c_int64(), C.c_int64()
        _bal_check(_lib.rba_bal_filter(C.byref(self.b), float(z_min), C.byref(ro), C.byref(rp)))
        return ro.value, rp.value

    def as_problem(self) -> dict:
        """Copies in the dict layout Solver / rba_create take (cameras_init, points_init, obs_*)."""
        b = self.b
        arr = lambda ptr, n, shape: np.ctypeslib.as_array(ptr, shape=(max(n, 1),))[:n].reshape(shape).copy()
        return dict(cameras_init=arr(b.cameras, 9 * b.n_cams, (b.n_cams, 9)),
                    points_init=arr(b.points, 3 * b.n_points, (b.n_points, 3)),
                    obs_cam=arr(b.obs_cam, b.n_obs, (b.n_obs,)), obs_pt=arr(b.obs_pt, b.n_obs, (b.n_obs,)),
                    obs_uv=arr(b.obs_uv, 2 * b.n_obs, (b.n_obs, 2)))

    def __del__(self):
        try:
            _lib.rba_bal_free(C.byref(self.b))
        except Exception:
            pass


def load_bal(path: str, normalize: bool = True, sigma_rot: float = 0.0, sigma_centre: float = 0.0,
             sigma_point: float = 0.0, seed: int = 0, z_min: float | None = 1e-8) -> dict:
    """BAL file -> problem dict with the paper's preprocessing: gauge normalization to
    median absolute deviation 100, seeded perturbation, z-filter."""
    p = BalProblem.read(path)
    if normalize:
        p.normalize(100.0)
    if sigma_rot or sigma_centre or sigma_point:
        p.perturb(sigma_rot, sigma_centre, sigma_point, seed)
    if z_min is not None:
        p.filter(z_min)
    return p.as_problem()


# ------------------------------------------------------------------------- convenience
class _TorchAllocator:
    """Routes librba's device allocations through torch's caching allocator."""

    def __init__(self, device, stream_ptr):
        import torch
        self.torch = torch
        self.device = device
        self.stream = stream_ptr
        self.alloc = _ALLOC_T(self._alloc)
        self.free = _FREE_T(self._free)

    def _alloc(self, nbytes, _ctx):
        try:
            return self.torch.cuda.caching_allocator_alloc(int(nbytes), self.device, self.stream)
        except Exception:  # OOM -> NULL -> RBA_ERR_OOM
            return None

    def _free(self, ptr, _ctx):
        torch = self.torch
        if torch is None or getattr(torch, "cuda", None) is None:  # interpreter shutdown
            return
        try:
            torch.cuda.caching_allocator_delete(ptr)
        except Exception:
            pass


class Solver:
    """One sqrt-BA problem on one GPU (or one landmark shard of a multi-GPU job)."""

    def __init__(self, prob: dict, device: int = 0, world: int = 1, rank: int = 0, nccl_id: bytes | None = None,
                 use_torch_alloc: bool = True, cams=None, pts=None, **opts):
        import torch
        self.opt = rba_default_options()
        self.opt.device = device
        self.opt.world, self.opt.rank = world, rank
        self._id = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        self.opt.nccl_unique_id = C.cast(self._id, C.c_void_p) if self._id is not None else None
        # librba runs on its own torch stream; device-pointer hooks order it against the caller's
        self.stream = torch.cuda.Stream(device)
        self.opt.stream = C.c_void_p(self.stream.cuda_stream)
        for k, v in opts.items():
            setattr(self.opt, k, v)
        self._alloc = None
        if use_torch_alloc:
            self._alloc = _TorchAllocator(device, self.stream.cuda_stream)
            self.opt.alloc, self.opt.free = self._alloc.alloc, self._alloc.free
        self.n_p = prob["cameras_init"].shape[0]
        self.n_l = prob["points_init"].shape[0]
        self.h = rba_create(prob["cameras_init"] if cams is None else cams,
                            prob["points_init"] if pts is None else pts,
                            prob["obs_cam"], prob["obs_pt"], prob["obs_uv"], self.opt)

    def close(self):
        if getattr(self, "h", None):
            rba_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def linearize(self):
        rba_linearize(self.h)

    def marginalize(self, lam):
        rba_marginalize_qr(self.h, lam)

    def pcg(self):
        return rba_pcg_solve(self.h)

    def backsub(self):
        rba_backsubstitute(self.h)

    def cost(self, at_trial=False):
        return rba_cost(self.h, at_trial)

    def lm_step(self):
        return rba_lm_step(self.h)

    def lm_solve(self, max_iters=50, ftol=1e-6):
        """The paper's LM loop on the device: reports of the iterations run."""
        return rba_lm_solve(self.h, max_iters, ftol)

    def set_lm(self, lam, nu=2.0):
        rba_set_lm(self.h, lam, nu)

    def get_lm(self):
        return rba_get_lm(self.h)

    def set_pcg_limits(self, rel_tol, max_iters):
        rba_set_pcg_limits(self.h, rel_tol, max_iters)

    def info(self):
        return rba_get_info(self.h)

    def checksums(self):
        return rba_checksums(self.h)

    def state(self, out=None):
        return rba_get_state(self.h, self.n_p, self.n_l, out)

    def set_state(self, cams, pts):
        rba_set_state(self.h, cams, pts)

    def reset_lm(self):
        rba_reset_lm(self.h)

    def matvec(self, v):
        """v: torch float32 CUDA tensor (9 n_p) -> H~ v (torch)."""
        import torch
        v = v.contiguous()
        out = torch.empty_like(v)
        cur = torch.cuda.current_stream(v.device)
        self.stream.wait_stream(cur)
        rba_matvec(self.h, v.data_ptr(), out.data_ptr())
        cur.wait_stream(self.stream)
        v.record_stream(self.stream)
        out.record_stream(self.stream)
        return out

    def rhs(self):
        return rba_get_rhs(self.h, self.n_p)

    def precond_sums(self):
        """(n_p, 54): upper triangles of sum_j A_j[:,i]^T A_j[:,i] and b~_i (last PCG solve)."""
        return rba_get_precond(self.h, self.n_p)

    def step(self):
        return rba_get_step(self.h, self.n_p, self.n_l)

    def scaling(self):
        return rba_get_scaling(self.h, self.n_p, self.n_l)

    def block(self, j):
        return rba_export_block(self.h, j)

    def arena_bytes(self):
        return rba_arena_bytes(self.h)

    def launches(self):
        return rba_kernel_launches(self.h)
