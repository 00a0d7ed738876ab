"""FP64 CPU oracle for the sqrt-BA hot path (ctypes wrapper over oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product path
(paper_2103_01843_b200) never imports it, and this package never imports the product path
(the seeded generator paper_2103_01843_b200/synth.py is the one shared module and carries none
of the method's arithmetic).  See oracle/rba_oracle.c for what each function computes and which
paper passage it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rba_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """gcc -O2 -fopenmp; returns the library path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp",
                               "-Wall", "-Wno-unused-result", _SRC, "-o", _LIB, "-lm"])
    return _LIB


_lib = None


class LMReport(C.Structure):
    _fields_ = [("iter", C.c_int64), ("accepted", C.c_int), ("pcg_iters", C.c_int),
                ("pcg_reason", C.c_int), ("cost", C.c_double), ("cost_trial", C.c_double),
                ("cost_after", C.c_double), ("model", C.c_double), ("rho", C.c_double),
                ("lambda_", C.c_double), ("lambda_next", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P, I64, D, I = C.c_void_p, C.c_int64, C.c_double, C.c_int
        sig = {
            "orc_project": (I, [P, P, P, P]),
            "orc_residual_jacobian": (I, [P, P, P, P, P, P]),
            "orc_givens": (None, [D, D, P, P, P]),
            "orc_create": (P, [P, I64, P, I64, P, P, P, I64]),
            "orc_destroy": (None, [P]),
            "orc_block_offset": (I64, [P, I64]),
            "orc_track_length": (I64, [P, I64]),
            "orc_block_doubles": (I64, [P]),
            "orc_cost": (D, [P]),
            "orc_linearize": (I, [P]),
            "orc_scaling": (I, [P]),
            "orc_marginalize": (I, [P]),
            "orc_damp": (I, [P, D]),
            "orc_undamp": (I, [P]),
            "orc_reduced_dense": (I, [P, P, P]),
            "orc_matvec": (None, [P, P, P]),
            "orc_precond_rhs": (I, [P]),
            "orc_pcg": (I, [P, D, I, P, P]),
            "orc_backsub": (I, [P]),
            "orc_model_decrease": (D, [P]),
            "orc_trial_cost": (D, [P]),
            "orc_lm_step": (I, [P, D, I, P]),
            "orc_get_state": (None, [P, P, P]),
            "orc_set_state": (None, [P, P, P]),
            "orc_set_lm": (None, [P, D, D]),
            "orc_set_huber": (None, [P, D]),
            "orc_huber_rho": (D, [D, D]),
            "orc_huber_weight": (D, [D, D]),
            "orc_get_lambda": (D, [P]),
            "orc_linearized_cost": (D, [P]),
            "orc_obs_order": (None, [P, P, P]),
            "orc_get_linearization": (None, [P, P, P, P]),
            "orc_get_scaling": (None, [P, P, P, P, P]),
            "orc_get_block": (None, [P, I64, P]),
            "orc_get_givens": (None, [P, I64, P]),
            "orc_get_rhs": (None, [P, P]),
            "orc_get_precond_factor": (None, [P, P]),
            "orc_block_arena": (None, [P, C.POINTER(C.c_void_p), P]),
            "orc_set_streaming": (None, [P, I]),
            "orc_products": (None, [P, I, P, P]),
            "orc_get_dp": (None, [P, P]),
            "orc_set_dp": (None, [P, P]),
            "orc_get_rho_cg": (None, [P, P]),
            "orc_get_dl": (None, [P, P]),
            "orc_get_trial": (None, [P, P, P]),
            "orc_get_q1r2": (D, [P]),
            "orc_get_damp_l": (D, [P]),
            "orc_get_block_lambda": (D, [P]),
            "orc_num_threads": (I, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def project(cam, X):
    cam = np.ascontiguousarray(cam, np.float64)
    X = np.ascontiguousarray(X, np.float64)
    uv = np.zeros(2)
    pz = np.zeros(1)
    lib().orc_project(_p(cam), _p(X), _p(uv), _p(pz))
    return uv, float(pz[0])


def residual_jacobian(cam, X, u):
    cam, X, u = (np.ascontiguousarray(a, np.float64) for a in (cam, X, u))
    r, Jc, Jl = np.zeros(2), np.zeros((2, 9)), np.zeros((2, 3))
    rc = lib().orc_residual_jacobian(_p(cam), _p(X), _p(u), _p(r), _p(Jc), _p(Jl))
    if rc:
        raise ValueError("degenerate projection")
    return r, Jc, Jl


def huber_rho(s, delta):
    return lib().orc_huber_rho(float(s), float(delta))


def huber_weight(s, delta):
    return lib().orc_huber_weight(float(s), float(delta))


def givens(a, b):
    c, s, rho = C.c_double(), C.c_double(), C.c_double()
    lib().orc_givens(a, b, C.byref(c), C.byref(s), C.byref(rho))
    return c.value, s.value, rho.value


class Oracle:
    """One FP64 sqrt-BA problem.  Landmark index j is the caller's landmark index."""

    def __init__(self, prob: dict, cams=None, pts=None):
        L = lib()
        self.cams0 = np.ascontiguousarray(prob["cameras_init"] if cams is None else cams, np.float64)
        self.pts0 = np.ascontiguousarray(prob["points_init"] if pts is None else pts, np.float64)
        self.obs_cam = np.ascontiguousarray(prob["obs_cam"], np.int32)
        self.obs_pt = np.ascontiguousarray(prob["obs_pt"], np.int32)
        self.obs_uv = np.ascontiguousarray(prob["obs_uv"], np.float64)
        self.n_p, self.n_l, self.n_obs = len(self.cams0), len(self.pts0), len(self.obs_cam)
        self.h = L.orc_create(_p(self.cams0), self.n_p, _p(self.pts0), self.n_l, _p(self.obs_cam),
                              _p(self.obs_pt), _p(self.obs_uv), self.n_obs)
        if not self.h:
            raise MemoryError("oracle: allocation failed")
        src = np.zeros(self.n_obs, np.int64)
        self.lm_ptr = np.zeros(self.n_l + 1, np.int64)
        L.orc_obs_order(self.h, _p(src), _p(self.lm_ptr))
        self.obs_src = src
        self.csr_cam = self.obs_cam[src]

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    # --- steps
    def linearize(self):
        rc = lib().orc_linearize(self.h)
        if rc == 3:
            raise MemoryError("oracle: landmark-block allocation failed")
        if rc:
            raise ValueError("oracle: degenerate projection")

    def linearize_scaling(self):
        """O1-O2 only (residuals, Jacobians, E, scaling, D^2): no landmark blocks are allocated."""
        if lib().orc_scaling(self.h):
            raise ValueError("oracle: degenerate projection")

    def marginalize(self):
        assert lib().orc_marginalize(self.h) == 0

    def damp(self, lam):
        assert lib().orc_damp(self.h, float(lam)) == 0

    def undamp(self):
        assert lib().orc_undamp(self.h) == 0

    def reduced_dense(self):
        N = 9 * self.n_p
        H = np.zeros((N, N))
        b = np.zeros(N)
        assert lib().orc_reduced_dense(self.h, _p(H), _p(b)) == 0
        return H, b

    def matvec(self, v):
        v = np.ascontiguousarray(v, np.float64)
        out = np.zeros_like(v)
        lib().orc_matvec(self.h, _p(v), _p(out))
        return out

    def precond_rhs(self):
        return lib().orc_precond_rhs(self.h)

    def pcg(self, tol=1e-2, max_iters=500):
        reason, relres = C.c_int(), C.c_double()
        it = lib().orc_pcg(self.h, tol, max_iters, C.byref(reason), C.byref(relres))
        return it, reason.value, relres.value

    def backsub(self):
        assert lib().orc_backsub(self.h) == 0

    def model_decrease(self):
        return lib().orc_model_decrease(self.h)

    def trial_cost(self):
        return lib().orc_trial_cost(self.h)

    def cost(self):
        return lib().orc_cost(self.h)

    def lm_step(self, pcg_tol=1e-2, pcg_max_iters=500):
        rep = LMReport()
        if lib().orc_lm_step(self.h, pcg_tol, pcg_max_iters, C.byref(rep)):
            raise ValueError("oracle: degenerate projection")
        return rep.as_dict()

    # --- accessors
    def state(self):
        c, p = np.zeros((self.n_p, 9)), np.zeros((self.n_l, 3))
        lib().orc_get_state(self.h, _p(c), _p(p))
        return c, p

    def set_state(self, cams, pts):
        cams = np.ascontiguousarray(cams, np.float64)
        pts = np.ascontiguousarray(pts, np.float64)
        lib().orc_set_state(self.h, _p(cams), _p(pts))

    def set_lm(self, lam, nu=2.0):
        lib().orc_set_lm(self.h, lam, nu)

    def set_huber(self, delta):
        """Huber robust loss with parameter delta px (IRLS); 0 = squared loss."""
        lib().orc_set_huber(self.h, float(delta))

    def linearization(self):
        """(r, Jc, Jl) unscaled, CSR order (use .obs_src / .lm_ptr / .csr_cam)."""
        r, Jc, Jl = np.zeros((self.n_obs, 2)), np.zeros((self.n_obs, 2, 9)), np.zeros((self.n_obs, 2, 3))
        lib().orc_get_linearization(self.h, _p(r), _p(Jc), _p(Jl))
        return r, Jc, Jl

    def scaling(self):
        sp, Dp2 = np.zeros(9 * self.n_p), np.zeros(9 * self.n_p)
        sl, Dl2 = np.zeros(3 * self.n_l), np.zeros(3 * self.n_l)
        lib().orc_get_scaling(self.h, _p(sp), _p(Dp2), _p(sl), _p(Dl2))
        return sp, Dp2, sl, Dl2

    def track_length(self, j):
        return int(lib().orc_track_length(self.h, j))

    def block(self, j):
        k = self.track_length(j)
        B = np.zeros((2 * k + 3, 9 * k + 4))
        lib().orc_get_block(self.h, j, _p(B))
        return B

    def givens_of(self, j):
        g = np.zeros(12)
        lib().orc_get_givens(self.h, j, _p(g))
        return g.reshape(6, 2)

    def rhs(self):
        b = np.zeros(9 * self.n_p)
        lib().orc_get_rhs(self.h, _p(b))
        return b

    def set_streaming(self, on=True):
        """Streaming mode (no block arena: every block is recomputed, O3-O5, where it is read) for
        problems whose FP64 blocks do not fit in host memory (config 5).  Relinearizes next."""
        lib().orc_set_streaming(self.h, int(bool(on)))

    def products(self, V):
        """H~ v for the rows v of V (nvec x 9 n_p) in one pass over the landmarks."""
        V = np.ascontiguousarray(np.atleast_2d(V), np.float64)
        out = np.zeros_like(V)
        lib().orc_products(self.h, V.shape[0], _p(V), _p(out))
        return out

    def block_arena(self):
        """(arena, offsets): a zero-copy read-only numpy view of every landmark block (landmark j at
        arena[offsets[j]:offsets[j+1]], row-major (2k+3) x (9k+4)); valid until the next
        linearization and while this Oracle lives."""
        ptr = C.c_void_p()
        off = np.zeros(self.n_l + 1, np.int64)
        lib().orc_block_arena(self.h, C.byref(ptr), _p(off))
        if not ptr.value:
            raise RuntimeError("oracle: no landmark blocks (linearize first)")
        arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_double)), shape=(int(off[-1]),))
        arr.flags.writeable = False
        return arr, off

    def precond_blocks(self):
        """The block-Jacobi blocks P_i (n_p x 9 x 9) as L_i L_i^T from the stored Cholesky factors."""
        L = np.zeros((self.n_p, 9, 9))
        lib().orc_get_precond_factor(self.h, _p(L))
        return L @ L.transpose(0, 2, 1)

    def dp(self):
        d = np.zeros(9 * self.n_p)
        lib().orc_get_dp(self.h, _p(d))
        return d

    def set_dp(self, d):
        d = np.ascontiguousarray(d, np.float64)
        lib().orc_set_dp(self.h, _p(d))

    def rho_cg(self):
        d = np.zeros(9 * self.n_p)
        lib().orc_get_rho_cg(self.h, _p(d))
        return d

    def dl(self):
        d = np.zeros(3 * self.n_l)
        lib().orc_get_dl(self.h, _p(d))
        return d

    def trial_state(self):
        c, p = np.zeros((self.n_p, 9)), np.zeros((self.n_l, 3))
        lib().orc_get_trial(self.h, _p(c), _p(p))
        return c, p

    def q1r2(self):
        return lib().orc_get_q1r2(self.h)

    def damp_l(self):
        return lib().orc_get_damp_l(self.h)

    def block_lambda(self):
        return lib().orc_get_block_lambda(self.h)

    def lambda_(self):
        return lib().orc_get_lambda(self.h)


def num_threads() -> int:
    return int(lib().orc_num_threads())
