"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU checkers.

Two interchangeable backends with identical entry points:
  * ``port``      — oracle/liboracle.so, the plain-C restatement (oracle/nufft_oracle.c)
  * ``reference`` — oracle/_ref/libnufft_ref.so, the reference headers compiled
                    unmodified (oracle/ref_capi.cpp), present only when built here
                    from /root/reference (it then travels to the GPU box).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module, and only as the checker / the timed CPU baseline.  The
product library (paper_1701_04492_b200) never touches it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libnufft_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_sp = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_sz = C.c_size_t
_vp = C.c_void_p


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code  # 1 invalid_argument, 2 domain_error, 3 other


def build(quiet: bool = True) -> None:
    """Compile the checkers (make -C oracle).  The reference leg only builds
    when /root/reference is present (this container)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _c2(a) -> np.ndarray:
    """complex128 array -> contiguous float64 view (re, im interleaved)."""
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a.view(np.float64)


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        p = "orc_" if kind == "port" else "ref_"
        self.p = p
        L = self.lib

        def fn(name, res, args):
            f = getattr(L, p + name)
            f.restype = res
            f.argtypes = args
            return f

        self._err = fn("last_error", C.c_char_p, [])
        self._lambert = fn("lambert_w", C.c_int, [C.c_double, C.POINTER(C.c_double)])
        self._bessel = fn("bessel_j_int", C.c_int, [C.c_int, C.c_double, C.POINTER(C.c_double)])
        self._select = fn("select_rank", C.c_int, [C.c_double, C.c_double, C.POINTER(_sz)])
        self._cheb = fn("cheb_coefficients", C.c_int, [C.c_double, _sz, _dp])
        self._chebeval = fn("cheb_eval_matrix", C.c_int, [_dp, _sz, _sz, _dp])
        self._factors = fn("build_factors", C.c_int,
                           [_dp, _sz, C.c_double, _dp, _sz, C.c_double, C.POINTER(_sz), _vp, _vp])
        self._fftf = fn("fft_forward", C.c_int, [_dp, _dp, _sz])
        self._ffti = fn("fft_inverse", C.c_int, [_dp, _dp, _sz])
        self._fft2 = fn("fft_2d_forward", C.c_int, [_dp, _dp, _sz, _sz])
        self._norm = fn("normalize_samples", C.c_int, [_dp, _sz, _dp])
        self._grid = fn("grid_assign", C.c_int, [_dp, _sz, _sz, _lp, _sp, C.POINTER(C.c_double)])
        self._p2c = fn("plan2_create", C.c_int, [_dp, _sz, C.c_double, C.POINTER(_vp)])
        self._p2d = fn("plan2_destroy", None, [_vp])
        self._p2rank = fn("plan2_rank", _sz, [_vp])
        self._p2gamma = fn("plan2_gamma", C.c_double, [_vp])
        self._p2samples = fn("plan2_samples", C.c_int, [_vp, _dp, _lp, _sp])
        self._p2factors = fn("plan2_factors", C.c_int, [_vp, _dp, _dp])
        self._p2e = fn("plan2_exec", C.c_int, [_vp, _dp, _dp, C.c_uint])
        self._p2adj = fn("plan2_adjoint", C.c_int, [_vp, _dp, _dp])
        self._p1c = fn("plan1_create", C.c_int, [_dp, _sz, C.c_double, C.POINTER(_vp)])
        self._p1d = fn("plan1_destroy", None, [_vp])
        self._p1rank = fn("plan1_rank", _sz, [_vp])
        self._p1gamma = fn("plan1_gamma", C.c_double, [_vp])
        self._p1e = fn("plan1_exec", C.c_int, [_vp, _dp, _dp])
        self._p1adj = fn("plan1_adjoint", C.c_int, [_vp, _dp, _dp])
        self._tcol = fn("toeplitz_column", C.c_int, [_dp, _sz, C.POINTER(_vp)])
        self._tnorm = fn("toeplitz_normal", C.c_int, [_vp, C.POINTER(_vp)])
        self._tgram = fn("toeplitz_gram", C.c_int, [_vp, C.POINTER(_vp)])
        self._tdel = fn("toeplitz_destroy", None, [_vp])
        self._tmem = fn("toeplitz_members", C.c_int, [_vp, _dp, _dp])
        self._tmv = fn("toeplitz_matvec", C.c_int, [_vp, _dp, _sz, _dp])
        self._cgmax = fn("default_cg_max_iter", _sz, [_sz])
        cg_args = [_dp, C.c_double, _dp, C.POINTER(_sz), C.POINTER(C.c_double), C.POINTER(C.c_int), _dp,
                   C.POINTER(_sz)]
        self._cgt = fn("cg_toeplitz", C.c_int, [_vp, _dp, _sz, C.c_double, _sz, _dp, C.POINTER(_sz),
                                                C.POINTER(C.c_double), C.POINTER(C.c_int), _dp, C.POINTER(_sz)])
        self._inv2 = fn("inufft2", C.c_int, [_vp, _vp] + cg_args)
        self._inv1 = fn("inufft1", C.c_int, [_vp, _vp] + cg_args)
        self._p3c = fn("plan3_create", C.c_int, [_dp, _dp, _sz, C.c_double, C.POINTER(_vp)])
        self._p3d = fn("plan3_destroy", None, [_vp])
        self._p3info = fn("plan3_info", C.c_int,
                          [_vp, C.POINTER(C.c_int), C.POINTER(_sz), C.POINTER(_sz), C.POINTER(_sz)])
        self._p3e = fn("plan3_exec", C.c_int, [_vp, _dp, _dp])
        self._pdc = fn("plan2d2_create", C.c_int,
                       [_dp, _dp, _sz, _sz, _sz, C.c_double, C.POINTER(_vp)])
        self._pdd = fn("plan2d2_destroy", None, [_vp])
        self._pdinfo = fn("plan2d2_info", C.c_int,
                          [_vp, C.POINTER(_sz), C.POINTER(_sz),
                           C.POINTER(C.c_double), C.POINTER(C.c_double)])
        self._pdflat = fn("plan2d2_flat_index", C.c_int, [_vp, _sp])
        self._pde = fn("plan2d2_exec", C.c_int, [_vp, _dp, _dp])
        self._direct = fn("nudft_direct", C.c_int, [_dp, _dp, _dp, _sz, _dp])
        self._direct2 = fn("nudft2d_direct", C.c_int, [_dp, _dp, _sz, _dp, _sz, _sz, _dp])
        self._worst = fn("worst_grid", C.c_int, [_sz, C.c_double, _dp])
        self._snew = fn("sampler_new", _vp, [C.c_ulonglong])
        self._sfree = fn("sampler_free", None, [_vp])
        self._snormal = fn("sampler_normal", C.c_double, [_vp])
        self._suni = fn("sampler_uniform_vector", None, [_vp, _sz, C.c_double, C.c_double, _dp])
        self._scplx = fn("sampler_complex_vector", None, [_vp, _sz, _dp])

    # ------------------------------------------------------------ helpers
    def _check(self, rc: int) -> None:
        if rc:
            raise OracleError(rc, self._err().decode())

    # ------------------------------------------------------------ lowrank
    def lambert_w(self, x: float) -> float:
        out = C.c_double()
        self._check(self._lambert(x, C.byref(out)))
        return out.value

    def bessel_j_int(self, order: int, z: float) -> float:
        out = C.c_double()
        self._check(self._bessel(order, z, C.byref(out)))
        return out.value

    def select_rank(self, gamma: float, eps: float) -> int:
        k = _sz()
        self._check(self._select(gamma, eps, C.byref(k)))
        return k.value

    def cheb_coefficients(self, gamma: float, K: int) -> np.ndarray:
        a = np.zeros(2 * K * K)
        self._check(self._cheb(gamma, K, a))
        return a.view(np.complex128).reshape(K, K)

    def cheb_eval_matrix(self, pts, K: int) -> np.ndarray:
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        out = np.zeros(len(pts) * K)
        self._check(self._chebeval(pts, len(pts), K, out))
        return out.reshape(len(pts), K)

    def build_factors(self, delta, gamma, omega_scaled, eps):
        delta = np.ascontiguousarray(delta, dtype=np.float64)
        om = np.ascontiguousarray(omega_scaled, dtype=np.float64)
        k = _sz()
        self._check(self._factors(delta, len(delta), gamma, om, len(om), eps, C.byref(k), None, None))
        u = np.zeros((k.value, len(delta)), np.complex128)
        v = np.zeros((k.value, len(om)), np.complex128)
        self._check(self._factors(delta, len(delta), gamma, om, len(om), eps, C.byref(k),
                                  u.ctypes.data, v.ctypes.data))
        return k.value, u, v

    # ------------------------------------------------------------ fft
    def fft_forward(self, v) -> np.ndarray:
        v = np.ascontiguousarray(v, np.complex128)
        out = np.zeros_like(v)
        self._check(self._fftf(_c2(v), out.view(np.float64), len(v)))
        return out

    def fft_inverse(self, v) -> np.ndarray:
        v = np.ascontiguousarray(v, np.complex128)
        out = np.zeros_like(v)
        self._check(self._ffti(_c2(v), out.view(np.float64), len(v)))
        return out

    def fft_2d_forward(self, m) -> np.ndarray:
        m = np.ascontiguousarray(m, np.complex128)
        out = np.zeros_like(m)
        self._check(self._fft2(_c2(m).ravel(), out.view(np.float64).ravel(), m.shape[0], m.shape[1]))
        return out

    def normalize_samples(self, raw) -> np.ndarray:
        raw = np.ascontiguousarray(raw, np.float64)
        out = np.zeros_like(raw)
        self._check(self._norm(raw, len(raw), out))
        return out

    def grid_assign(self, x, grid: int):
        x = np.ascontiguousarray(x, np.float64)
        s = np.zeros(len(x), np.int64)
        t = np.zeros(len(x), np.uint64)
        g = C.c_double()
        self._check(self._grid(x, len(x), grid, s, t, C.byref(g)))
        return s, t, g.value

    # ------------------------------------------------------------ plans
    def plan2(self, x, eps):
        return _Plan(self, "2", np.ascontiguousarray(x, np.float64), eps)

    def plan1(self, omega, eps):
        return _Plan(self, "1", np.ascontiguousarray(omega, np.float64), eps)

    def plan3(self, x, omega, eps):
        return _Plan(self, "3", (np.ascontiguousarray(x, np.float64),
                                 np.ascontiguousarray(omega, np.float64)), eps)

    def plan2d2(self, x, y, m, n, eps):
        return _Plan(self, "2d2", (np.ascontiguousarray(x, np.float64),
                                   np.ascontiguousarray(y, np.float64), m, n), eps)

    # ------------------------------------------------------------ direct sums
    def nudft_direct(self, x, omega, c) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        omega = np.ascontiguousarray(omega, np.float64)
        c = np.ascontiguousarray(c, np.complex128)
        f = np.zeros(len(x), np.complex128)
        self._check(self._direct(x, omega, _c2(c), len(x), f.view(np.float64)))
        return f

    def nudft2d_direct(self, x, y, C2) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        C2 = np.ascontiguousarray(C2, np.complex128)
        f = np.zeros(len(x), np.complex128)
        self._check(self._direct2(x, y, len(x), _c2(C2).ravel(), C2.shape[0], C2.shape[1],
                                  f.view(np.float64)))
        return f

    def worst_grid(self, n: int, gamma: float) -> np.ndarray:
        out = np.zeros(n)
        self._check(self._worst(n, gamma, out))
        return out

    def sampler(self, seed: int) -> "_Sampler":
        return _Sampler(self, seed)

    # ------------------------------------------------------------ inverse.hpp
    def toeplitz_from_first_column(self, col) -> "_Toeplitz":
        col = np.ascontiguousarray(col, np.complex128)
        h = _vp()
        self._check(self._tcol(_c2(col), len(col), C.byref(h)))
        return _Toeplitz(self, h, len(col))

    def toeplitz_from_normal(self, plan) -> "_Toeplitz":
        h = _vp()
        self._check(self._tnorm(plan.h, C.byref(h)))
        return _Toeplitz(self, h, plan.n)

    def toeplitz_from_gram(self, plan) -> "_Toeplitz":
        h = _vp()
        self._check(self._tgram(plan.h, C.byref(h)))
        return _Toeplitz(self, h, plan.n)

    def default_cg_max_iter(self, n: int) -> int:
        return self._cgmax(n)

    def _cg_call(self, f, n, *head):
        sol = np.zeros(n, np.complex128)
        cap = max(self.default_cg_max_iter(n), 1) + 1
        hist = np.zeros(cap)
        it, rr, cv, hl = _sz(), C.c_double(), C.c_int(), _sz()
        self._check(f(*head, sol.view(np.float64), C.byref(it), C.byref(rr), C.byref(cv), hist, C.byref(hl)))
        return {"solution": sol, "iterations": it.value, "relativeResidual": rr.value,
                "converged": bool(cv.value), "residualHistory": hist[:hl.value].copy()}

    def cg_toeplitz(self, op, rhs, tol, max_iter):
        rhs = np.ascontiguousarray(rhs, np.complex128)
        sol = np.zeros(len(rhs), np.complex128)
        hist = np.zeros(max_iter + 1)
        it, rr, cv, hl = _sz(), C.c_double(), C.c_int(), _sz()
        self._check(self._cgt(op.h, _c2(rhs), len(rhs), tol, max_iter, sol.view(np.float64), C.byref(it),
                              C.byref(rr), C.byref(cv), hist, C.byref(hl)))
        return {"solution": sol, "iterations": it.value, "relativeResidual": rr.value,
                "converged": bool(cv.value), "residualHistory": hist[:hl.value].copy()}

    def inufft2(self, plan, f, tol, op=None):
        f = np.ascontiguousarray(f, np.complex128)
        return self._cg_call(self._inv2, plan.n, plan.h, op.h if op else None, _c2(f), tol)

    def inufft1(self, plan, f, tol, op=None):
        f = np.ascontiguousarray(f, np.complex128)
        return self._cg_call(self._inv1, plan.n, plan.h, op.h if op else None, _c2(f), tol)


class _Toeplitz:
    def __init__(self, o: Oracle, h, n: int):
        self.o, self.h, self.n = o, h, n

    def __del__(self):
        try:
            self.o._tdel(self.h)
        except Exception:
            pass

    def _members(self):
        sp = np.zeros(2 * self.n, np.complex128)
        fc = np.zeros(self.n, np.complex128)
        self.o._check(self.o._tmem(self.h, sp.view(np.float64), fc.view(np.float64)))
        return sp, fc

    @property
    def spectrum(self) -> np.ndarray:
        return self._members()[0]

    @property
    def firstColumn(self) -> np.ndarray:  # noqa: N802 (reference member name)
        return self._members()[1]

    def matvec(self, v) -> np.ndarray:
        v = np.ascontiguousarray(v, np.complex128)
        out = np.zeros(len(v), np.complex128)
        self.o._check(self.o._tmv(self.h, _c2(v), len(v), out.view(np.float64)))
        return out


class _Sampler:
    def __init__(self, o: Oracle, seed: int):
        self.o = o
        self.h = o._snew(seed)

    def __del__(self):
        try:
            self.o._sfree(self.h)
        except Exception:
            pass

    def normal(self) -> float:
        return self.o._snormal(self.h)

    def uniform_vector(self, n, lo, hi) -> np.ndarray:
        out = np.zeros(n)
        self.o._suni(self.h, n, lo, hi, out)
        return out

    def complex_vector(self, n) -> np.ndarray:
        out = np.zeros(n, np.complex128)
        self.o._scplx(self.h, n, out.view(np.float64))
        return out


class _Plan:
    def __init__(self, o: Oracle, kind: str, args, eps: float):
        self.o, self.kind = o, kind
        h = _vp()
        if kind == "2":
            self.n = len(args)
            o._check(o._p2c(args, len(args), eps, C.byref(h)))
        elif kind == "1":
            self.n = len(args)
            o._check(o._p1c(args, len(args), eps, C.byref(h)))
        elif kind == "3":
            x, w = args
            if len(x) != len(w):
                raise OracleError(1, "plan_nufft3: sample/frequency length mismatch")
            self.n = len(x)
            o._check(o._p3c(x, w, len(x), eps, C.byref(h)))
        else:
            x, y, m, n = args
            self.n, self.m_, self.n_ = len(x), m, n
            o._check(o._pdc(x, y, len(x), m, n, eps, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            d = {"2": self.o._p2d, "1": self.o._p1d, "3": self.o._p3d, "2d2": self.o._pdd}[self.kind]
            d(self.h)
        except Exception:
            pass

    # type II / I
    @property
    def rank(self) -> int:
        if self.kind == "2":
            return self.o._p2rank(self.h)
        if self.kind == "1":
            return self.o._p1rank(self.h)
        if self.kind == "3":
            return self.info3()[1]
        return self.info2d()[:2]

    @property
    def gamma(self) -> float:
        return self.o._p2gamma(self.h) if self.kind == "2" else self.o._p1gamma(self.h)

    def samples(self):
        x = np.zeros(self.n)
        s = np.zeros(self.n, np.int64)
        t = np.zeros(self.n, np.uint64)
        self.o._check(self.o._p2samples(self.h, x, s, t))
        return x, s, t

    def factors(self):
        K = self.rank
        u = np.zeros((K, self.n), np.complex128)
        v = np.zeros((K, self.n), np.complex128)
        self.o._check(self.o._p2factors(self.h, u.view(np.float64).ravel(), v.view(np.float64).ravel()))
        return u, v

    def info3(self):
        bt, ka, ke, ki = C.c_int(), _sz(), _sz(), _sz()
        self.o._p3info(self.h, C.byref(bt), C.byref(ka), C.byref(ke), C.byref(ki))
        return bool(bt.value), ka.value, ke.value, ki.value

    def info2d(self):
        kx, ky, gx, gy = _sz(), _sz(), C.c_double(), C.c_double()
        self.o._pdinfo(self.h, C.byref(kx), C.byref(ky), C.byref(gx), C.byref(gy))
        return kx.value, ky.value, gx.value, gy.value

    def flat_index(self):
        out = np.zeros(self.n, np.uint64)
        self.o._pdflat(self.h, out)
        return out

    def execute(self, c, threads: int = 1) -> np.ndarray:
        f = np.zeros(self.n, np.complex128)
        if self.kind == "2d2":
            c = np.ascontiguousarray(c, np.complex128)
            if c.shape != (self.m_, self.n_):
                raise OracleError(1, "exec_nufft2d2: coefficient dimensions mismatch")
            self.o._check(self.o._pde(self.h, _c2(c).ravel(), f.view(np.float64)))
            return f
        c = np.ascontiguousarray(c, np.complex128)
        if len(c) != self.n:
            raise OracleError(1, "length mismatch")
        if self.kind == "2":
            self.o._check(self.o._p2e(self.h, _c2(c), f.view(np.float64), threads))
        elif self.kind == "1":
            self.o._check(self.o._p1e(self.h, _c2(c), f.view(np.float64)))
        else:
            self.o._check(self.o._p3e(self.h, _c2(c), f.view(np.float64)))
        return f

    def adjoint(self, f) -> np.ndarray:
        f = np.ascontiguousarray(f, np.complex128)
        out = np.zeros(self.n, np.complex128)
        adj = self.o._p1adj if self.kind == "1" else self.o._p2adj
        self.o._check(adj(self.h, _c2(f), out.view(np.float64)))
        return out


def available(kind: str) -> bool:
    return os.path.exists(PORT_SO if kind == "port" else REF_SO)
