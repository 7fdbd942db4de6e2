"""Python mirror of the reference's C++ entry points (proj/include/nufft/*.hpp),
over the C-ABI of libnufft_b200.so.  Names, argument meaning and error
behaviour follow the reference: std::invalid_argument -> InvalidArgument,
std::domain_error -> DomainError (both ValueError subclasses).

Host-array calls (numpy) copy to and from the GPU; the ``*_device`` methods
take device pointers (e.g. ``torch.Tensor.data_ptr()``) and a CUDA stream
handle, which is the path the throughput metric is measured on.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import CgReport, PlanInfo, lib

__all__ = [
    "InvalidArgument", "DomainError", "NufftError",
    "lambert_w", "bessel_j_int", "bessel_j_signed", "select_rank", "cheb_coefficients",
    "cheb_eval_matrix", "build_factors", "fft_forward", "fft_inverse", "fft_2d_forward",
    "fft_cols_forward", "fft_rows_forward", "fft_exec_count", "fft_reset_exec_counts",
    "normalize_samples", "grid_assign", "Plan2", "Plan1", "Plan3", "Plan2D",
    "plan_nufft2", "exec_nufft2", "exec_nufft2_adjoint", "plan_nufft1", "exec_nufft1",
    "plan_nufft3", "exec_nufft3", "plan_nufft2d2", "exec_nufft2d2", "exec_nufft2d2_impl",
    "device_count", "ToeplitzOperator", "toeplitz_from_first_column", "toeplitz_from_normal",
    "toeplitz_from_gram", "toeplitz_matvec", "cg_solve_toeplitz", "inufft2", "inufft1",
    "default_cg_max_iter", "exec_nufft1_adjoint", "inufft2_device", "nudft_direct", "nudft2d_direct",
    "GaussianSampler",
]


class NufftError(RuntimeError):
    pass


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class DomainError(ValueError):
    """std::domain_error in the reference."""


class CudaError(NufftError):
    pass


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().nufft_last_error().decode()
    if rc == 1:
        raise InvalidArgument(msg)
    if rc == 2:
        raise DomainError(msg)
    if rc == 3:
        raise CudaError(msg)
    raise NufftError(f"status {rc}: {msg}")


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def _ptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


def device_count() -> int:
    n = C.c_int()
    _check(lib().nufft_device_count(C.byref(n)))
    return n.value


# ------------------------------------------------------------------ special
def lambert_w(x: float) -> float:
    out = C.c_double()
    _check(lib().nufft_lambert_w(x, C.byref(out)))
    return out.value


def bessel_j_int(order: int, z: float) -> float:
    out = C.c_double()
    _check(lib().nufft_bessel_j_int(order, z, C.byref(out)))
    return out.value


def bessel_j_signed(order: int, z: float) -> float:
    out = C.c_double()
    _check(lib().nufft_bessel_j_signed(order, z, C.byref(out)))
    return out.value


# ------------------------------------------------------------------ lowrank
def select_rank(gamma: float, epsilon: float) -> int:
    k = C.c_size_t()
    _check(lib().nufft_select_rank(gamma, epsilon, C.byref(k)))
    return k.value


def cheb_coefficients(gamma: float, K: int) -> np.ndarray:
    """K x K complex, a[p, r] (lowrank.hpp:36-65)."""
    a = np.zeros((K, K), np.complex128)
    _check(lib().nufft_cheb_coefficients(gamma, K, a.ctypes.data))
    return a


def cheb_eval_matrix(points, K: int) -> np.ndarray:
    p = _f64(points)
    out = np.zeros((len(p), K))
    _check(lib().nufft_cheb_eval_matrix(_ptr(p), len(p), K, _ptr(out)))
    return out


def build_factors(delta, gamma: float, omega_scaled, epsilon: float):
    """(rank, u[K, n], v[K, m]) — lowrank.hpp:161-210."""
    d, w = _f64(delta), _f64(omega_scaled)
    k = C.c_size_t()
    _check(lib().nufft_build_factors(_ptr(d), len(d), gamma, _ptr(w), len(w), epsilon,
                                     C.byref(k), None, None))
    u = np.zeros((k.value, len(d)), np.complex128)
    v = np.zeros((k.value, len(w)), np.complex128)
    _check(lib().nufft_build_factors(_ptr(d), len(d), gamma, _ptr(w), len(w), epsilon,
                                     C.byref(k), _ptr(u), _ptr(v)))
    return k.value, u, v


# ------------------------------------------------------------------ fft
def fft_forward(v) -> np.ndarray:
    v = _c128(v)
    out = np.empty_like(v)
    _check(lib().nufft_fft_forward_host(_ptr(v), _ptr(out), len(v)))
    return out


def fft_inverse(v) -> np.ndarray:
    v = _c128(v)
    out = np.empty_like(v)
    _check(lib().nufft_fft_inverse_host(_ptr(v), _ptr(out), len(v)))
    return out


def fft_2d_forward(m) -> np.ndarray:
    m = _c128(m)
    if m.ndim != 2:
        raise InvalidArgument("fft_2d_forward: expected a matrix")
    out = np.empty_like(m)
    _check(lib().nufft_fft_2d_forward_host(_ptr(m), _ptr(out), m.shape[0], m.shape[1]))
    return out


def fft_cols_forward(m) -> np.ndarray:
    out = _c128(m).copy()
    _check(lib().nufft_fft_cols_forward_host(_ptr(out), out.shape[0], out.shape[1]))
    return out


def fft_rows_forward(m) -> np.ndarray:
    out = _c128(m).copy()
    _check(lib().nufft_fft_rows_forward_host(_ptr(out), out.shape[0], out.shape[1]))
    return out


def fft_exec_count(n: int) -> int:
    return int(lib().nufft_fft_exec_count(n))


def fft_reset_exec_counts() -> None:
    lib().nufft_fft_reset_exec_counts()


# ------------------------------------------------------------------ samples
def normalize_samples(raw) -> np.ndarray:
    r = _f64(raw)
    out = np.zeros_like(r)
    _check(lib().nufft_normalize_samples(_ptr(r), len(r), _ptr(out)))
    return out


def grid_assign(x, grid: int):
    """(s, t, gamma) — transforms.hpp:77-92."""
    x = _f64(x)
    s = np.zeros(len(x), np.int64)
    t = np.zeros(len(x), np.uint64)
    g = C.c_double()
    _check(lib().nufft_grid_assign(_ptr(x), len(x), grid, _ptr(s), _ptr(t), C.byref(g)))
    return s, t, g.value


# ------------------------------------------------------------------ plans
class _PlanBase:
    _kind = ""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        self._info = PlanInfo()
        _check(getattr(lib(), f"nufft_{self._kind}_info")(self._h, C.byref(self._info)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                getattr(lib(), f"nufft_{self._kind}_destroy")(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def info(self) -> PlanInfo:
        return self._info

    def size(self) -> int:
        return self._info.n

    @property
    def device(self) -> int:
        return self._info.device

    @property
    def fused(self) -> bool:
        return self._info.path == 1


class Plan2(_PlanBase):
    """Type-II plan (transforms.hpp:105-114)."""
    _kind = "plan2"

    def rank(self) -> int:
        return self._info.rank

    def gamma(self) -> float:
        return self._info.gamma

    def samples(self):
        n = self.size()
        x, s, t = np.zeros(n), np.zeros(n, np.int64), np.zeros(n, np.uint64)
        _check(lib().nufft_plan2_samples(self._h, _ptr(x), _ptr(s), _ptr(t)))
        return x, s, t

    def factors(self):
        K, n = self.rank(), self.size()
        u, v = np.zeros((K, n), np.complex128), np.zeros((K, n), np.complex128)
        _check(lib().nufft_plan2_factors(self._h, _ptr(u), _ptr(v)))
        return u, v

    def execute(self, c, threads: int = 1) -> np.ndarray:
        c = _c128(c)
        batch = 1 if c.ndim == 1 else c.shape[0]
        length = c.shape[-1]
        f = np.empty_like(c)
        _check(lib().nufft_plan2_exec_host(self._h, _ptr(c), length, _ptr(f), batch))
        return f

    def execute_device(self, c_ptr: int, f_ptr: int, batch: int = 1, stream: int = 0) -> None:
        _check(lib().nufft_plan2_exec(self._h, c_ptr, f_ptr, batch, stream or None))

    def execute_terms_device(self, c_ptr: int, f_ptr: int, r_begin: int, r_end: int,
                             batch: int = 1, stream: int = 0) -> None:
        _check(lib().nufft_plan2_exec_terms(self._h, c_ptr, f_ptr, batch, r_begin, r_end,
                                            stream or None))

    def execute_timed_device(self, c_ptr: int, f_ptr: int, stream: int, slot: int) -> None:
        """exec with per-pass CUDA events recorded in timing slot `slot` (no sync)."""
        _check(lib().nufft_plan2_exec_timed(self._h, c_ptr, f_ptr, stream or None, slot))

    def timing_read(self, nslots: int):
        """(ms_pass1_total, ms_pass2_total) over slots [0, nslots)."""
        a, b = C.c_double(), C.c_double()
        _check(lib().nufft_plan2_timing_read(self._h, nslots, C.byref(a), C.byref(b)))
        return a.value, b.value

    def execute_host_ptr(self, c_ptr: int, f_ptr: int, batch: int = 1) -> None:
        """exec through the host-pointer C-ABI call (copies inside)."""
        _check(lib().nufft_plan2_exec_host(self._h, c_ptr, self.size(), f_ptr, batch))

    # ---- multi-GPU (nufft_plan2_exec_multi and its pieces; parallel.py)
    def execute_multi_device(self, c_ptr: int, f_ptr: int, comm, batch: int = 1, stream: int = 0,
                             root: int = 0, allreduce: bool = False) -> None:
        """Rank-split exec over an NCCL communicator (parallel.NcclComm): this rank's
        terms, chunked reduce, f complete on `root` (or on every rank)."""
        _check(lib().nufft_plan2_exec_multi(self._h, c_ptr, f_ptr, batch, comm.handle, root,
                                            1 if allreduce else 0, stream or None))

    def execute_terms_sorted_device(self, c_ptr: int, fs_ptr: int, r_begin: int, r_end: int,
                                    stream: int = 0) -> None:
        """Partial sum over terms [r_begin, r_end) in bucket (plan) order."""
        _check(lib().nufft_plan2_exec_terms_sorted(self._h, c_ptr, fs_ptr, r_begin, r_end, stream or None))

    def reduce_chunks(self, nchunks: int) -> np.ndarray:
        """Bucket-order offsets [0 .. N] of the row chunks exec_multi reduces one at a time."""
        off = np.zeros(nchunks + 1, np.uint64)
        _check(lib().nufft_plan2_reduce_chunks(self._h, nchunks, _ptr(off)))
        return off.astype(np.int64)

    def unpermute_device(self, fs_ptr: int, f_ptr: int, batch: int = 1, stream: int = 0) -> None:
        """f[perm[i]] = fs[i] (bucket order -> sample order)."""
        _check(lib().nufft_plan2_unpermute(self._h, fs_ptr, f_ptr, batch, stream or None))

    def adjoint(self, f) -> np.ndarray:
        f = _c128(f)
        out = np.empty_like(f)
        _check(lib().nufft_plan2_adjoint_host(self._h, _ptr(f), len(f), _ptr(out)))
        return out


class Plan1(_PlanBase):
    """Type-I plan (transforms.hpp:237-244)."""
    _kind = "plan1"

    def __init__(self, handle, freqs):
        super().__init__(handle)
        self.freqs = freqs

    def rank(self) -> int:
        return self._info.rank

    def gamma(self) -> float:
        return self._info.gamma

    def execute(self, c) -> np.ndarray:
        c = _c128(c)
        batch = 1 if c.ndim == 1 else c.shape[0]
        f = np.empty_like(c)
        _check(lib().nufft_plan1_exec_host(self._h, _ptr(c), c.shape[-1], _ptr(f), batch))
        return f

    def execute_device(self, c_ptr: int, f_ptr: int, batch: int = 1, stream: int = 0) -> None:
        _check(lib().nufft_plan1_exec(self._h, c_ptr, f_ptr, batch, stream or None))

    def execute_terms_device(self, c_ptr: int, f_ptr: int, r_begin: int, r_end: int,
                             batch: int = 1, stream: int = 0) -> None:
        """Partial sum over the terms [r_begin, r_end) (one rank's share)."""
        _check(lib().nufft_plan1_exec_terms(self._h, c_ptr, f_ptr, batch, r_begin, r_end, stream or None))

    def execute_multi_device(self, c_ptr: int, f_ptr: int, comm, batch: int = 1, stream: int = 0,
                             root: int = 0, allreduce: bool = False) -> None:
        """r-split over an NCCL communicator (parallel.NcclComm); f complete on `root`."""
        _check(lib().nufft_plan1_exec_multi(self._h, c_ptr, f_ptr, batch, comm.handle, root,
                                            1 if allreduce else 0, stream or None))


class Plan3(_PlanBase):
    """Type-III plan (transforms.hpp:308-319)."""
    _kind = "plan3"

    @property
    def bTrivial(self) -> bool:  # noqa: N802 (reference member name)
        return bool(self._info.btrivial)

    def effective_rank(self) -> int:
        return self._info.effective_rank

    @property
    def rank_a(self) -> int:
        return self._info.rank

    @property
    def rank_inner(self) -> int:
        return self._info.rank2

    def execute(self, c) -> np.ndarray:
        c = _c128(c)
        batch = 1 if c.ndim == 1 else c.shape[0]
        f = np.empty_like(c)
        _check(lib().nufft_plan3_exec_host(self._h, _ptr(c), c.shape[-1], _ptr(f), batch))
        return f

    def execute_device(self, c_ptr: int, f_ptr: int, batch: int = 1, stream: int = 0) -> None:
        _check(lib().nufft_plan3_exec(self._h, c_ptr, f_ptr, batch, stream or None))

    def execute_terms_device(self, c_ptr: int, f_ptr: int, r_begin: int, r_end: int,
                             batch: int = 1, stream: int = 0) -> None:
        """Partial sum over the outer terms [r_begin, r_end) (one rank's share)."""
        _check(lib().nufft_plan3_exec_terms(self._h, c_ptr, f_ptr, batch, r_begin, r_end, stream or None))

    def execute_multi_device(self, c_ptr: int, f_ptr: int, comm, batch: int = 1, stream: int = 0,
                             root: int = 0, allreduce: bool = False) -> None:
        """Outer-term split over an NCCL communicator (parallel.NcclComm)."""
        _check(lib().nufft_plan3_exec_multi(self._h, c_ptr, f_ptr, batch, comm.handle, root,
                                            1 if allreduce else 0, stream or None))


class Plan2D(_PlanBase):
    """2D type-II plan (transform2d.hpp:51-59)."""
    _kind = "plan2d2"

    @property
    def m(self) -> int:
        return self._info.m

    @property
    def n(self) -> int:
        return self._info.ncols

    def rank_x(self) -> int:
        return self._info.rank

    def rank_y(self) -> int:
        return self._info.rank2

    def grid(self):
        c = self.size()
        arrs = [np.zeros(c), np.zeros(c), np.zeros(c, np.int64), np.zeros(c, np.int64),
                np.zeros(c, np.uint64), np.zeros(c, np.uint64), np.zeros(c, np.uint64)]
        _check(lib().nufft_plan2d2_samples(self._h, *[_ptr(a) for a in arrs]))
        keys = ["x", "y", "sx", "sy", "tx", "ty", "flatIndex"]
        out = dict(zip(keys, arrs))
        out["gammaX"], out["gammaY"] = self._info.gamma, self._info.gamma2
        return out

    def execute(self, C2, reuse_row_stage: bool = True) -> np.ndarray:
        C2 = _c128(C2)
        if C2.ndim != 2:
            raise InvalidArgument("exec_nufft2d2: coefficient dimensions mismatch")
        f = np.empty(self.size(), np.complex128)
        _check(lib().nufft_plan2d2_exec_host_impl(self._h, _ptr(C2), C2.shape[0], C2.shape[1],
                                                  _ptr(f), 1, 1 if reuse_row_stage else 0))
        return f

    def execute_device(self, C_ptr: int, f_ptr: int, batch: int = 1, stream: int = 0) -> None:
        _check(lib().nufft_plan2d2_exec(self._h, C_ptr, f_ptr, batch, stream or None))

    def execute_terms_device(self, C_ptr: int, f_ptr: int, r1_begin: int, r1_end: int,
                             batch: int = 1, stream: int = 0) -> None:
        """Partial sum over the row-stage terms [r1_begin, r1_end) (one rank's share)."""
        _check(lib().nufft_plan2d2_exec_terms(self._h, C_ptr, f_ptr, batch, r1_begin, r1_end, stream or None))

    def execute_multi_device(self, C_ptr: int, f_ptr: int, comm, batch: int = 1, stream: int = 0,
                             root: int = 0, allreduce: bool = False) -> None:
        """r1 split over an NCCL communicator (parallel.NcclComm)."""
        _check(lib().nufft_plan2d2_exec_multi(self._h, C_ptr, f_ptr, batch, comm.handle, root,
                                              1 if allreduce else 0, stream or None))


class GaussianSampler:
    """The reference's seeded sampler (random.hpp:14-60; drop-in include/nufft/random.hpp):
    mt19937_64, 53-bit uniforms, Box-Muller normals in pairs.  Host-only."""

    def __init__(self, seed: int):
        h = C.c_void_p()
        _check(lib().nufft_sampler_create(seed, C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            lib().nufft_sampler_destroy(self._h)
        except Exception:
            pass

    def __call__(self) -> float:
        return lib().nufft_sampler_normal(self._h)

    def uniform(self) -> float:
        return lib().nufft_sampler_uniform(self._h)

    def uniform_vector(self, n: int, lo: float, hi: float) -> np.ndarray:
        out = np.empty(n)
        _check(lib().nufft_sampler_uniform_vector(self._h, n, lo, hi, _ptr(out)))
        return out

    def complex_vector(self, n: int) -> np.ndarray:
        out = np.empty(n, np.complex128)
        _check(lib().nufft_sampler_complex_vector(self._h, n, _ptr(out)))
        return out


def plan_nufft2(x_raw, epsilon: float, device: int = -1) -> Plan2:
    x = _f64(x_raw)
    h = C.c_void_p()
    _check(lib().nufft_plan2_create(_ptr(x), len(x), epsilon, device, C.byref(h)))
    return Plan2(h)


def plan_nufft2_device(x_ptr: int, n: int, epsilon: float, device: int = -1) -> Plan2:
    h = C.c_void_p()
    _check(lib().nufft_plan2_create_device(x_ptr, n, epsilon, device, C.byref(h)))
    return Plan2(h)


def exec_nufft2(plan: Plan2, c, threads: int = 1) -> np.ndarray:
    return plan.execute(c, threads)


def exec_nufft2_adjoint(plan: Plan2, f) -> np.ndarray:
    return plan.adjoint(f)


def plan_nufft1(omega, epsilon: float, device: int = -1) -> Plan1:
    w = _f64(omega)
    h = C.c_void_p()
    _check(lib().nufft_plan1_create(_ptr(w), len(w), epsilon, device, C.byref(h)))
    return Plan1(h, w.copy())


def exec_nufft1(plan: Plan1, c) -> np.ndarray:
    return plan.execute(c)


def plan_nufft3(x_raw, omega, epsilon: float, device: int = -1) -> Plan3:
    x, w = _f64(x_raw), _f64(omega)
    h = C.c_void_p()
    _check(lib().nufft_plan3_create(_ptr(x), _ptr(w), len(x), len(w), epsilon, device, C.byref(h)))
    return Plan3(h)


def exec_nufft3(plan: Plan3, c) -> np.ndarray:
    return plan.execute(c)


def plan_nufft2d2(x_raw, y_raw, m: int, n: int, epsilon: float, device: int = -1) -> Plan2D:
    x, y = _f64(x_raw), _f64(y_raw)
    h = C.c_void_p()
    _check(lib().nufft_plan2d2_create(_ptr(x), _ptr(y), len(x), len(y), m, n, epsilon, device,
                                      C.byref(h)))
    return Plan2D(h)


def exec_nufft2d2(plan: Plan2D, C2) -> np.ndarray:
    return plan.execute(C2, True)


def exec_nufft2d2_impl(plan: Plan2D, C2, reuse_row_stage: bool) -> np.ndarray:
    return plan.execute(C2, reuse_row_stage)


# ---------------------------------------------------------------- inverse (inverse.hpp)
def exec_nufft1_adjoint(plan: Plan1, g) -> np.ndarray:
    """F1~* g (transforms.hpp:294-300)."""
    g = _c128(g)
    out = np.empty_like(g)
    _check(lib().nufft_plan1_adjoint_host(plan._h, _ptr(g), len(g), _ptr(out)))
    return out


class ToeplitzOperator:
    """Hermitian Toeplitz operator in its 2N circulant embedding (inverse.hpp:22-27),
    resident on the device; ``spectrum`` / ``firstColumn`` are host copies."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        n = C.c_size_t()
        _check(lib().nufft_toeplitz_size(self._h, C.byref(n)))
        self.n = n.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().nufft_toeplitz_destroy(h)
            except Exception:
                pass
            self._h = None

    def _members(self):
        sp = np.zeros(2 * self.n, np.complex128)
        fc = np.zeros(self.n, np.complex128)
        _check(lib().nufft_toeplitz_members(self._h, _ptr(sp), _ptr(fc)))
        return sp, fc

    @property
    def spectrum(self) -> np.ndarray:
        return self._members()[0]

    @property
    def firstColumn(self) -> np.ndarray:  # noqa: N802 (reference member name)
        return self._members()[1]

    def matvec_device(self, v_ptr: int, out_ptr: int, stream: int = 0) -> None:
        _check(lib().nufft_toeplitz_matvec(self._h, v_ptr, out_ptr, stream or None))


def toeplitz_from_first_column(column, device: int = -1) -> ToeplitzOperator:
    col = _c128(column)
    h = C.c_void_p()
    _check(lib().nufft_toeplitz_from_first_column(_ptr(col), len(col), device, C.byref(h)))
    return ToeplitzOperator(h)


def toeplitz_from_normal(plan: Plan2) -> ToeplitzOperator:
    h = C.c_void_p()
    _check(lib().nufft_toeplitz_from_normal(plan._h, C.byref(h)))
    return ToeplitzOperator(h)


def toeplitz_from_gram(plan: Plan1) -> ToeplitzOperator:
    h = C.c_void_p()
    _check(lib().nufft_toeplitz_from_gram(plan._h, C.byref(h)))
    return ToeplitzOperator(h)


def toeplitz_matvec(op: ToeplitzOperator, v) -> np.ndarray:
    v = _c128(v)
    out = np.empty_like(v)
    _check(lib().nufft_toeplitz_matvec_host(op._h, _ptr(v), len(v), _ptr(out)))
    return out


def default_cg_max_iter(n: int) -> int:
    return int(lib().nufft_default_cg_max_iter(n))


def _report(rep: CgReport, sol: np.ndarray, hist: np.ndarray) -> dict:
    return {"solution": sol, "iterations": rep.iterations, "relativeResidual": rep.relative_residual,
            "converged": bool(rep.converged), "residualHistory": hist[:rep.history_len].copy()}


def cg_solve_toeplitz(op: ToeplitzOperator, rhs, tol: float, max_iter: int) -> dict:
    """cg_solve (inverse.hpp:118-157) with the Toeplitz operator, on the device."""
    rhs = _c128(rhs)
    sol = np.empty_like(rhs)
    hist = np.zeros(max(max_iter, 1))
    rep = CgReport()
    _check(lib().nufft_cg_toeplitz_host(op._h, _ptr(rhs), len(rhs), tol, max_iter, _ptr(sol), C.byref(rep),
                                        _ptr(hist), len(hist)))
    return _report(rep, sol, hist)


def inufft2(plan: Plan2, f, tol: float, op: ToeplitzOperator | None = None) -> dict:
    """Inverse type II (inverse.hpp:171-183): CG on the normal equations, on the device."""
    f = _c128(f)
    sol = np.empty_like(f)
    hist = np.zeros(default_cg_max_iter(len(f)))
    rep = CgReport()
    _check(lib().nufft_inufft2_host(plan._h, op._h if op else None, _ptr(f), len(f), tol, _ptr(sol),
                                    C.byref(rep), _ptr(hist), len(hist)))
    return _report(rep, sol, hist)


def inufft2_device(plan: Plan2, f_ptr: int, tol: float, sol_ptr: int, op: ToeplitzOperator | None = None,
                   stream: int = 0) -> dict:
    """Device-pointer inufft2 (nufft_inufft2): f and the solution stay in HBM."""
    rep = CgReport()
    _check(lib().nufft_inufft2(plan._h, op._h if op else None, f_ptr, tol, sol_ptr, C.byref(rep),
                               stream or None))
    return {"iterations": rep.iterations, "relativeResidual": rep.relative_residual,
            "converged": bool(rep.converged)}


def inufft1(plan: Plan1, f, tol: float, op: ToeplitzOperator | None = None) -> dict:
    """Inverse type I (inverse.hpp:187-200): CG on the Gram matrix, then c = F1~* y."""
    f = _c128(f)
    sol = np.empty_like(f)
    hist = np.zeros(default_cg_max_iter(len(f)))
    rep = CgReport()
    _check(lib().nufft_inufft1_host(plan._h, op._h if op else None, _ptr(f), len(f), tol, _ptr(sol),
                                    C.byref(rep), _ptr(hist), len(hist)))
    return _report(rep, sol, hist)


# ---------------------------------------------------------------- direct sums (oracle.hpp:70-107)
def nudft_direct(x, omega, c, device: int = -1) -> np.ndarray:
    """f_j = sum_k c_k exp(-2 pi i x_j w_k) on the GPU (exact phase split, Neumaier sums).
    Unlike the reference, len(x) may differ from len(omega) == len(c) (output subsets)."""
    x, w, c = _f64(x), _f64(omega), _c128(c)
    if len(w) != len(c):
        raise InvalidArgument("nudft_direct: length mismatch")
    f = np.empty(len(x), np.complex128)
    _check(lib().nufft_nudft_direct_host(_ptr(x), len(x), _ptr(w), _ptr(c), len(c), _ptr(f), device))
    return f


def nudft2d_direct(x, y, C2, device: int = -1) -> np.ndarray:
    x, y, C2 = _f64(x), _f64(y), _c128(C2)
    if len(x) != len(y):
        raise InvalidArgument("nudft2d_direct: sample length mismatch")
    f = np.empty(len(x), np.complex128)
    _check(lib().nufft_nudft2d_direct_host(_ptr(x), _ptr(y), len(x), _ptr(C2), C2.shape[0], C2.shape[1],
                                           _ptr(f), device))
    return f
