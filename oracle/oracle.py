"""ctypes bindings of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Imported by tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) as the checker; never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libppa_oracle.so")
_L = None
vp = C.c_void_p
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class _SolveOut(C.Structure):
    _fields_ = [("cap_nev", C.c_int), ("cap_roots", C.c_int), ("cap_cycles", C.c_int),
                ("eig_re", _dp), ("eig_im", _dp), ("residuals", _dp), ("conv", _ip),
                ("poly_re", _dp), ("poly_im", _dp), ("inner_re", _dp), ("inner_im", _dp),
                ("cycle_max", _dp),
                ("n_eig", C.c_int), ("n_poly", C.c_int), ("n_inner", C.c_int), ("n_cycles", C.c_int),
                ("converged", C.c_int), ("cycles", C.c_int), ("composite", C.c_int),
                ("discarded", C.c_int),
                ("rtol", C.c_double), ("max_err", C.c_double), ("norm_est", C.c_double),
                ("mvps", C.c_longlong), ("dots", C.c_longlong), ("vops", C.c_longlong),
                ("wall", C.c_double)]


def lib():
    global _L
    if _L is None:
        if not os.path.exists(LIB_PATH):
            from .build_oracle import build  # type: ignore

            build()
        L = C.CDLL(LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_set_threads.restype = None
        L.orc_set_variant.argtypes = [C.c_int]
        L.orc_set_variant.restype = None
        L.orc_max_threads.restype = C.c_int
        sig = {
            "orc_gen_config": [C.c_int, C.POINTER(vp)],
            "orc_gen_convdiff_ref": [C.c_int, C.POINTER(vp)],
            "orc_gen_convdiff_const": [C.c_int, C.c_double, C.POINTER(vp)],
            "orc_gen_laplace3d": [C.c_int, C.POINTER(vp)],
            "orc_gen_bidiag": [C.c_int, C.POINTER(vp)],
            "orc_gen_random_poisson": [C.c_int, C.c_double, C.c_ulonglong, C.POINTER(vp)],
            "orc_csr_create": [C.c_int, C.c_longlong, vp, vp, vp, C.POINTER(vp)],
            "orc_csr_from_triplets": [C.c_int, C.c_longlong, vp, vp, vp, C.POINTER(vp)],
            "orc_csr_info": [vp, _ip, C.POINTER(C.c_longlong), C.POINTER(C.c_ulonglong)],
            "orc_csr_arrays": [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)],
            "orc_normal_vector": [C.c_longlong, C.c_ulonglong, C.c_ulonglong, vp],
            "orc_csr_operator": [vp, C.POINTER(vp)],
            "orc_diag_operator": [C.c_int, vp, C.POINTER(vp)],
            "orc_poly_operator": [vp, vp, vp, C.c_int, C.c_int, C.POINTER(vp)],
            "orc_op_apply": [vp, vp, vp, vp],
            "orc_spmv": [vp, vp, vp],
            "orc_apply_poly": [vp, vp, C.c_int, vp, vp, vp, vp],
            "orc_build_gmres_poly": [vp, vp, C.c_int, vp, vp, _ip, _ip, vp],
            "orc_leja_order": [vp, vp, C.c_int, vp, vp],
            "orc_compute_pof": [vp, vp, C.c_int, vp, vp, _ip, _dp, _ip],
            "orc_add_stability_roots": [vp, vp, C.c_int, C.c_int, C.c_int, vp, vp, _ip],
            "orc_eval_poly": [vp, vp, C.c_int, C.c_double, C.c_double, _dp, _dp],
            "orc_arnoldi": [vp, vp, C.c_int, C.c_int, vp, _ip, _ip, vp, vp],
            "orc_harmonic_from_H": [vp, C.c_int, C.c_int, vp, vp],
            "orc_ritz_from_H": [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp],
            "orc_solve": [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                          C.c_int, C.c_int, C.c_int, C.c_int, C.c_ulonglong, C.c_int,
                          C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_double,
                          C.c_int, C.POINTER(_SolveOut)],
            "orc_block2_operator": [vp, C.POINTER(vp)],
            "orc_shifted_operator": [vp, C.c_double, C.POINTER(vp)],
            "orc_build_two_vector_poly": [vp, vp, vp, C.c_int, vp, vp, _ip, vp],
            "orc_damped_start": [vp, vp, C.c_double, C.c_int, vp, vp],
            "orc_check_ideal_order": [vp, vp, C.c_int, C.c_int, _ip],
            "orc_read_matrix_market": [C.c_char_p, C.POINTER(vp)],
        }
        for k, a in sig.items():
            getattr(L, k).argtypes = a
            getattr(L, k).restype = C.c_int
        L.orc_csr_free.argtypes = [vp]
        L.orc_csr_free.restype = None
        L.orc_op_free.argtypes = [vp]
        L.orc_op_free.restype = None
        L.orc_time_poly_factors.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.c_int]
        L.orc_time_poly_factors.restype = C.c_double
        L.orc_time_mgs2_step.argtypes = [C.c_long, C.c_int, C.c_int]
        L.orc_time_mgs2_step.restype = C.c_double
        _L = L
    return _L


class OracleError(RuntimeError):
    pass


class OracleLogicError(RuntimeError):
    pass


def _ck(s):
    if s == 0:
        return
    m = lib().orc_last_error().decode()
    if s == 1:
        raise ValueError(m)
    if s == 3:
        raise OracleLogicError(m)
    raise OracleError(m)


def _p(a):
    return a.ctypes.data_as(vp)


def _ri(roots):
    r = np.asarray(roots, dtype=np.complex128).ravel()
    return np.ascontiguousarray(r.real), np.ascontiguousarray(r.imag)


def set_threads(t: int) -> None:
    lib().orc_set_threads(int(t))


def set_variant(v: int) -> None:
    """Roundoff-floor probes (not the reference): 0 = reference MGS2 with
    sequential dots (default), 1 = classical CGS2 + blocked dots, 2 = MGS2 +
    blocked dots (ppa_oracle.cpp g_variant)."""
    lib().orc_set_variant(int(v))


def get_variant() -> int:
    return int(lib().orc_get_variant())


def max_threads() -> int:
    return int(lib().orc_max_threads())


class Csr:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _L is not None:
            _L.orc_csr_free(self.h)
            self.h = None

    @classmethod
    def _g(cls, fn, *a):
        h = vp()
        _ck(fn(*a, C.byref(h)))
        return cls(h)

    @classmethod
    def config(cls, k):
        return cls._g(lib().orc_gen_config, k)

    @classmethod
    def convection_diffusion(cls, N):
        return cls._g(lib().orc_gen_convdiff_ref, N)

    @classmethod
    def convection_diffusion_const(cls, N, pe=0.5):
        return cls._g(lib().orc_gen_convdiff_const, N, C.c_double(pe))

    @classmethod
    def laplacian_3d(cls, N):
        return cls._g(lib().orc_gen_laplace3d, N)

    @classmethod
    def bidiagonal(cls, n):
        return cls._g(lib().orc_gen_bidiag, n)

    @classmethod
    def random_poisson(cls, n, lam=16.0, seed=4):
        return cls._g(lib().orc_gen_random_poisson, n, C.c_double(lam), C.c_ulonglong(seed))

    @classmethod
    def from_arrays(cls, n, rp, ci, v):
        rp = np.ascontiguousarray(rp, dtype=np.int32)
        ci = np.ascontiguousarray(ci, dtype=np.int32)
        v = np.ascontiguousarray(v, dtype=np.float64)
        return cls._g(lib().orc_csr_create, n, len(v), _p(rp), _p(ci), _p(v))

    @classmethod
    def from_triplets(cls, n, r, c, v):
        r = np.ascontiguousarray(r, dtype=np.int32)
        c = np.ascontiguousarray(c, dtype=np.int32)
        v = np.ascontiguousarray(v, dtype=np.float64)
        return cls._g(lib().orc_csr_from_triplets, n, len(v), _p(r), _p(c), _p(v))

    def info(self):
        n, nnz, fp = C.c_int(), C.c_longlong(), C.c_ulonglong()
        _ck(lib().orc_csr_info(self.h, C.byref(n), C.byref(nnz), C.byref(fp)))
        return n.value, nnz.value, fp.value

    def arrays(self):
        n, nnz, _ = self.info()
        a, b, c = vp(), vp(), vp()
        _ck(lib().orc_csr_arrays(self.h, C.byref(a), C.byref(b), C.byref(c)))
        rp = np.ctypeslib.as_array(C.cast(a, C.POINTER(C.c_int)), (n + 1,)).copy()
        ci = np.ctypeslib.as_array(C.cast(b, C.POINTER(C.c_int)), (max(nnz, 1),))[:nnz].copy()
        v = np.ctypeslib.as_array(C.cast(c, C.POINTER(C.c_double)), (max(nnz, 1),))[:nnz].copy()
        return rp, ci, v


class Op:
    def __init__(self, h, keep=()):
        self.h = h
        self.keep = keep

    def __del__(self):
        if getattr(self, "h", None) and _L is not None:
            _L.orc_op_free(self.h)
            self.h = None

    def apply(self, x, cost=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        c = np.zeros(3) if cost is None else cost
        _ck(lib().orc_op_apply(self.h, _p(x), _p(y), _p(c)))
        return y


def csr_operator(m: Csr) -> Op:
    h = vp()
    _ck(lib().orc_csr_operator(m.h, C.byref(h)))
    return Op(h, (m,))


def diagonal_operator(d) -> Op:
    d = np.ascontiguousarray(d, dtype=np.float64)
    h = vp()
    _ck(lib().orc_diag_operator(len(d), _p(d), C.byref(h)))
    return Op(h)


def poly_operator(a: Op, roots, complement=False) -> Op:
    re, im = _ri(roots)
    h = vp()
    _ck(lib().orc_poly_operator(a.h, _p(re), _p(im), len(re), int(complement), C.byref(h)))
    return Op(h, (a,))


def normal_vector(n, seed, stream):
    out = np.empty(n)
    _ck(lib().orc_normal_vector(n, seed, stream, _p(out)))
    return out


def apply_poly(roots, a: Op, v, cost=None):
    re, im = _ri(roots)
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.empty_like(v)
    c = np.zeros(3) if cost is None else cost
    _ck(lib().orc_apply_poly(_p(re), _p(im), len(re), a.h, _p(v), _p(out), _p(c)))
    return out


def build_gmres_poly(a: Op, b, degree, cost=None):
    b = np.ascontiguousarray(b, dtype=np.float64)
    re, im = np.zeros(max(degree, 1)), np.zeros(max(degree, 1))
    nr, tr = C.c_int(), C.c_int()
    c = np.zeros(3) if cost is None else cost
    _ck(lib().orc_build_gmres_poly(a.h, _p(b), degree, _p(re), _p(im), C.byref(nr), C.byref(tr), _p(c)))
    return re[:nr.value] + 1j * im[:nr.value], bool(tr.value)


def leja_order(roots):
    re, im = _ri(roots)
    a, b = np.zeros_like(re), np.zeros_like(im)
    _ck(lib().orc_leja_order(_p(re), _p(im), len(re), _p(a), _p(b)))
    return a + 1j * b


def compute_pof(roots):
    re, im = _ri(roots)
    n = len(re)
    lg, cp = np.zeros(max(n, 1)), np.zeros(max(n, 1), dtype=np.int32)
    nd, tot, mx = C.c_int(), C.c_int(), C.c_double()
    _ck(lib().orc_compute_pof(_p(re), _p(im), n, _p(lg), _p(cp), C.byref(nd), C.byref(mx), C.byref(tot)))
    return {"log10_pof": lg[:nd.value], "copies_needed": cp[:nd.value], "max_log10_pof": mx.value,
            "total_copies": tot.value}


def add_stability_roots(roots, max_copies=1 << 20):
    re, im = _ri(roots)
    cap = 8 * len(re) + 64
    a, b, on = np.zeros(cap), np.zeros(cap), C.c_int()
    _ck(lib().orc_add_stability_roots(_p(re), _p(im), len(re), max_copies, cap, _p(a), _p(b), C.byref(on)))
    return a[:on.value] + 1j * b[:on.value]


def eval_poly(roots, z):
    re, im = _ri(roots)
    a, b = C.c_double(), C.c_double()
    _ck(lib().orc_eval_poly(_p(re), _p(im), len(re), C.c_double(complex(z).real),
                            C.c_double(complex(z).imag), C.byref(a), C.byref(b)))
    return complex(a.value, b.value)


def arnoldi(a: Op, v0, m, to_dim=None, want_V=False, cost=None):
    v0 = np.ascontiguousarray(v0, dtype=np.float64)
    n = len(v0)
    H = np.zeros((m + 1) * m)
    V = np.zeros(n * (m + 1)) if want_V else None
    cur, bd = C.c_int(), C.c_int()
    c = np.zeros(3) if cost is None else cost
    _ck(lib().orc_arnoldi(a.h, _p(v0), m, to_dim or m, _p(H), C.byref(cur), C.byref(bd),
                          _p(V) if want_V else None, _p(c)))
    out = {"H": H.reshape((m, m + 1)).T.copy(), "cur_dim": cur.value, "breakdown": bool(bd.value)}
    if want_V:
        out["V"] = V.reshape((m + 1, n)).T.copy()
    return out


def harmonic_from_H(H, d):
    m = H.shape[1]
    h = np.ascontiguousarray(H.T.ravel())
    re, im = np.zeros(d), np.zeros(d)
    _ck(lib().orc_harmonic_from_H(_p(h), m, d, _p(re), _p(im)))
    return re + 1j * im


def ritz_from_H(H, d, ordering=0):
    m = H.shape[1]
    h = np.ascontiguousarray(H.T.ravel())
    re, im, rs = np.zeros(d), np.zeros(d), np.zeros(d)
    _ck(lib().orc_ritz_from_H(_p(h), m, d, ordering, _p(re), _p(im), _p(rs)))
    return re + 1j * im, rs


def block2_operator(a: Op) -> Op:
    h = vp()
    _ck(lib().orc_block2_operator(a.h, C.byref(h)))
    return Op(h, (a,))


def shifted_operator(a: Op, mu) -> Op:
    h = vp()
    _ck(lib().orc_shifted_operator(a.h, C.c_double(mu), C.byref(h)))
    return Op(h, (a,))


def build_two_vector_poly(a: Op, b1, b2, degree, cost=None):
    b1 = np.ascontiguousarray(b1, dtype=np.float64)
    b2 = np.ascontiguousarray(b2, dtype=np.float64)
    re, im, nr = np.zeros(max(degree, 1)), np.zeros(max(degree, 1)), C.c_int()
    c = np.zeros(3) if cost is None else cost
    _ck(lib().orc_build_two_vector_poly(a.h, _p(b1), _p(b2), degree, _p(re), _p(im), C.byref(nr), _p(c)))
    return re[:nr.value] + 1j * im[:nr.value]


def damped_start(a: Op, b, alpha, power, cost=None):
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = np.empty_like(b)
    c = np.zeros(3) if cost is None else cost
    _ck(lib().orc_damped_start(a.h, _p(b), C.c_double(alpha), power, _p(out), _p(c)))
    return out


def check_ideal_order(mu, nev):
    re, im = _ri(mu)
    h = C.c_int()
    _ck(lib().orc_check_ideal_order(_p(re), _p(im), len(re), nev, C.byref(h)))
    return bool(h.value)


def read_matrix_market(path) -> Csr:
    h = vp()
    _ck(lib().orc_read_matrix_market(str(path).encode(), C.byref(h)))
    return Csr(h)


def solve(a: Op, m, k, nev, degree=0, rtol_multiplier=1e-8, rtol_absolute=0.0, stability=False,
          double=None, max_cycles=100, seed=1, allow_nev_above_k=False, damping=0,
          damping_alpha=0.0, damping_power=1, mid_cycle_stride=0, stagnation_window=0,
          stagnation_rtol=0.01, variant="ritz"):
    """mid_cycle_stride > 0 turns on check_mid_cycle; stagnation_window > 0
    turns on stagnation_stop (SolveConfig, inc/solver.hpp:45-52)."""
    cap_r, cap_c = 4096, max(max_cycles, 1)
    er, ei, rs = np.zeros(nev), np.zeros(nev), np.zeros(nev)
    cv = np.zeros(nev, dtype=np.int32)
    pr, pi, ir, ii = (np.zeros(cap_r) for _ in range(4))
    cm = np.zeros(cap_c)
    o = _SolveOut()
    o.cap_nev, o.cap_roots, o.cap_cycles = nev, cap_r, cap_c
    o.eig_re, o.eig_im, o.residuals = (x.ctypes.data_as(_dp) for x in (er, ei, rs))
    o.conv = cv.ctypes.data_as(_ip)
    o.poly_re, o.poly_im, o.inner_re, o.inner_im = (x.ctypes.data_as(_dp) for x in (pr, pi, ir, ii))
    o.cycle_max = cm.ctypes.data_as(_dp)
    d1, d2 = double if double else (0, 0)
    _ck(lib().orc_solve(a.h, m, k, nev, degree, rtol_multiplier, rtol_absolute, int(bool(stability)),
                        1 if double else 0, d1, d2, max_cycles, seed, int(allow_nev_above_k),
                        int(damping), C.c_double(damping_alpha), int(damping_power),
                        int(mid_cycle_stride), int(stagnation_window),
                        C.c_double(stagnation_rtol), 1 if variant == "harmonic" else 0,
                        C.byref(o)))
    ne = min(o.n_eig, nev)
    return {
        "eigenvalues": er[:ne] + 1j * ei[:ne], "residuals": rs[:ne].copy(),
        "converged_flags": cv[:ne].astype(bool), "converged": bool(o.converged), "cycles": o.cycles,
        "composite_degree": o.composite, "poly": pr[:o.n_poly] + 1j * pi[:o.n_poly],
        "inner_poly": ir[:o.n_inner] + 1j * ii[:o.n_inner], "rtol": o.rtol, "max_err": o.max_err,
        "norm_estimate": o.norm_est, "cost": {"mvps": o.mvps, "dots": o.dots, "vops": o.vops},
        "cycle_max_residual": cm[:o.n_cycles].copy(), "wall": o.wall, "discarded": o.discarded,
    }


def time_poly_factors(a: Op, roots, nfactors, reps=1) -> float:
    re, im = _ri(roots)
    return float(lib().orc_time_poly_factors(a.h, _p(re), _p(im), len(re), nfactors, reps))


def time_mgs2_step(n: int, c: int, reps: int = 1) -> float:
    """Seconds per orthogonalisation step of arnoldi_extend at basis size c
    (src/arnoldi.cpp:129-150 without the operator application)."""
    return float(lib().orc_time_mgs2_step(n, c, reps))
