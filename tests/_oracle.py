"""ctypes binding of the C oracle (oracle/tpdg_oracle.c) + golden-fixture loader.

Test infrastructure: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg import this module.
"""
import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
LIB_PATH = os.path.join(ROOT, "oracle", "build", "liboracle.so")

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
i64p = C.POINTER(C.c_int64)


class OrSys(C.Structure):
    _fields_ = [("dim", C.c_int), ("n_c", C.c_int), ("q", C.c_int), ("mu", C.c_int), ("n_elements", C.c_int),
                ("g", dp), ("d", dp), ("gw", dp), ("dw", dp), ("w", dp), ("jdet", dp), ("face_w", dp),
                ("conn", i64p), ("dft", dp), ("dfm", dp), ("dfp", dp)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "port"])
        L = C.CDLL(LIB_PATH)
        L.or_form_ksvd.restype = C.c_void_p
        L.or_form_ksvd.argtypes = [C.POINTER(OrSys), C.c_double, C.c_double, C.c_int, C.c_int, dp, dp]
        for name in ["or_pc_free"]:
            getattr(L, name).argtypes = [C.c_void_p]
        for name in ["or_pc_num_fallbacks", "or_pc_factor_len"]:
            getattr(L, name).argtypes = [C.c_void_p]
            getattr(L, name).restype = C.c_int
        L.or_pc_fallbacks.argtypes = [C.c_void_p, i64p]
        L.or_pc_has_factors.argtypes = [C.c_void_p, C.c_int]
        L.or_pc_factors.argtypes = [C.c_void_p, C.c_int, dp]
        L.or_pc_apply.argtypes = [C.c_void_p, dp, dp]
        L.or_pc_record_len.argtypes = [C.c_void_p]
        L.or_pc_record_len.restype = C.c_int
        L.or_pc_piv_len.argtypes = [C.c_void_p]
        L.or_pc_piv_len.restype = C.c_int
        L.or_pc_record.argtypes = [C.c_void_p, C.c_int, dp, ip]
        L.or_gmres.argtypes = [C.POINTER(OrSys), C.c_double, C.c_double, C.c_int, C.c_void_p, dp, C.c_double,
                               C.c_int, C.c_int, C.c_int, dp, ip, dp, C.c_int, ip]
        _lib = L
    return _lib


def ptr(a, t=dp):
    return a.ctypes.data_as(t)


class System:
    """Flat reference-layout arrays of one discretization (+ linearization cache)."""

    def __init__(self, arrays):
        self.a = {k: np.ascontiguousarray(v) for k, v in arrays.items()}
        m = self.a["meta"]
        self.dim, self.n_c, self.p, self.mu, self.n_elements = (int(x) for x in m[:5])
        self.dt = float(m[5])
        self.small = int(m[6])
        self.q = self.p + 1
        self.npe = self.q ** self.dim
        self.N = self.n_elements * self.n_c * self.npe
        self.a["conn"] = self.a["conn"].astype(np.int64)
        self._or = OrSys(self.dim, self.n_c, self.q, self.mu, self.n_elements,
                         *(ptr(self.a[k]) for k in ["ref_g", "ref_d", "ref_gw", "ref_dw", "ref_w", "jdet", "face_w"]),
                         ptr(self.a["conn"], i64p), *(ptr(self.a[k]) for k in ["dft", "dfm", "dfp"]))

    def __getitem__(self, k):
        return self.a[k]

    def __contains__(self, k):
        return k in self.a

    @property
    def coeffs(self):
        return 1.0, -self.dt  # LinearizedOperator a = 1, b = -dt (ops/linearized.hpp:177-178)

    # ---- oracle calls
    def jv(self, v):
        out = np.zeros(self.N)
        a, b = self.coeffs
        lib().or_jv(C.byref(self._or), C.c_double(a), C.c_double(b), self.small, ptr(np.ascontiguousarray(v)), ptr(out))
        return out

    def shuffled(self, e, vec, transpose=False, comp=0):
        q, ncb = self.q, (1 if self.small else self.n_c)
        m1 = ncb * q
        m2 = q if self.dim == 2 else q * q
        out = np.zeros(m2 * m2 if transpose else m1 * m1)
        a, b = self.coeffs
        lib().or_shuffled(C.byref(self._or), e, C.c_double(a), C.c_double(b), self.small, comp, int(transpose),
                          ptr(np.ascontiguousarray(vec)), ptr(out))
        return out

    def block(self, e, comp=0):
        n = self.npe if self.small else self.n_c * self.npe
        out = np.zeros(n * n)
        a, b = self.coeffs
        lib().or_assemble_block(C.byref(self._or), e, C.c_double(a), C.c_double(b), self.small, comp, ptr(out))
        return out.reshape(n, n)

    def form(self, start_vec=None, start_vec2=None, terms=2):
        sv = start_vec if start_vec is not None else self.a["start_vec"]
        sv2 = start_vec2 if start_vec2 is not None else self.a.get("start_vec2", sv)
        a, b = self.coeffs
        h = lib().or_form_ksvd(C.byref(self._or), C.c_double(a), C.c_double(b), self.small, terms,
                               ptr(np.ascontiguousarray(sv)), ptr(np.ascontiguousarray(sv2)))
        return OraclePC(h, self)


class OraclePC:
    def __init__(self, handle, sys):
        self.h = C.c_void_p(handle)
        self.sys = sys
        self.nblk = sys.n_elements * (sys.n_c if sys.small else 1)

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_pc_free(self.h)
            self.h = None

    def fallbacks(self):
        n = lib().or_pc_num_fallbacks(self.h)
        out = np.zeros(2 * max(n, 1), dtype=np.int64)
        lib().or_pc_fallbacks(self.h, ptr(out, i64p))
        return out[: 2 * n].reshape(n, 2)

    def has(self):
        return np.array([lib().or_pc_has_factors(self.h, i) for i in range(self.nblk)], dtype=np.int64)

    def factors(self, blk):
        out = np.zeros(lib().or_pc_factor_len(self.h))
        lib().or_pc_factors(self.h, blk, ptr(out))
        return out

    def record(self, blk):
        """(LU factors + Schur pairs, pivots) of one factored block."""
        rec = np.zeros(lib().or_pc_record_len(self.h))
        piv = np.zeros(lib().or_pc_piv_len(self.h), dtype=np.int32)
        lib().or_pc_record(self.h, blk, ptr(rec), piv.ctypes.data_as(ip))
        return rec, piv

    def apply(self, x):
        out = np.zeros(self.sys.N)
        lib().or_pc_apply(self.h, ptr(np.ascontiguousarray(x)), ptr(out))
        return out

    def gmres(self, rhs, tol=1e-10, restart=30, max_it=2000, left=False):
        s = self.sys
        x = np.zeros(s.N)
        its = C.c_int()
        conv = C.c_int()
        hist = np.zeros(max_it + 1)
        a, b = s.coeffs
        nh = lib().or_gmres(C.byref(s._or), C.c_double(a), C.c_double(b), s.small, self.h,
                            ptr(np.ascontiguousarray(rhs)), C.c_double(tol), restart, max_it, int(left), ptr(x),
                            C.byref(its), ptr(hist), len(hist), C.byref(conv))
        return x, its.value, hist[:nh], bool(conv.value)


def load(case):
    with np.load(os.path.join(GOLDEN, case + ".npz")) as z:
        return System({k: z[k] for k in z.files})


def load_raw(case):
    with np.load(os.path.join(GOLDEN, case + ".npz")) as z:
        return {k: z[k] for k in z.files}


def uniform_vector(seed, n, scale=1.0):
    out = np.zeros(n)
    lib().or_uniform_vector(C.c_uint64(seed), C.c_long(n), C.c_double(scale), ptr(out))
    return out


def seeded_unit_vector(n, seed=0x5EED):
    out = np.zeros(n)
    lib().or_seeded_unit_vector(C.c_long(n), C.c_uint64(seed), ptr(out))
    return out


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
