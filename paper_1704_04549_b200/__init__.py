"""B200-native (sm_100a) KSVD-preconditioned matrix-free GMRES for very-high-order DG.

Python mirror of the reference's operator / preconditioner interface
(reference proj/include/tpdg/: make_linearized_operator + jacobian_apply
ops/linearized.hpp:187-240, form_ksvd_2d/3d + KsvdPC*::apply precond/ksvd.hpp:161-372,
gmres solve/gmres.hpp:52-179, the Error hierarchy common/error.hpp:9-42), bound with
ctypes to the C ABI of ``libtpdg_gpu.so`` (include/tpdg_gpu.h). All compute runs in the
CUDA library; there is no host fallback: if the library is missing, importing the
compute entry points raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TPDG_GPU_LIB") or os.path.join(_HERE, "libtpdg_gpu.so")  # override: A/B builds

__all__ = [
    "Error", "ShapeError", "SingularError", "StateError", "ConvergenceError", "ConfigError", "GmresFailure",
    "Context", "System", "LinearizedOperator", "KsvdConfig", "GmresConfig", "GmresResult", "KsvdPC",
    "form_ksvd", "gmres", "setup_advection", "uniform_vector", "seeded_unit_vector", "lib", "build", "build_advection_cache",
]


# --------------------------------------------------------------------------- errors (common/error.hpp)
class Error(RuntimeError):
    pass


class ShapeError(Error):
    pass


class SingularError(Error):
    pass


class StateError(Error):
    pass


class ConvergenceError(Error):
    pass


class ConfigError(Error):
    pass


class CudaError(Error):
    pass


class GmresFailure(ConvergenceError):
    """Budget exhausted; carries the best iterate (solve/gmres.hpp:39-44)."""

    def __init__(self, what, result):
        super().__init__(what)
        self.result = result


_STATUS = {1: ShapeError, 2: SingularError, 3: StateError, 4: ConvergenceError, 5: ConfigError, 6: CudaError}

dp = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)
ip = C.POINTER(C.c_int)


class _System(C.Structure):
    _fields_ = [("dim", C.c_int), ("n_c", C.c_int), ("p", C.c_int), ("mu", C.c_int), ("n_elements", C.c_int),
                ("g", dp), ("d", dp), ("gw", dp), ("dw", dp), ("w", dp), ("jdet", dp), ("face_w", dp),
                ("conn", i64p), ("dft", dp), ("dfm", dp), ("dfp", dp), ("state_hash", C.c_uint64)]


class _KsvdCfg(C.Structure):
    _fields_ = [("terms", C.c_int), ("lanczos_max_it", C.c_int), ("breakdown_tol", C.c_double),
                ("seed", C.c_uint64), ("degenerate_tol", C.c_double)]


class _GmresCfg(C.Structure):
    _fields_ = [("tol", C.c_double), ("restart", C.c_int), ("max_iterations", C.c_int), ("side", C.c_int)]


_lib = None

EXPORTS = [
    "tpdg_gpu_last_error", "tpdg_gpu_version", "tpdg_gpu_nccl_unique_id", "tpdg_gpu_ctx_create",
    "tpdg_gpu_ctx_destroy", "tpdg_gpu_ctx_stream", "tpdg_gpu_ctx_sync", "tpdg_gpu_ctx_launches",
    "tpdg_gpu_ctx_profile", "tpdg_gpu_ctx_profile_read",
    "tpdg_gpu_op_create", "tpdg_gpu_op_destroy", "tpdg_gpu_op_local_size", "tpdg_gpu_op_check_hash",
    "tpdg_gpu_jv", "tpdg_gpu_jv_host", "tpdg_gpu_shuffled_host", "tpdg_gpu_form_ksvd",
    "tpdg_gpu_pc_import_factors", "tpdg_gpu_pc_import_record", "tpdg_gpu_form_block_jacobi", "tpdg_gpu_pc_destroy", "tpdg_gpu_pc_num_fallbacks", "tpdg_gpu_pc_fallbacks",
    "tpdg_gpu_pc_factor_len", "tpdg_gpu_pc_export_factors", "tpdg_gpu_pc_apply", "tpdg_gpu_pc_apply_host",
    "tpdg_gpu_gmres", "tpdg_gpu_gmres_host", "tpdg_setup_advection", "tpdg_setup_system", "tpdg_setup_destroy", "tpdg_setup_geometry",
    "tpdg_gpu_build_cache_advection", "tpdg_gpu_libm_eval", "tpdg_gpu_mgs_step", "tpdg_gpu_build_cache_euler", "tpdg_setup_euler",
    "tpdg_setup_state", "tpdg_gpu_residual_euler", "tpdg_gpu_step_backward_euler",
    "tpdg_uniform_vector", "tpdg_seeded_unit_vector", "tpdg_halo_plan_create", "tpdg_halo_plan_query",
    "tpdg_halo_plan_conn", "tpdg_halo_plan_halo_gid", "tpdg_halo_plan_peer", "tpdg_halo_plan_destroy",
    "tpdg_gpu_loopback_create", "tpdg_gpu_loopback_destroy", "tpdg_gpu_ctx_create_loopback",
]


def build():
    """Compile libtpdg_gpu.so for sm_100a in-tree (nvcc cross-compiles without a GPU)."""
    import subprocess
    subprocess.check_call(["make", "-C", os.path.join(_HERE, "csrc"), "-j8"])


def lib():
    """Load the CUDA library; raises if it is missing (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run paper_1704_04549_b200.build() (there is no CPU fallback)")
    try:  # torch first: its bundled libnccl.so.2 (newer) then also serves this library's NCCL dependency;
        import torch  # noqa: F401  loading ours first would bind the older system NCCL and break torch's import
    except ImportError:
        pass
    L = C.CDLL(LIB_PATH)
    v = C.c_void_p
    L.tpdg_gpu_last_error.restype = C.c_char_p
    L.tpdg_gpu_version.restype = C.c_char_p
    sig = {
        "tpdg_gpu_nccl_unique_id": [v],
        "tpdg_gpu_ctx_create": [C.c_int, C.c_int, C.c_int, v, C.POINTER(v)],
        "tpdg_gpu_ctx_destroy": [v], "tpdg_gpu_ctx_stream": [v, C.POINTER(v)], "tpdg_gpu_ctx_sync": [v],
        "tpdg_gpu_ctx_launches": [v, i64p], "tpdg_gpu_ctx_profile": [v, C.c_int],
        "tpdg_gpu_ctx_profile_read": [v, dp, i64p],
        "tpdg_gpu_op_create": [v, C.POINTER(_System), C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(v)],
        "tpdg_gpu_op_destroy": [v], "tpdg_gpu_op_local_size": [v, i64p], "tpdg_gpu_op_check_hash": [v, C.c_uint64],
        "tpdg_gpu_jv": [v, v, v], "tpdg_gpu_jv_host": [v, dp, dp],
        "tpdg_gpu_shuffled_host": [v, C.c_int, C.c_int, C.c_int, dp, dp],
        "tpdg_gpu_form_ksvd": [v, C.POINTER(_KsvdCfg), C.POINTER(v)],
        "tpdg_gpu_pc_import_factors": [v, dp, i64p, C.POINTER(v)],
        "tpdg_gpu_pc_import_record": [v, dp, i64p, dp, ip, C.POINTER(v)],
        "tpdg_gpu_form_block_jacobi": [v, C.c_int64, C.POINTER(v)],
        "tpdg_gpu_pc_destroy": [v], "tpdg_gpu_pc_num_fallbacks": [v, C.POINTER(C.c_int)],
        "tpdg_gpu_pc_fallbacks": [v, i64p], "tpdg_gpu_pc_factor_len": [v, C.POINTER(C.c_int)],
        "tpdg_gpu_pc_export_factors": [v, C.c_int, dp, C.POINTER(C.c_int)],
        "tpdg_gpu_pc_apply": [v, v, v], "tpdg_gpu_pc_apply_host": [v, dp, dp],
        "tpdg_gpu_gmres": [v, v, v, v, C.POINTER(_GmresCfg), C.POINTER(C.c_int), dp, C.c_int, C.POINTER(C.c_int)],
        "tpdg_gpu_gmres_host": [v, v, dp, dp, C.POINTER(_GmresCfg), C.POINTER(C.c_int), dp, C.c_int,
                                C.POINTER(C.c_int)],
        "tpdg_setup_advection": [C.c_int, dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(v)],
        "tpdg_setup_system": [v, C.POINTER(_System)], "tpdg_setup_destroy": [v],
        "tpdg_setup_geometry": [v, C.POINTER(dp), C.POINTER(dp), C.POINTER(dp), C.POINTER(dp), C.POINTER(C.c_int),
                                C.POINTER(C.c_int)],
        "tpdg_gpu_build_cache_advection": [v, C.c_int, C.c_int, C.c_int, C.c_int, v, v, v, v, v, C.c_int, dp, v, v, v],
        "tpdg_gpu_libm_eval": [v, C.c_int, C.c_int64, v, v, v],
        "tpdg_gpu_mgs_step": [v, v, C.c_int64, C.c_int, C.c_int64, v],
        "tpdg_gpu_build_cache_euler": [v, C.c_int, C.c_int, C.c_int, C.c_int, v, v, v, v, v, v, v, v],
        "tpdg_setup_euler": [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(v)],
        "tpdg_setup_state": [v, C.POINTER(dp), C.POINTER(C.c_int64)],
        "tpdg_gpu_residual_euler": [v, C.c_int, C.c_int, C.c_int, C.c_int, v, v, v, v, v, v, v, v, v],
        "tpdg_gpu_step_backward_euler": [v, C.POINTER(_System), dp, dp, dp, C.c_double, C.c_double, C.c_int,
                                         C.c_double, C.POINTER(_GmresCfg), C.POINTER(_KsvdCfg), C.c_int,
                                         C.POINTER(C.c_int), C.POINTER(C.c_int), dp, C.c_int],
        "tpdg_uniform_vector": [C.c_uint64, C.c_int64, C.c_double, dp],
        "tpdg_seeded_unit_vector": [C.c_int64, C.c_uint64, dp],
        "tpdg_halo_plan_create": [C.POINTER(_System), C.c_int, C.c_int, C.POINTER(v)],
        "tpdg_halo_plan_query": [v] + [C.POINTER(C.c_int)] * 4,
        "tpdg_halo_plan_conn": [v, C.POINTER(C.c_int)], "tpdg_halo_plan_halo_gid": [v, C.POINTER(C.c_int)],
        "tpdg_halo_plan_peer": [v, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                C.POINTER(C.c_int), C.POINTER(C.c_int)],
        "tpdg_gpu_loopback_create": [C.c_int, C.POINTER(v)], "tpdg_gpu_loopback_destroy": [v],
        "tpdg_gpu_ctx_create_loopback": [C.c_int, C.c_int, v, C.POINTER(v)],
        "tpdg_halo_plan_destroy": [v],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    _lib = L
    return L


def _check(rc):
    if rc != 0:
        msg = lib().tpdg_gpu_last_error().decode()
        raise _STATUS.get(rc, Error)(msg)


def _ptr(a):
    return a.ctypes.data_as(dp)


def _dptr(x):
    """Device pointer of a torch CUDA tensor (or an int address)."""
    if isinstance(x, int):
        return C.c_void_p(x)
    return C.c_void_p(x.data_ptr())


# --------------------------------------------------------------------------- host-side inputs
def uniform_vector(seed, n, scale=1.0):
    """std::mt19937_64(seed) + uniform_real_distribution(-scale, scale) (tests/support/test_rng.hpp)."""
    out = np.empty(int(n))
    _check(lib().tpdg_uniform_vector(C.c_uint64(seed), C.c_int64(n), C.c_double(scale), _ptr(out)))
    return out


def seeded_unit_vector(n, seed=0x5EED):
    """tpdg::detail::seeded_unit_vector (tensor/lanczos.hpp:61-72)."""
    out = np.empty(int(n))
    _check(lib().tpdg_seeded_unit_vector(C.c_int64(n), C.c_uint64(seed), _ptr(out)))
    return out


class System:
    """Discretization + linearization cache as flat reference-layout arrays.

    Keys: meta-free attributes dim, n_c, p, mu, n_elements and arrays g, d, gw, dw, w, jdet,
    face_w, conn ([E][2d][3] int64), dft, dfm, dfp.
    """

    def __init__(self, dim, n_c, p, mu, n_elements, arrays, state_hash=0):
        self.dim, self.n_c, self.p, self.mu, self.n_elements = int(dim), int(n_c), int(p), int(mu), int(n_elements)
        self.q = self.p + 1
        self.npe = self.q ** self.dim
        self.N = self.n_elements * self.n_c * self.npe
        self.arrays = {k: np.ascontiguousarray(v, dtype=np.int64 if k == "conn" else np.float64)
                       for k, v in arrays.items()}
        self.state_hash = int(state_hash)

    @classmethod
    def from_golden(cls, z):
        m = z["meta"]
        keys = {"g": "ref_g", "d": "ref_d", "gw": "ref_gw", "dw": "ref_dw", "w": "ref_w", "jdet": "jdet",
                "face_w": "face_w", "conn": "conn", "dft": "dft", "dfm": "dfm", "dfp": "dfp"}
        return cls(m[0], m[1], m[2], m[3], m[4], {k: z[v] for k, v in keys.items()})

    def _c(self):
        a = self.arrays
        return _System(self.dim, self.n_c, self.p, self.mu, self.n_elements,
                       *(_ptr(a[k]) for k in ["g", "d", "gw", "dw", "w", "jdet", "face_w"]),
                       a["conn"].ctypes.data_as(i64p), *(_ptr(a[k]) for k in ["dft", "dfm", "dfp"]),
                       C.c_uint64(self.state_hash))


def _system_from_setup(h, field, v):
    s = _System()
    _check(lib().tpdg_setup_system(h, C.byref(s)))
    dim, nc = s.dim, s.n_c
    q, mu = s.p + 1, s.mu
    E = s.n_elements
    nqv = mu ** dim
    nqf = nqv // mu

    def arr(ptr, n, dtype=np.float64):
        return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)

    arrays = {"g": arr(s.g, mu * q), "d": arr(s.d, mu * q), "gw": arr(s.gw, mu * q), "dw": arr(s.dw, mu * q),
              "w": arr(s.w, mu), "jdet": arr(s.jdet, E * nqv), "face_w": arr(s.face_w, E * 2 * dim * nqf),
              "conn": arr(s.conn, E * 2 * dim * 3, np.int64), "dft": arr(s.dft, E * dim * nqv * nc * nc),
              "dfm": arr(s.dfm, E * 2 * dim * nqf * nc * nc), "dfp": arr(s.dfp, E * 2 * dim * nqf * nc * nc)}
    sysm = System(dim, nc, s.p, mu, E, arrays, s.state_hash)
    ga, gx, gn, gf = dp(), dp(), dp(), dp()
    nv, nf = C.c_int(), C.c_int()
    _check(lib().tpdg_setup_geometry(h, C.byref(ga), C.byref(gx), C.byref(gn), C.byref(gf), C.byref(nv),
                                     C.byref(nf)))
    sysm.geometry = {"adj": arr(ga, E * nv.value * dim * dim), "vol_x": arr(gx, E * nv.value * dim),
                     "face_n": arr(gn, E * 2 * dim * nf.value * dim), "face_x": arr(gf, E * 2 * dim * nf.value * dim),
                     "field": field, "vel": np.array([v[0], v[1], v[2] if dim == 3 else 0.0])}
    if nc > 1:
        sp, ns = dp(), C.c_int64()
        _check(lib().tpdg_setup_state(h, C.byref(sp), C.byref(ns)))
        sysm.state = arr(sp, ns.value)
    return sysm


def setup_advection(kind, nx, ny=None, nz=1, p=1, vel=(1.0, 0.5, 0.0), periodic=True):
    """Host input production for the BASELINE advection configs.

    kind: "const2d" (velocity vel[:2]), "swirl2d" (sin 2 pi y, cos 2 pi x), "const3d" (vel)."""
    k = {"const2d": 0, "swirl2d": 1, "const3d": 2}[kind]
    ny = nx if ny is None else ny
    h = C.c_void_p()
    v = np.asarray(vel, dtype=np.float64)
    _check(lib().tpdg_setup_advection(k, _ptr(v), nx, ny, nz, p, int(periodic), C.byref(h)))
    try:
        return _system_from_setup(h, k, v)
    finally:
        lib().tpdg_setup_destroy(h)


def setup_euler(case, nx, ny=None, nz=1, p=1):
    """Euler stand-ins of BASELINE configs[2] ("cfg3": 2D, [0,10]^2, Gaussian density + swirl, p = rho^gamma)
    and configs[4] ("cfg5": 3D Taylor-Green on [0,2pi]^3, Mach 0.1), LLF flux (the reference's euler_law; the
    Roe flux of cfg3 and the BR2 viscous terms of cfg5 have no reference implementation). Returns a System with
    the interpolated nodal state in .state and a zero cache: fill it with build_euler_cache."""
    k = {"cfg3": 3, "cfg5": 5}[case]
    ny = nx if ny is None else ny
    h = C.c_void_p()
    _check(lib().tpdg_setup_euler(k, nx, ny, nz, p, C.byref(h)))
    try:
        return _system_from_setup(h, k, np.zeros(3))
    finally:
        lib().tpdg_setup_destroy(h)


def build_euler_cache(ctx: "Context", sysm: "System", state=None):
    """build_cache (ops/linearized.hpp:38-100) of the LLF Euler law on the device; stores host copies of
    (dft, dfm, dfp) in sysm.arrays and returns them."""
    import torch
    g = sysm.geometry
    dim, E, mu, q = sysm.dim, sysm.n_elements, sysm.mu, sysm.q
    nc = sysm.n_c
    nvol, nface = mu ** dim, mu ** (dim - 1)
    dev = torch.device("cuda", ctx.device)
    st = np.ascontiguousarray(sysm.state if state is None else state, dtype=np.float64)
    t = {k: torch.from_numpy(np.ascontiguousarray(g[k])).to(dev) for k in ("adj", "face_n")}
    dg = torch.from_numpy(np.ascontiguousarray(sysm.arrays["g"])).to(dev)
    dst = torch.from_numpy(st).to(dev)
    conn = torch.from_numpy(sysm.arrays["conn"]).to(dev)
    dft = torch.zeros(E * dim * nvol * nc * nc, dtype=torch.float64, device=dev)
    dfm = torch.zeros(E * 2 * dim * nface * nc * nc, dtype=torch.float64, device=dev)
    dfp = torch.zeros_like(dfm)
    _check(lib().tpdg_gpu_build_cache_euler(ctx.h, dim, q - 1, mu, E, C.c_void_p(dg.data_ptr()),
                                            C.c_void_p(dst.data_ptr()), C.c_void_p(t["adj"].data_ptr()),
                                            C.c_void_p(t["face_n"].data_ptr()), C.c_void_p(conn.data_ptr()),
                                            C.c_void_p(dft.data_ptr()), C.c_void_p(dfm.data_ptr()),
                                            C.c_void_p(dfp.data_ptr())))
    out = dft.cpu().numpy(), dfm.cpu().numpy(), dfp.cpu().numpy()
    sysm.arrays["dft"], sysm.arrays["dfm"], sysm.arrays["dfp"] = out
    return out


def build_advection_cache(ctx: "Context", sysm: "System"):
    """build_cache (ops/linearized.hpp:38-100) of scalar upwind advection on the device from the geometry of a
    setup_advection system: returns host copies (dft, dfm, dfp) in the reference layouts."""
    import torch
    g = sysm.geometry
    dim, E, mu = sysm.dim, sysm.n_elements, sysm.mu
    nvol, nface = mu ** dim, mu ** (dim - 1)
    dev = torch.device("cuda", ctx.device)
    t = {k: torch.from_numpy(np.ascontiguousarray(g[k])).to(dev) for k in ("adj", "vol_x", "face_n", "face_x")}
    conn = torch.from_numpy(sysm.arrays["conn"]).to(dev)
    dft = torch.empty(E * dim * nvol, dtype=torch.float64, device=dev)
    dfm = torch.empty(E * 2 * dim * nface, dtype=torch.float64, device=dev)
    dfp = torch.empty_like(dfm)
    vel = np.ascontiguousarray(g["vel"], dtype=np.float64)
    _check(lib().tpdg_gpu_build_cache_advection(ctx.h, dim, E, nvol, nface, *(C.c_void_p(t[k].data_ptr()) for k in
                                                ("adj", "vol_x", "face_n", "face_x")), C.c_void_p(conn.data_ptr()),
                                                int(g["field"]), _ptr(vel), C.c_void_p(dft.data_ptr()),
                                                C.c_void_p(dfm.data_ptr()), C.c_void_p(dfp.data_ptr())))
    return dft.cpu().numpy(), dfm.cpu().numpy(), dfp.cpu().numpy()


def residual_euler(ctx: "Context", sysm: "System", state=None) -> np.ndarray:
    """residual r(u, t) (ops/discretization.hpp:188-254) of the LLF Euler law on the device (host in/out)."""
    import torch
    g = sysm.geometry
    dev = torch.device("cuda", ctx.device)
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in
         (("g", sysm.arrays["g"]), ("gw", sysm.arrays["gw"]), ("dw", sysm.arrays["dw"]), ("adj", g["adj"]),
          ("face_n", g["face_n"]), ("face_w", sysm.arrays["face_w"]), ("conn", sysm.arrays["conn"]),
          ("state", sysm.state if state is None else np.asarray(state, dtype=np.float64)))}
    out = torch.empty_like(t["state"])
    _check(lib().tpdg_gpu_residual_euler(ctx.h, sysm.dim, sysm.p, sysm.mu, sysm.n_elements,
                                         *(C.c_void_p(t[k].data_ptr()) for k in
                                           ("g", "gw", "dw", "state", "adj", "face_n", "face_w", "conn")),
                                         C.c_void_p(out.data_ptr())))
    return out.cpu().numpy()


@dataclass
class NewtonConfig:
    """NewtonConfig (solve/newton.hpp:11-21)."""
    tol: float = 1e-8
    max_iterations: int = 30
    absolute_floor: float = 1e-14


@dataclass
class StepStats:
    newton_steps: int = 0
    gmres_per_solve: list = field(default_factory=list)
    residual_norms: list = field(default_factory=list)


def step_backward_euler(ctx: "Context", sysm: "System", u, dt: float, gmres_cfg: "GmresConfig | None" = None,
                        newton_cfg: NewtonConfig | None = None, ksvd_cfg: "KsvdConfig | None" = None,
                        block_mode="full"):
    """One backward Euler step of the Euler law by Newton-GMRES with the KSVD preconditioner on the device
    (step_backward_euler, solve/time_step.hpp:136-146). Returns (u', StepStats)."""
    gmres_cfg = gmres_cfg or GmresConfig(tol=1e-10, restart=30, max_iterations=2000)
    newton_cfg = newton_cfg or NewtonConfig()
    ksvd_cfg = ksvd_cfg or KsvdConfig()
    uu = np.array(u, dtype=np.float64, copy=True)
    g = sysm.geometry
    adj = np.ascontiguousarray(g["adj"])
    fn = np.ascontiguousarray(g["face_n"])
    cap = newton_cfg.max_iterations + 1
    gits = np.zeros(cap, dtype=np.int32)
    norms = np.zeros(cap + 1)
    steps = C.c_int()
    gc = _gcfg(gmres_cfg)
    kc = _KsvdCfg(ksvd_cfg.terms, ksvd_cfg.lanczos_max_it, ksvd_cfg.breakdown_tol, C.c_uint64(ksvd_cfg.seed),
                  ksvd_cfg.degenerate_tol)
    cs = sysm._c()
    _check(lib().tpdg_gpu_step_backward_euler(ctx.h, C.byref(cs), _ptr(adj), _ptr(fn), _ptr(uu), C.c_double(dt),
                                              C.c_double(newton_cfg.tol), newton_cfg.max_iterations,
                                              C.c_double(newton_cfg.absolute_floor), C.byref(gc), C.byref(kc),
                                              {"full": 0, "small": 1}[block_mode], C.byref(steps),
                                              gits.ctypes.data_as(C.POINTER(C.c_int)), _ptr(norms), cap))
    n = steps.value
    return uu, StepStats(n, [int(x) for x in gits[:n]], [float(x) for x in norms[:n + 1]])


def libm_eval(ctx: "Context", fn: str, x, y=None) -> np.ndarray:
    """Test hook: the formation's device libm (csrc/glibm.cuh: glibc 2.39 sin/cos/atan/atan2 restated, as
    standardize_2x2 calls them, tensor/schur.hpp:91-108) over the host arrays x (and y for atan2(x, y))."""
    import torch
    code = {"sin": 0, "cos": 1, "atan": 2, "atan2": 3}[fn]
    dev = torch.device("cuda", ctx.device)
    dx = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev)
    dy = torch.from_numpy(np.ascontiguousarray(y, dtype=np.float64)).to(dev) if y is not None else None
    out = torch.empty_like(dx)
    _check(lib().tpdg_gpu_libm_eval(ctx.h, code, dx.numel(), C.c_void_p(dx.data_ptr()),
                                    C.c_void_p(dy.data_ptr()) if dy is not None else None, C.c_void_p(out.data_ptr())))
    return out.cpu().numpy()


def mgs_step(ctx: "Context", V, k: int, n: int) -> np.ndarray:
    """Test hook: one modified Gram-Schmidt step (solve/gmres.hpp:112-121) on the device tensor V (rows v_0 .. v_k
    and w = row k + 1, row stride V.stride(0)), in place; returns h[0 .. k + 1] (projections, then the norm)."""
    h = np.zeros(k + 2)
    _check(lib().tpdg_gpu_mgs_step(ctx.h, C.c_void_p(V.data_ptr()), V.stride(0), k, n,
                                   h.ctypes.data_as(C.c_void_p)))
    return h


def face_layer_nodes(dim: int, q: int, face: int) -> np.ndarray:
    """Element-block offsets of the node layer of `face` (lower tangential axis fastest): the nodal trace
    of ops/discretization.hpp:89-97 with Gauss-Lobatto nodes; host mirror of face_layer_index."""
    axis, layer = face // 2, (0 if face % 2 == 0 else q - 1)
    t = np.arange(q ** (dim - 1))
    if dim == 2:
        return layer + q * t if axis == 0 else t + q * layer
    u, w = t % q, t // q
    return {0: layer + q * (u + q * w), 1: u + q * (layer + q * w), 2: u + q * (w + q * layer)}[axis]


def halo_plan(sys: "System", rank: int, nranks: int) -> dict:
    """Element partition + face-neighbour halo plan of one rank (host only; op_create uses the
    same plan for nranks > 1). See include/tpdg_gpu.h."""
    h = C.c_void_p()
    cs = sys._c()
    _check(lib().tpdg_halo_plan_create(C.byref(cs), rank, nranks, C.byref(h)))
    try:
        eb, ee, nh, npeer = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(lib().tpdg_halo_plan_query(h, C.byref(eb), C.byref(ee), C.byref(nh), C.byref(npeer)))
        nl = ee.value - eb.value
        conn = np.zeros(max(1, nl * 2 * sys.dim * 3), dtype=np.int32)
        _check(lib().tpdg_halo_plan_conn(h, conn.ctypes.data_as(C.POINTER(C.c_int))))
        gid = np.zeros(max(1, nh.value), dtype=np.int32)
        _check(lib().tpdg_halo_plan_halo_gid(h, gid.ctypes.data_as(C.POINTER(C.c_int))))
        peers = []
        for i in range(npeer.value):
            r, ns, nr = C.c_int(), C.c_int(), C.c_int()
            _check(lib().tpdg_halo_plan_peer(h, i, C.byref(r), C.byref(ns), None, C.byref(nr), None))
            sp = np.zeros(max(2, 2 * ns.value), dtype=np.int32)
            rp = np.zeros(max(2, 2 * nr.value), dtype=np.int32)
            _check(lib().tpdg_halo_plan_peer(h, i, C.byref(r), C.byref(ns), sp.ctypes.data_as(C.POINTER(C.c_int)),
                                             C.byref(nr), rp.ctypes.data_as(C.POINTER(C.c_int))))
            peers.append({"rank": r.value, "send_pairs": sp[: 2 * ns.value].reshape(-1, 2).copy(),
                          "recv_pairs": rp[: 2 * nr.value].reshape(-1, 2).copy()})
        return {"e_begin": eb.value, "e_end": ee.value, "n_halo": nh.value,
                "conn": conn[: nl * 2 * sys.dim * 3].copy(), "halo_gid": gid[: nh.value].copy(), "peers": peers}
    finally:
        lib().tpdg_halo_plan_destroy(h)


# --------------------------------------------------------------------------- device objects
class Context:
    """One per GPU / rank: CUDA stream (+ NCCL communicator for nranks > 1)."""

    def __init__(self, device=0, rank=0, nranks=1, nccl_id=None, loopback=None):
        """loopback: a Loopback hub; the context then runs the multi-rank data plane in-process (one
        host thread per rank) instead of over NCCL."""
        self.h = C.c_void_p()
        self.rank, self.nranks, self.device = rank, nranks, device
        self._hub = loopback
        if loopback is not None:
            self.nranks = loopback.nranks
            _check(lib().tpdg_gpu_ctx_create_loopback(device, rank, loopback.h, C.byref(self.h)))
            return
        idbuf = None
        if nccl_id is not None:
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        _check(lib().tpdg_gpu_ctx_create(device, rank, nranks, idbuf, C.byref(self.h)))

    @staticmethod
    def nccl_unique_id():
        buf = C.create_string_buffer(128)
        _check(lib().tpdg_gpu_nccl_unique_id(buf))
        return buf.raw

    def stream(self):
        s = C.c_void_p()
        _check(lib().tpdg_gpu_ctx_stream(self.h, C.byref(s)))
        return s.value

    def sync(self):
        _check(lib().tpdg_gpu_ctx_sync(self.h))

    def launches(self):
        n = C.c_int64()
        _check(lib().tpdg_gpu_ctx_launches(self.h, C.byref(n)))
        return n.value

    def profile(self, enable=True):
        _check(lib().tpdg_gpu_ctx_profile(self.h, int(enable)))

    def profile_read(self):
        """{class: (total ms, count)} for classes pc_apply, jv, mgs, other."""
        ms = np.zeros(4)
        cnt = np.zeros(4, dtype=np.int64)
        _check(lib().tpdg_gpu_ctx_profile_read(self.h, _ptr(ms), cnt.ctypes.data_as(i64p)))
        return {name: (float(ms[i]), int(cnt[i])) for i, name in enumerate(["pc_apply", "jv", "mgs", "other"])}

    def close(self):
        if self.h:
            lib().tpdg_gpu_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Loopback:
    """In-process transport hub for nranks contexts (tpdg_gpu_loopback_create)."""

    def __init__(self, nranks):
        self.nranks = nranks
        self.h = C.c_void_p()
        _check(lib().tpdg_gpu_loopback_create(nranks, C.byref(self.h)))

    def close(self):
        if self.h:
            lib().tpdg_gpu_loopback_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def partition(n_elements, nranks, rank):
    """Contiguous element range of a rank: [E r / N, E (r+1) / N) (rows in 2D, slabs in 3D)."""
    return (n_elements * rank) // nranks, (n_elements * (rank + 1)) // nranks


class LinearizedOperator:
    """(M - dt J) (or J alone) bound to a linearization; mirrors make_linearized_operator."""

    def __init__(self, ctx: Context, sys: System, dt: float, jacobian_only=False, block_mode="full", e_range=None):
        self.ctx, self.sys, self.dt = ctx, sys, float(dt)
        self.block_mode = block_mode
        self.small = {"full": 0, "small": 1}[block_mode]
        if e_range is None:
            e_range = partition(sys.n_elements, ctx.nranks, ctx.rank)
        self.e_begin, self.e_end = e_range
        self.h = C.c_void_p()
        self._cs = sys._c()
        _check(lib().tpdg_gpu_op_create(ctx.h, C.byref(self._cs), C.c_double(dt), int(jacobian_only), self.small,
                                        self.e_begin, self.e_end, C.byref(self.h)))
        n = C.c_int64()
        _check(lib().tpdg_gpu_op_local_size(self.h, C.byref(n)))
        self.n_local = n.value

    def check_cache(self, expected_hash):
        _check(lib().tpdg_gpu_op_check_hash(self.h, C.c_uint64(expected_hash)))

    def jacobian_apply(self, v):
        """Host arrays in/out (jacobian_apply, ops/linearized.hpp:201)."""
        v = np.ascontiguousarray(v, dtype=np.float64)
        if v.size != self.n_local:
            raise ShapeError("jacobian_apply: state shape mismatch")
        out = np.empty(self.n_local)
        _check(lib().tpdg_gpu_jv_host(self.h, _ptr(v), _ptr(out)))
        return out

    def apply_device(self, d_in, d_out):
        _check(lib().tpdg_gpu_jv(self.h, _dptr(d_in), _dptr(d_out)))

    def shuffled_apply(self, e, v, transpose=False, comp=0):
        q, ncb = self.sys.q, (1 if self.small else self.sys.n_c)
        m1 = ncb * q
        m2 = q if self.sys.dim == 2 else q * q
        v = np.ascontiguousarray(v, dtype=np.float64)
        if v.size != (m1 * m1 if transpose else m2 * m2):
            raise ShapeError("shuffled_apply: input length mismatch")
        out = np.empty(m2 * m2 if transpose else m1 * m1)
        _check(lib().tpdg_gpu_shuffled_host(self.h, e, comp, int(transpose), _ptr(v), _ptr(out)))
        return out

    def close(self):
        if self.h:
            lib().tpdg_gpu_op_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class KsvdConfig:
    """KsvdConfig + LanczosConfig (precond/ksvd.hpp:16-20, tensor/lanczos.hpp:15-30)."""
    terms: int = 2
    lanczos_max_it: int = 0
    breakdown_tol: float = 1e-12
    seed: int = 0x5EED
    degenerate_tol: float = 1e-12


@dataclass
class GmresConfig:
    """GmresConfig (solve/gmres.hpp:14-29)."""
    tol: float = 1e-5
    restart: int = 60
    max_iterations: int = 2000
    side: str = "right"


@dataclass
class GmresResult:
    x: np.ndarray
    iterations: int = 0
    residual_history: list = field(default_factory=list)
    converged: bool = False


class KsvdPC:
    """Formed preconditioner (KsvdPC2D / KsvdPC3D, precond/ksvd.hpp:161-234)."""

    def __init__(self, op: LinearizedOperator, handle):
        self.op, self.h = op, handle
        self.mode = op.block_mode
        self.n_elements = op.e_end - op.e_begin
        self.n_c, self.npe, self.n1d = op.sys.n_c, op.sys.npe, op.sys.q
        self.nblk = self.n_elements * (op.sys.n_c if op.small else 1)
        n = C.c_int()
        _check(lib().tpdg_gpu_pc_num_fallbacks(self.h, C.byref(n)))
        fb = np.zeros(2 * max(n.value, 1), dtype=np.int64)
        _check(lib().tpdg_gpu_pc_fallbacks(self.h, fb.ctypes.data_as(i64p)))
        self.fallbacks = [(int(fb[2 * i]), int(fb[2 * i + 1])) for i in range(n.value)]

    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty(self.op.n_local)
        _check(lib().tpdg_gpu_pc_apply_host(self.h, _ptr(x), _ptr(out)))
        return out

    def apply_device(self, d_in, d_out):
        _check(lib().tpdg_gpu_pc_apply(self.h, _dptr(d_in), _dptr(d_out)))

    def factors(self, blk):
        """Raw factors of one block (2D: a1 b1 a2 b2, 3D: a1 b1 c1 b2 c2) and whether it has them."""
        n = C.c_int()
        _check(lib().tpdg_gpu_pc_factor_len(self.h, C.byref(n)))
        out = np.empty(n.value)
        has = C.c_int()
        _check(lib().tpdg_gpu_pc_export_factors(self.h, blk, _ptr(out), C.byref(has)))
        return out, bool(has.value)

    def close(self):
        if self.h:
            lib().tpdg_gpu_pc_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def form_ksvd(op: LinearizedOperator, cfg: KsvdConfig | None = None) -> KsvdPC:
    """form_ksvd_2d / form_ksvd_3d (dimension from the operator), formed on the device."""
    cfg = cfg or KsvdConfig()
    c = _KsvdCfg(cfg.terms, cfg.lanczos_max_it, cfg.breakdown_tol, C.c_uint64(cfg.seed), cfg.degenerate_tol)
    h = C.c_void_p()
    _check(lib().tpdg_gpu_form_ksvd(op.h, C.byref(c), C.byref(h)))
    return KsvdPC(op, h)


def form_block_jacobi(op: LinearizedOperator, max_total_entries: int = 300_000_000) -> KsvdPC:
    """form_block_jacobi (precond/block_jacobi.hpp:38-72): exact block-LU preconditioner on the device
    (same apply contract as the KSVD preconditioner)."""
    h = C.c_void_p()
    _check(lib().tpdg_gpu_form_block_jacobi(op.h, C.c_int64(max_total_entries), C.byref(h)))
    return KsvdPC(op, h)


def import_factors(op: LinearizedOperator, factors, has) -> KsvdPC:
    """Test hook: preconditioner from externally formed raw factors (e.g. the reference's)."""
    f = np.ascontiguousarray(factors, dtype=np.float64)
    hs = np.ascontiguousarray(has, dtype=np.int64)
    h = C.c_void_p()
    _check(lib().tpdg_gpu_pc_import_factors(op.h, _ptr(f), hs.ctypes.data_as(i64p), C.byref(h)))
    return KsvdPC(op, h)


def import_record(op: LinearizedOperator, factors, has, rec, piv) -> KsvdPC:
    """Test hook: preconditioner from an externally formed apply state (LU + Schur pairs and
    pivots of every factored block, e.g. the reference's), not recomputed on the device."""
    f = np.ascontiguousarray(factors, dtype=np.float64)
    hs = np.ascontiguousarray(has, dtype=np.int64)
    r = np.ascontiguousarray(rec, dtype=np.float64)
    pv = np.ascontiguousarray(piv, dtype=np.int32)
    h = C.c_void_p()
    _check(lib().tpdg_gpu_pc_import_record(op.h, _ptr(f), hs.ctypes.data_as(i64p), _ptr(r),
                                           pv.ctypes.data_as(ip), C.byref(h)))
    return KsvdPC(op, h)


def _gcfg(cfg):
    return _GmresCfg(cfg.tol, cfg.restart, cfg.max_iterations, 0 if cfg.side == "right" else 1)


def gmres(op: LinearizedOperator, pc: KsvdPC | None, b, cfg: GmresConfig | None = None, out=None) -> GmresResult:
    """Restarted GMRES (solve/gmres.hpp:52) with host arrays; raises GmresFailure on budget.
    out: optional preallocated (e.g. pinned) float64 host array for x."""
    cfg = cfg or GmresConfig()
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = out if out is not None else np.empty(op.n_local)
    if x.dtype != np.float64 or not x.flags["C_CONTIGUOUS"] or x.size != op.n_local:
        raise ShapeError("gmres: out must be a contiguous float64 array of the local size")
    its = C.c_int()
    conv = C.c_int()
    hist = np.zeros(cfg.max_iterations + 1)
    c = _gcfg(cfg)
    rc = lib().tpdg_gpu_gmres_host(op.h, pc.h if pc else None, _ptr(b), _ptr(x), C.byref(c), C.byref(its),
                                   _ptr(hist), len(hist), C.byref(conv))
    res = GmresResult(x, its.value, list(hist[: min(its.value, len(hist))]), bool(conv.value))
    if rc == 4:
        raise GmresFailure(lib().tpdg_gpu_last_error().decode(), res)
    _check(rc)
    return res


def gmres_device(op: LinearizedOperator, pc: KsvdPC | None, d_b, d_x, cfg: GmresConfig | None = None,
                 hist_cap=0):
    """Device-pointer GMRES (no host copies of b / x). Returns (iterations, converged, history)."""
    cfg = cfg or GmresConfig()
    its = C.c_int()
    conv = C.c_int()
    hist = np.zeros(max(hist_cap, 1))
    c = _gcfg(cfg)
    rc = lib().tpdg_gpu_gmres(op.h, pc.h if pc else None, _dptr(d_b), _dptr(d_x), C.byref(c), C.byref(its),
                              _ptr(hist), hist_cap, C.byref(conv))
    if rc not in (0, 4):
        _check(rc)
    return its.value, bool(conv.value), hist[: min(its.value, hist_cap)]
