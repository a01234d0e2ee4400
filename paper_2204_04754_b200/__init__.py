"""Python binding of libsrmra.so — B200-native projected EM for 2-D SR-MRA (arXiv 2204.04754).

Argument marshalling only: every step of the EM iteration runs in the CUDA kernels of
libsrmra.so (csrc/), behind the C ABI declared in include/srmra.h.  The module-level functions
carry the ABI's names; `Context` is a thin owner of one srmra_ctx.  There is no CPU fallback:
importing this package without the built library raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SRMRA_LIB: an alternative in-tree build of the same library (A/B timing of kernel variants, tools/)
LIB_PATH = os.environ.get("SRMRA_LIB") or os.path.join(_HERE, "libsrmra.so")

SRMRA_OK = 0
SRMRA_ERR_INVALID_ARG = -1
SRMRA_ERR_UNSUPPORTED = -2
SRMRA_ERR_CUDA = -3
SRMRA_ERR_NCCL = -4
SRMRA_ERR_OOM = -5
SRMRA_ERR_STATE = -6
SRMRA_ERR_NUMERIC = -7

PATH_AUTO, PATH_GEMM, PATH_FFT, PATH_DIRECT = 0, 1, 2, 3
PATH_NAMES = {PATH_AUTO: "auto", PATH_GEMM: "gemm", PATH_FFT: "fft", PATH_DIRECT: "direct"}
PATH_IDS = {v: k for k, v in PATH_NAMES.items()}

# every symbol include/srmra.h declares (checked by tests/test_abi.py)
ABI_SYMBOLS = ("srmra_default_options", "srmra_init", "srmra_load", "srmra_load_iterate", "srmra_em_iter", "srmra_get_estimate",
               "srmra_get_loglik_trace", "srmra_get_stats", "srmra_get_obs_loglik", "srmra_local_stats",
               "srmra_get_path", "srmra_launches_per_iter", "srmra_profile", "srmra_profile_read", "srmra_debug_timestamps",
               "srmra_nccl_unique_id", "srmra_free",
               "srmra_last_error", "srmra_run", "srmra_set_denoiser", "srmra_relative_error",
               "srmra_set_joint_rho", "srmra_get_joint_rho", "srmra_moments",
               "srmra_mom_set_moments", "srmra_mom_objective", "srmra_mom_run", "srmra_generate", "srmra_get_observations")


class SrmraError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libsrmra error {code}: {msg}")
        self.code = code


# int (*)(double* buf_dev, uint64_t n, void* stream, void* user): exchange provider (srmra_options.allreduce)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p)


class srmra_options(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int32), ("proj_every", ctypes.c_int32), ("floor_tau", ctypes.c_double),
                ("device", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("nccl_id", ctypes.c_void_p), ("stream", ctypes.c_void_p), ("trace_cap", ctypes.c_int32),
                ("allreduce", ALLREDUCE_FN), ("allreduce_user", ctypes.c_void_p), ("grid_cap", ctypes.c_int32),
                ("nccl_timeout_ms", ctypes.c_int32)]


# int (*)(double* x_dev, int32_t L_high, double sigma_t, void* stream, void* user)
DENOISER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p,
                               ctypes.c_void_p)

_fp = ctypes.POINTER(ctypes.c_float)
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int32)
_ctxp = ctypes.c_void_p


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    sig = {
        "srmra_default_options": (None, [ctypes.POINTER(srmra_options)]),
        "srmra_init": (ctypes.c_int, [ctypes.POINTER(_ctxp), _fp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_int32, ctypes.c_double, _fp, _dp, _dp, ctypes.POINTER(srmra_options)]),
        "srmra_load": (ctypes.c_int, [_ctxp, _fp, _fp, _dp, _dp]),
        "srmra_load_iterate": (ctypes.c_int, [_ctxp, _fp, _fp, _dp, _dp, ctypes.c_int32]),
        "srmra_em_iter": (ctypes.c_int, [_ctxp, ctypes.c_int32]),
        "srmra_get_estimate": (ctypes.c_int, [_ctxp, _fp, _dp, _dp, _dp, _ip]),
        "srmra_get_loglik_trace": (ctypes.c_int, [_ctxp, _dp, ctypes.c_int32, _ip]),
        "srmra_get_stats": (ctypes.c_int, [_ctxp, _dp, _dp, _dp, _dp]),
        "srmra_get_obs_loglik": (ctypes.c_int, [_ctxp, _dp]),
        "srmra_local_stats": (ctypes.c_int, [_ctxp, _dp]),
        "srmra_get_path": (ctypes.c_int, [_ctxp]),
        "srmra_launches_per_iter": (ctypes.c_int, [_ctxp]),
        "srmra_profile": (ctypes.c_int, [_ctxp, ctypes.c_int32]),
        "srmra_profile_read": (ctypes.c_int, [_ctxp, _dp, _dp, _ip]),
        "srmra_debug_timestamps": (ctypes.c_int, [_ctxp, ctypes.POINTER(ctypes.c_uint64)]),
        "srmra_nccl_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
        "srmra_free": (None, [_ctxp]),
        "srmra_last_error": (ctypes.c_char_p, [_ctxp]),
        "srmra_run": (ctypes.c_int, [_ctxp, ctypes.c_int32, ctypes.c_double]),
        "srmra_set_denoiser": (ctypes.c_int, [_ctxp, DENOISER_FN, ctypes.c_void_p]),
        "srmra_relative_error": (ctypes.c_int, [_ctxp, _fp, _dp, _ip, _ip]),
        "srmra_set_joint_rho": (ctypes.c_int, [_ctxp, _dp]),
        "srmra_get_joint_rho": (ctypes.c_int, [_ctxp, _dp]),
        "srmra_moments": (ctypes.c_int, [_ctxp, _dp, _dp]),
        "srmra_get_observations": (ctypes.c_int, [_ctxp, ctypes.c_int64, ctypes.c_int64, _fp]),
        "srmra_generate": (ctypes.c_int, [_ctxp, _fp, _dp, _dp, ctypes.c_uint64, ctypes.c_int64, _fp, _dp, _dp, _ip]),
        "srmra_mom_set_moments": (ctypes.c_int, [_ctxp, _dp, _dp]),
        "srmra_mom_objective": (ctypes.c_int, [_ctxp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]),
        "srmra_mom_run": (ctypes.c_int, [_ctxp, ctypes.c_int32, ctypes.c_int32, ctypes.c_double, _dp, _ip]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _check(rc: int, ctx=None):
    if rc != SRMRA_OK:
        msg = _lib.srmra_last_error(ctx)
        raise SrmraError(rc, msg.decode() if msg else "")
    return rc


# ------------------------------------------------------------------ ABI-named functions
def srmra_default_options() -> srmra_options:
    o = srmra_options()
    _lib.srmra_default_options(ctypes.byref(o))
    return o


def srmra_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.srmra_nccl_unique_id(buf))
    return buf.raw


def srmra_init(y, L_high, L_low, K, sigma, x0, rho1_0, rho2_0, opt: srmra_options | None = None,
               n_local: int | None = None):
    """Returns the opaque context handle (int).  y: float32 [n][L_low][L_low] host array, or None with
    n_local given (observations to come from srmra_generate / srmra_load)."""
    if y is None:
        if n_local is None:
            raise ValueError("y is None: pass n_local")
        yp, n = None, int(n_local)
    else:
        y = np.ascontiguousarray(y, dtype=np.float32)
        yp, n = _ptr(y, _fp), int(y.shape[0])
    x0 = np.ascontiguousarray(x0, dtype=np.float32)
    r1 = np.ascontiguousarray(rho1_0, dtype=np.float64)
    r2 = np.ascontiguousarray(rho2_0, dtype=np.float64)
    h = _ctxp()
    rc = _lib.srmra_init(ctypes.byref(h), yp, n, int(L_high), int(L_low), int(K),
                         float(sigma), _ptr(x0, _fp), _ptr(r1, _dp), _ptr(r2, _dp),
                         ctypes.byref(opt) if opt is not None else None)
    _check(rc, None)
    return h.value


def srmra_load(ctx, y, x0, rho1_0, rho2_0):
    y = np.ascontiguousarray(y, dtype=np.float32)
    _check(_lib.srmra_load(ctx, _ptr(y, _fp), _ptr(np.ascontiguousarray(x0, dtype=np.float32), _fp),
                           _ptr(np.ascontiguousarray(rho1_0, dtype=np.float64), _dp),
                           _ptr(np.ascontiguousarray(rho2_0, dtype=np.float64), _dp)), ctx)


def srmra_load_iterate(ctx, y, x0, rho1_0, rho2_0, n_iters: int):
    y = np.ascontiguousarray(y, dtype=np.float32)
    _check(_lib.srmra_load_iterate(ctx, _ptr(y, _fp), _ptr(np.ascontiguousarray(x0, dtype=np.float32), _fp),
                                   _ptr(np.ascontiguousarray(rho1_0, dtype=np.float64), _dp),
                                   _ptr(np.ascontiguousarray(rho2_0, dtype=np.float64), _dp), int(n_iters)), ctx)


def srmra_generate(ctx, x_true, rho1_true, rho2_true, seed: int, first_index: int, x0, rho1_0, rho2_0,
                   n_local: int, want_shifts: bool = False):
    """Device-generated observations (NEXT-4; synth/philox.py is the reference) + theta_0, like srmra_load.
    Returns the shifts (int32 [n_local][2]) if want_shifts."""
    xt = np.ascontiguousarray(x_true, dtype=np.float32)
    t1 = np.ascontiguousarray(rho1_true, dtype=np.float64)
    t2 = np.ascontiguousarray(rho2_true, dtype=np.float64)
    x0 = np.ascontiguousarray(x0, dtype=np.float32)
    r1 = np.ascontiguousarray(rho1_0, dtype=np.float64)
    r2 = np.ascontiguousarray(rho2_0, dtype=np.float64)
    sh = np.empty((n_local, 2), dtype=np.int32) if want_shifts else None
    _check(_lib.srmra_generate(ctx, _ptr(xt, _fp), _ptr(t1, _dp), _ptr(t2, _dp), ctypes.c_uint64(int(seed) & (2 ** 64 - 1)),
                               int(first_index), _ptr(x0, _fp), _ptr(r1, _dp), _ptr(r2, _dp),
                               _ptr(sh, _ip) if sh is not None else None), ctx)
    return sh


def srmra_get_observations(ctx, first: int, count: int, L_low: int):
    out = np.empty((count, L_low, L_low), dtype=np.float32)
    _check(_lib.srmra_get_observations(ctx, int(first), int(count), _ptr(out, _fp)), ctx)
    return out


def srmra_em_iter(ctx, n_iters: int = 1):
    _check(_lib.srmra_em_iter(ctx, int(n_iters)), ctx)


def srmra_run(ctx, max_iters: int, rel_tol: float = 0.0):
    _check(_lib.srmra_run(ctx, int(max_iters), float(rel_tol)), ctx)


def srmra_set_denoiser(ctx, fn):
    """fn: a DENOISER_FN (keep a reference while it is installed) or None for the built-in stand-in."""
    _check(_lib.srmra_set_denoiser(ctx, fn if fn is not None else DENOISER_FN(), None), ctx)


def srmra_relative_error(ctx, x_true):
    """(error, (s1, s2)): min_s ||R_s x_hat - x_true||_F / ||x_true||_F and its shift."""
    xt = np.ascontiguousarray(x_true, dtype=np.float32)
    err = ctypes.c_double()
    s1 = ctypes.c_int32()
    s2 = ctypes.c_int32()
    _check(_lib.srmra_relative_error(ctx, _ptr(xt, _fp), ctypes.byref(err), ctypes.byref(s1), ctypes.byref(s2)), ctx)
    return err.value, (s1.value, s2.value)


def srmra_set_joint_rho(ctx, rho):
    r = np.ascontiguousarray(rho, dtype=np.float64)
    _check(_lib.srmra_set_joint_rho(ctx, _ptr(r, _dp)), ctx)


def srmra_get_joint_rho(ctx, L_high: int):
    out = np.empty((L_high, L_high))
    _check(_lib.srmra_get_joint_rho(ctx, _ptr(out, _dp)), ctx)
    return out


def srmra_moments(ctx, L_low: int):
    """(M1 [L_low^2], M2 [L_low^2, L_low^2]): the empirical moments of eq:empiric_MOM."""
    d = L_low * L_low
    m1 = np.empty(d)
    m2 = np.empty((d, d))
    _check(_lib.srmra_moments(ctx, _ptr(m1, _dp), _ptr(m2, _dp)), ctx)
    return m1, m2


def srmra_mom_set_moments(ctx, m1=None, m2=None):
    """Data term of eq:LS_SR: the loaded observations' empirical moments (None, None) or given ones."""
    if (m1 is None) != (m2 is None):
        raise ValueError("m1 and m2: both or neither")
    if m1 is None:
        _check(_lib.srmra_mom_set_moments(ctx, None, None), ctx)
    else:
        a = np.ascontiguousarray(m1, dtype=np.float64)
        b = np.ascontiguousarray(m2, dtype=np.float64)
        _check(_lib.srmra_mom_set_moments(ctx, _ptr(a, _dp), _ptr(b, _dp)), ctx)


def srmra_mom_objective(ctx, x, rho1, rho2):
    """(f, grad_x, grad_rho1, grad_rho2) of eq:LS_SR."""
    xx = np.ascontiguousarray(x, dtype=np.float64)
    r1 = np.ascontiguousarray(rho1, dtype=np.float64)
    r2 = np.ascontiguousarray(rho2, dtype=np.float64)
    L = r1.shape[0]
    f = ctypes.c_double()
    gx = np.empty((L, L))
    g1 = np.empty(L)
    g2 = np.empty(L)
    _check(_lib.srmra_mom_objective(ctx, _ptr(xx, _dp), _ptr(r1, _dp), _ptr(r2, _dp), ctypes.byref(f),
                                    _ptr(gx, _dp), _ptr(g1, _dp), _ptr(g2, _dp)), ctx)
    return f.value, gx, g1, g2


def srmra_mom_run(ctx, max_steps: int, F: int = 5, gtol: float = 0.0):
    """Algorithm 1 from the context's estimate: (final objective, steps taken)."""
    f = ctypes.c_double()
    st = ctypes.c_int32()
    _check(_lib.srmra_mom_run(ctx, int(max_steps), int(F), float(gtol), ctypes.byref(f), ctypes.byref(st)), ctx)
    return f.value, st.value


def snr(x_true, sigma: float) -> float:
    """SNR = ||x||_F^2 / (L_high^2 sigma^2); a definition, evaluated on the host."""
    x = np.asarray(x_true, dtype=np.float64)
    return float((x * x).sum() / (x.shape[0] * x.shape[1] * sigma * sigma))


def srmra_get_estimate(ctx, L_high: int):
    x = np.empty((L_high, L_high), np.float32)
    r1 = np.empty(L_high)
    r2 = np.empty(L_high)
    ll = ctypes.c_double()
    it = ctypes.c_int32()
    _check(_lib.srmra_get_estimate(ctx, _ptr(x, _fp), _ptr(r1, _dp), _ptr(r2, _dp), ctypes.byref(ll),
                                   ctypes.byref(it)), ctx)
    return x, r1, r2, ll.value, it.value


def srmra_get_loglik_trace(ctx, cap: int = 4096):
    out = np.empty(cap)
    n = ctypes.c_int32()
    _check(_lib.srmra_get_loglik_trace(ctx, _ptr(out, _dp), cap, ctypes.byref(n)), ctx)
    return out[:min(n.value, cap)].copy()


def srmra_get_stats(ctx, L_high: int, K: int):
    b = np.empty((L_high, L_high)); cm = np.empty((K, K)); m1 = np.empty(L_high); m2 = np.empty(L_high)
    _check(_lib.srmra_get_stats(ctx, _ptr(b, _dp), _ptr(cm, _dp), _ptr(m1, _dp), _ptr(m2, _dp)), ctx)
    return b, cm, m1, m2


def srmra_get_obs_loglik(ctx, n_local: int):
    out = np.empty(n_local)
    _check(_lib.srmra_get_obs_loglik(ctx, _ptr(out, _dp)), ctx)
    return out


def srmra_local_stats(ctx, L_high: int, K: int):
    out = np.empty(L_high * L_high + K * K + 2 * L_high + 1)
    _check(_lib.srmra_local_stats(ctx, _ptr(out, _dp)), ctx)
    return out


def srmra_get_path(ctx) -> int:
    return int(_lib.srmra_get_path(ctx))


def srmra_launches_per_iter(ctx) -> int:
    return int(_lib.srmra_launches_per_iter(ctx))


def srmra_profile(ctx, enable: bool = True):
    _check(_lib.srmra_profile(ctx, int(bool(enable))), ctx)


def srmra_profile_read(ctx):
    """(summed E/M-kernel ms, summed iteration ms, iterations) since srmra_profile(ctx, True)."""
    em = ctypes.c_double()
    it = ctypes.c_double()
    n = ctypes.c_int32()
    _check(_lib.srmra_profile_read(ctx, ctypes.byref(em), ctypes.byref(it), ctypes.byref(n)), ctx)
    return em.value, it.value, n.value


def srmra_debug_timestamps(ctx):
    out = np.zeros(8, dtype=np.uint64)
    _check(_lib.srmra_debug_timestamps(ctx, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))), ctx)
    return out


def srmra_free(ctx):
    _lib.srmra_free(ctx)


def srmra_last_error(ctx=None) -> str:
    m = _lib.srmra_last_error(ctx)
    return m.decode() if m else ""


# ------------------------------------------------------------------ thin owner
class Context:
    """Owns one srmra_ctx for this rank's shard.  Methods map 1:1 onto the ABI."""

    def __init__(self, y, L_high, L_low, K, sigma, x0, rho1_0, rho2_0, path="auto", proj_every=1,
                 floor_tau=-1.0, device=-1, rank=0, world=1, nccl_id: bytes | None = None, stream=None,
                 trace_cap=4096, n_local: int | None = None, allreduce=None, grid_cap=0, nccl_timeout_ms=0):
        """y None: n_local observations to come from generate() / load().  allreduce: exchange provider
        fn(buf_dev_ptr: int, n: int, stream: int) -> int (0 = ok) used instead of NCCL for world > 1
        (include/srmra.h, srmra_allreduce_fn)."""
        o = srmra_default_options()
        o.path = PATH_IDS[path] if isinstance(path, str) else int(path)
        o.proj_every = int(proj_every)
        o.floor_tau = float(floor_tau)
        o.device = int(device)
        o.rank, o.world = int(rank), int(world)
        self._id_buf = None
        if nccl_id is not None:
            self._id_buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_id = ctypes.cast(self._id_buf, ctypes.c_void_p)
        o.stream = stream
        o.trace_cap = int(trace_cap)
        o.grid_cap = int(grid_cap)
        o.nccl_timeout_ms = int(nccl_timeout_ms)
        self._allreduce = None
        if allreduce is not None:
            self._allreduce = ALLREDUCE_FN(lambda buf, n, st, user: int(allreduce(buf, n, st)))
            o.allreduce = self._allreduce
        self.L_high, self.L_low, self.K = int(L_high), int(L_low), int(K)
        self.n_local = int(np.asarray(y).shape[0]) if y is not None else int(n_local)
        self.handle = srmra_init(y, L_high, L_low, K, sigma, x0, rho1_0, rho2_0, o, n_local=self.n_local)

    @property
    def path(self) -> str:
        return PATH_NAMES[srmra_get_path(self.handle)]

    def generate(self, x_true, rho1_true, rho2_true, seed, x0, rho1_0, rho2_0, first_index=0, want_shifts=False):
        """Observations drawn on the device (counter-based; synth/philox.py is the reference) + theta_0."""
        return srmra_generate(self.handle, x_true, rho1_true, rho2_true, seed, first_index, x0, rho1_0, rho2_0,
                              self.n_local, want_shifts)

    def observations(self, first=0, count=None):
        count = self.n_local - first if count is None else count
        return srmra_get_observations(self.handle, first, count, self.L_low)

    def load(self, y, x0, rho1_0, rho2_0):
        """Replace the observations (same n_local as at init: srmra_load takes no size) and theta."""
        if np.asarray(y).size != self.n_local * self.L_low * self.L_low:
            raise ValueError(f"srmra_load: y must hold n_local = {self.n_local} observations of "
                             f"{self.L_low} x {self.L_low}")
        srmra_load(self.handle, y, x0, rho1_0, rho2_0)

    def load_iterate(self, y, x0, rho1_0, rho2_0, n_iters=1):
        """load + n_iters iterations, the first one overlapped with the upload (srmra_load_iterate)."""
        if np.asarray(y).size != self.n_local * self.L_low * self.L_low:
            raise ValueError(f"srmra_load_iterate: y must hold n_local = {self.n_local} observations of "
                             f"{self.L_low} x {self.L_low}")
        srmra_load_iterate(self.handle, y, x0, rho1_0, rho2_0, n_iters)

    def em_iter(self, n_iters=1):
        srmra_em_iter(self.handle, n_iters)

    def run(self, max_iters, rel_tol=0.0):
        """Algorithm 2 to convergence (srmra_run)."""
        srmra_run(self.handle, max_iters, rel_tol)

    def set_denoiser(self, fn):
        """fn(x_dev_ptr: int, L_high: int, sigma_t: float, stream: int) -> int (0 = ok), or None."""
        if fn is None:
            self._denoiser = None
            srmra_set_denoiser(self.handle, None)
            return
        self._denoiser = DENOISER_FN(lambda x, L, sig, st, user: int(fn(x, L, sig, st)))
        srmra_set_denoiser(self.handle, self._denoiser)

    def set_joint_rho(self, rho):
        srmra_set_joint_rho(self.handle, rho)

    def joint_rho(self):
        return srmra_get_joint_rho(self.handle, self.L_high)

    def relative_error(self, x_true):
        return srmra_relative_error(self.handle, x_true)

    def moments(self):
        return srmra_moments(self.handle, self.L_low)

    def mom_set_moments(self, m1=None, m2=None):
        srmra_mom_set_moments(self.handle, m1, m2)

    def mom_objective(self, x, rho1, rho2):
        return srmra_mom_objective(self.handle, x, rho1, rho2)

    def mom_run(self, max_steps, F=5, gtol=0.0):
        return srmra_mom_run(self.handle, max_steps, F, gtol)

    def get_estimate(self):
        return srmra_get_estimate(self.handle, self.L_high)

    def loglik_trace(self, cap=4096):
        return srmra_get_loglik_trace(self.handle, cap)

    def stats(self):
        return srmra_get_stats(self.handle, self.L_high, self.K)

    def obs_loglik(self):
        return srmra_get_obs_loglik(self.handle, self.n_local)

    def local_stats(self):
        return srmra_local_stats(self.handle, self.L_high, self.K)

    def profile(self, enable=True):
        srmra_profile(self.handle, enable)

    def profile_read(self):
        return srmra_profile_read(self.handle)

    def launches_per_iter(self):
        return srmra_launches_per_iter(self.handle)

    def close(self):
        if getattr(self, "handle", None):
            srmra_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
