"""Python binding of the sm_100a direct inverse NFFT library (libinft.so).

Argument marshalling only: every step of the method runs in the CUDA kernels
behind the C ABI declared in include/inft.h.  There is no CPU fallback -- if
the shared library is missing this module raises on import.

Low-level functions carry the C names (inft_plan, inft_precompute, inft_apply,
inft_adjoint_apply, inft_destroy, inft_get_bins, inft_get_bopt, inft_set_bopt,
inft_get_deconv, inft_get_info) and take raw pointers; ``Plan`` wraps them for
torch tensors (CUDA or CPU/pinned) and numpy arrays.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("INFT_LIB") or os.path.join(_HERE, "libinft.so")  # INFT_LIB: A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python build_native.py` "
                      "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

# enums (include/inft.h)
INFT_OK = 0
STATUS = {0: "INFT_OK", 1: "INFT_ERR_INVALID_ARG", 2: "INFT_ERR_NODE_RANGE", 3: "INFT_ERR_ZERO_WINDOW_HAT",
          4: "INFT_ERR_NOT_PRECOMPUTED", 5: "INFT_ERR_CUDA", 6: "INFT_ERR_CUFFT", 7: "INFT_ERR_OOM",
          8: "INFT_ERR_UNSUPPORTED"}
INFT_KAISER_BESSEL, INFT_DIRICHLET, INFT_BSPLINE = 0, 1, 2
INFT_AUTO, INFT_ALG1_NODEWISE, INFT_ALG2_GRIDWISE, INFT_PLAIN_NFFT = 0, 1, 2, 3
INFT_C128, INFT_C64 = 0, 1
INFT_WEIGHTS_REAL, INFT_WEIGHTS_COMPLEX = 0, 1
METHODS = {"auto": 0, "alg1": 1, "alg2": 2, "plain": 3}


class InftInfo(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("M", ctypes.c_int64 * 2), ("Msigma", ctypes.c_int64 * 2),
                ("N", ctypes.c_int64), ("m", ctypes.c_int32), ("P", ctypes.c_int32), ("tile", ctypes.c_int32 * 2),
                ("precision", ctypes.c_int32), ("method", ctypes.c_int32), ("weights", ctypes.c_int32),
                ("scale", ctypes.c_double), ("tau", ctypes.c_double), ("n_rank_deficient", ctypes.c_int64),
                ("n_empty_cols", ctypes.c_int64), ("max_col_size", ctypes.c_int64), ("max_abs_w", ctypes.c_double),
                ("perm_identity", ctypes.c_int32), ("fast_path", ctypes.c_int32), ("fused_fft", ctypes.c_int32),
                ("max_lowrank_rank", ctypes.c_int32), ("workspace_bytes", ctypes.c_size_t)]


class InftProfile(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 6), ("count", ctypes.c_int64 * 6)]


STAGES = ("spread", "fft_forward", "trunc_deconv", "deconv_pad", "fft_inverse", "gather")

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int

EXPORTS = {
    "inft_plan": ([ctypes.POINTER(_P), _I, ctypes.POINTER(_I64), _I64, _P, ctypes.c_double, _I, _I, _I, _I, _P], _I),
    "inft_precompute": ([_P, _I, _I, ctypes.c_double, _P], _I),
    "inft_apply": ([_P, _P, _P, _I64, _P], _I),
    "inft_adjoint_apply": ([_P, _P, _P, _I64, _P], _I),
    "inft_destroy": ([_P], _I),
    "inft_get_bins": ([_P, _P, _P, _P], _I),
    "inft_get_bopt": ([_P, _P], _I),
    "inft_set_bopt": ([_P, _I, _I, _P], _I),
    "inft_get_deconv": ([_P, _P], _I),
    "inft_get_info": ([_P, ctypes.POINTER(InftInfo)], _I),
    "inft_set_profiling": ([_P, _I], _I),
    "inft_get_profile": ([_P, ctypes.POINTER(InftProfile), _I], _I),
    "inft_kernel_launches": ([_P], _I64),
    "inft_quad_plan": ([ctypes.POINTER(_P), _I64, _P, ctypes.c_double, _I, _P], _I),
    "inft_quad_apply": ([_P, _P, _P, _I64, _P], _I),
    "inft_quad_adjoint_apply": ([_P, _P, _P, _I64, _P], _I),
    "inft_quad_get_coeffs": ([_P, _P, _P, _P, _P], _I),
    "inft_quad_kernel_launches": ([_P, ctypes.POINTER(_I64)], _I),
    "inft_quad_destroy": ([_P], _I),
    "inft_status_string": ([_I], ctypes.c_char_p),
    "inft_last_error": ([], ctypes.c_char_p),
}
for _name, (_args, _res) in EXPORTS.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res
    globals()[_name] = _fn


class InftError(RuntimeError):
    def __init__(self, status, where):
        msg = _lib.inft_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(status, status)} {msg}")
        self.status = status


def _check(st, where):
    if st != INFT_OK:
        raise InftError(st, where)


def _ptr(a):
    """Raw data pointer of a torch tensor or numpy array (must be contiguous)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    raise TypeError(f"unsupported buffer type {type(a)}")


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


def _check_nodes_shape(nd, d):
    """Nodes are float64 [N] (1-D) or [N][2] (2-D); the C side reads N*d doubles."""
    ok = (nd.ndim == 1) if d == 1 else (nd.ndim == 2 and nd.shape[1] == d)
    if d == 1 and nd.ndim == 2 and nd.shape[1] == 1:
        ok = True
    if not ok:
        raise ValueError(f"nodes: shape {tuple(nd.shape)}, expected [N]" + ("" if d == 1 else f"[{d}]"))


class Plan:
    """A plan for fixed nodes: nodes [N] or [N][2] float64 in [-1/2, 1/2)."""

    def __init__(self, nodes, M, sigma, m, precision="c128", device=0, stream=None, window="kb"):
        if isinstance(M, int):
            M = (M,)
        self.d = len(M)
        self.M = tuple(int(v) for v in M)
        if hasattr(nodes, "data_ptr"):
            import torch
            nd = nodes.to(torch.float64).contiguous()
            self._nodes_ref = nd
        else:
            nd = np.ascontiguousarray(np.asarray(nodes, dtype=np.float64))
            self._nodes_ref = nd
        _check_nodes_shape(nd, self.d)
        N = nd.shape[0]
        nptr = (nd.data_ptr() if hasattr(nd, "data_ptr") else nd.ctypes.data) if N > 0 else None
        self.N = int(N)
        self.prec = INFT_C128 if precision in ("c128", INFT_C128) else INFT_C64
        Marr = (ctypes.c_int64 * self.d)(*self.M)
        h = ctypes.c_void_p()
        win = {"kb": INFT_KAISER_BESSEL, "dirichlet": INFT_DIRICHLET, "bspline": INFT_BSPLINE}[window] if isinstance(window, str) \
            else int(window)
        _check(inft_plan(ctypes.byref(h), self.d, Marr, self.N, nptr, float(sigma), int(m), win,
                         self.prec, int(device), _stream_ptr(stream)), "inft_plan")
        self.window = window
        self._h = h
        self.sigma = float(sigma)
        self.m = int(m)
        self.device = int(device)
        self.Mtot = int(np.prod(self.M))
        self.P = (2 * self.m + 1) ** self.d

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            inft_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # setup
    def precompute(self, method="auto", weights="real", tau=0.0, stream=None):
        meth = METHODS[method] if isinstance(method, str) else int(method)
        wt = INFT_WEIGHTS_COMPLEX if weights == "complex" else INFT_WEIGHTS_REAL
        _check(inft_precompute(self._h, meth, wt, float(tau), _stream_ptr(stream)), "inft_precompute")
        return self

    def set_bopt(self, w, method="alg2"):
        w = np.ascontiguousarray(w)
        meth = METHODS[method] if isinstance(method, str) else int(method)
        if np.iscomplexobj(w):
            buf = np.ascontiguousarray(w.astype(np.complex128))
            wt = INFT_WEIGHTS_COMPLEX
        else:
            buf = np.ascontiguousarray(w.astype(np.float64))
            wt = INFT_WEIGHTS_REAL
        if buf.shape != (self.N, self.P):
            raise ValueError(f"B_opt weights must be [{self.N}][{self.P}]")
        _check(inft_set_bopt(self._h, meth, wt, buf.ctypes.data if buf.size else None), "inft_set_bopt")
        return self

    def get_bopt(self):
        info = self.info()
        dt = np.complex128 if info["weights"] == INFT_WEIGHTS_COMPLEX else np.float64
        out = np.zeros((self.N, self.P), dtype=dt)
        _check(inft_get_bopt(self._h, out.ctypes.data), "inft_get_bopt")
        return out

    def get_bins(self):
        l0 = np.zeros((self.N, self.d), dtype=np.int32)
        b = np.zeros(self.N, dtype=np.int32)
        perm = np.zeros(self.N, dtype=np.int32)
        if self.N:
            _check(inft_get_bins(self._h, l0.ctypes.data, b.ctypes.data, perm.ctypes.data), "inft_get_bins")
        return (l0[:, 0] if self.d == 1 else l0), b, perm

    def get_deconv(self):
        out = np.zeros(sum(self.M), dtype=np.float64)
        _check(inft_get_deconv(self._h, out.ctypes.data), "inft_get_deconv")
        return out

    def info(self):
        inf = InftInfo()
        _check(inft_get_info(self._h, ctypes.byref(inf)), "inft_get_info")
        return {k: (list(getattr(inf, k)) if k in ("M", "Msigma", "tile") else getattr(inf, k))
                for k, _ in InftInfo._fields_}

    def set_profiling(self, enable=True):
        _check(inft_set_profiling(self._h, 1 if enable else 0), "inft_set_profiling")

    def get_profile(self, reset=False):
        """{stage: (total ms, launches)} from CUDA events on the launching stream."""
        pr = InftProfile()
        _check(inft_get_profile(self._h, ctypes.byref(pr), 1 if reset else 0), "inft_get_profile")
        return {s: (pr.ms[i], pr.count[i]) for i, s in enumerate(STAGES)}

    def kernel_launches(self):
        return int(inft_kernel_launches(self._h))

    # apply
    def _out(self, like, shape):
        import torch
        dt = torch.complex128 if self.prec == INFT_C128 else torch.complex64
        if hasattr(like, "device"):
            return torch.empty(shape, dtype=dt, device=like.device, pin_memory=False)
        return np.empty(shape, dtype=np.complex128 if self.prec == INFT_C128 else np.complex64)

    def _dtype_ok(self, a):
        want = "complex128" if self.prec == INFT_C128 else "complex64"
        return str(a.dtype).replace("torch.", "") == want

    def _check_buf(self, a, width, what, R=None):
        """dtype = the plan's precision, trailing size = width, [R][width] or [width], and
        CUDA tensors on the plan's device: the C side trusts these sizes."""
        if not self._dtype_ok(a):
            raise TypeError(f"{what}: dtype {a.dtype} does not match the plan's precision "
                            f"({'complex128' if self.prec == INFT_C128 else 'complex64'})")
        if a.ndim not in (1, 2) or a.shape[-1] != width:
            raise ValueError(f"{what}: shape {tuple(a.shape)}, expected [R][{width}]")
        if R is not None and (a.shape[0] if a.ndim == 2 else 1) != R:
            raise ValueError(f"{what}: {a.shape[0] if a.ndim == 2 else 1} rows, expected {R}")
        dev = getattr(a, "device", None)
        if getattr(dev, "type", None) == "cuda" and dev.index != self.device:
            raise ValueError(f"{what}: tensor on {dev}, the plan on cuda:{self.device}")

    def apply(self, f, out=None, stream=None):
        """Inverse NFFT (problem (1)): fhat = s D^* F^* B_opt^* f; f [R][N] -> [R][prod M]."""
        self._check_buf(f, self.N, "apply input f")
        R = f.shape[0] if f.ndim == 2 else 1
        if out is None:
            out = self._out(f, (R, self.Mtot))
        self._check_buf(out, self.Mtot, "apply output fhat", R)
        _check(inft_apply(self._h, _ptr(f), _ptr(out), R, _stream_ptr(stream)), "inft_apply")
        return out

    def adjoint_apply(self, h, out=None, stream=None):
        """Inverse adjoint NFFT (problem (2)): f = s B_opt F D h; h [R][prod M] -> [R][N]."""
        self._check_buf(h, self.Mtot, "adjoint_apply input h")
        R = h.shape[0] if h.ndim == 2 else 1
        if out is None:
            out = self._out(h, (R, self.N))
        self._check_buf(out, self.N, "adjoint_apply output f", R)
        _check(inft_adjoint_apply(self._h, _ptr(h), _ptr(out), R, _stream_ptr(stream)), "inft_adjoint_apply")
        return out


class QuadPlan:
    """Quadratic case M = N (inft_quad_*): nodes [N] float64 in
    [-1/2, 1/2), N even; targets x_l = -1/2 + l/N + delta (delta = 0: 1/(2N)).  Complex128."""

    def __init__(self, nodes, delta=0.0, device=0, stream=None):
        if hasattr(nodes, "data_ptr"):
            import torch
            nd = nodes.to(torch.float64).contiguous()
            N, nptr = nd.shape[0], nd.data_ptr()
        else:
            nd = np.ascontiguousarray(np.asarray(nodes, dtype=np.float64))
            N, nptr = nd.shape[0], nd.ctypes.data
        _check_nodes_shape(nd, 1)
        self._nodes_ref = nd
        self.N = int(N)
        self.device = int(device)
        h = ctypes.c_void_p()
        _check(inft_quad_plan(ctypes.byref(h), self.N, nptr, float(delta), self.device, _stream_ptr(stream)),
               "inft_quad_plan")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            inft_quad_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def coeffs(self):
        """(x, a, b, s): targets, signed stabilised a_l and b_j, shift s (host copies)."""
        x, a, b = (np.empty(self.N) for _ in range(3))
        s = ctypes.c_double()
        _check(inft_quad_get_coeffs(self._h, x.ctypes.data, a.ctypes.data, b.ctypes.data, ctypes.byref(s)),
               "inft_quad_get_coeffs")
        return x, a, b, s.value

    def kernel_launches(self):
        c = ctypes.c_int64()
        _check(inft_quad_kernel_launches(self._h, ctypes.byref(c)), "inft_quad_kernel_launches")
        return int(c.value)

    def _out(self, like, shape):
        if hasattr(like, "device"):
            import torch
            return torch.empty(shape, dtype=torch.complex128, device=like.device)
        return np.empty(shape, dtype=np.complex128)

    def _check_buf(self, a, what, R=None):
        if str(a.dtype).replace("torch.", "") != "complex128":
            raise TypeError(f"{what}: dtype {a.dtype}, the quadratic case is complex128")
        if a.ndim not in (1, 2) or a.shape[-1] != self.N:
            raise ValueError(f"{what}: shape {tuple(a.shape)}, expected [R][{self.N}]")
        if R is not None and (a.shape[0] if a.ndim == 2 else 1) != R:
            raise ValueError(f"{what}: row count does not match the input")
        dev = getattr(a, "device", None)
        if getattr(dev, "type", None) == "cuda" and dev.index != self.device:
            raise ValueError(f"{what}: tensor on {dev}, the plan on cuda:{self.device}")

    def apply(self, f, out=None, stream=None):
        """Inverse NFFT, quadratic case: f [R][N] -> fhat [R][N] (k = -N/2..N/2-1)."""
        self._check_buf(f, "quad apply input")
        R = f.shape[0] if f.ndim == 2 else 1
        if out is None:
            out = self._out(f, (R, self.N))
        self._check_buf(out, "quad apply output", R)
        _check(inft_quad_apply(self._h, _ptr(f), _ptr(out), R, _stream_ptr(stream)), "inft_quad_apply")
        return out

    def adjoint_apply(self, h, out=None, stream=None):
        """Inverse adjoint NFFT, quadratic case: h [R][N] -> f [R][N]."""
        self._check_buf(h, "quad adjoint input")
        R = h.shape[0] if h.ndim == 2 else 1
        if out is None:
            out = self._out(h, (R, self.N))
        self._check_buf(out, "quad adjoint output", R)
        _check(inft_quad_adjoint_apply(self._h, _ptr(h), _ptr(out), R, _stream_ptr(stream)),
               "inft_quad_adjoint_apply")
        return out


__all__ = ["Plan", "QuadPlan", "InftError", "LIB_PATH", "EXPORTS", "STAGES"] + list(EXPORTS)
