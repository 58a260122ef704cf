"""Device side of the drop-in: ctypes binding of libkb_b200.so and the uploaded operator handle.

The shared library exports the C ABI declared in ``include/kronblur_b200.h``. Buffers are torch
CUDA tensors (plumbing only: allocation, streams, host<->device copies); every arithmetic step of
the hot path runs in the library's sm_100a kernels. There is no CPU fallback: if the library is
missing or no GPU is present, every entry point raises.
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import threading
import weakref

import numpy as np

from .errors import ArgumentError, NumericError
from .psf import bc_name
from .structured import factor_band, kind_name

_HERE = os.path.dirname(os.path.abspath(__file__))
# KB_LIB_PATH: load another build of the same library (compile-time variants in experiments)
LIB_PATH = os.environ.get("KB_LIB_PATH") or os.path.join(_HERE, "libkb_b200.so")

KB_OK, KB_ERR_ARGUMENT, KB_ERR_CUDA, KB_ERR_NUMERIC = 0, 2, 3, 4
KB_F64, KB_F32 = 0, 1
KB_PEAK_TC_TF32 = 2
# pass engines (kb_last_engines)
ENGINES = {0: "generic", 1: "ffma", 2: "dmma", 3: "mma_tf32", 4: "tcgen05_tf32", 5: "persist_f64", 6: "tcgen05_fused"}
KB_BC_ZERO, KB_BC_REFLECTIVE = 0, 1
KB_RESID_NORMS_WORK = 2 * 8 * 296  # include/kronblur_b200.h
INT_MAX = 2**31 - 1

# Band trimming threshold relative to max|c|: removes the ~1e-16 leakage that the reference's
# triangular back-solve leaves on reflective generators; exact zeros are always cut.
BAND_REL_TOL = 1e-14

_lib = None
_lib_lock = threading.Lock()

_c_int, _c_double, _vp = ctypes.c_int, ctypes.c_double, ctypes.c_void_p
_c_dp = ctypes.POINTER(ctypes.c_double)

EXPORTS = {
    "kb_version": (ctypes.c_char_p, []),
    "kb_last_error": (ctypes.c_char_p, []),
    "kb_max_half_width": (_c_int, []),
    "kb_op_create": (
        _c_int,
        [ctypes.POINTER(_vp), _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
         _c_int, _c_int, _c_dp, _c_int, _c_int, _c_dp],
    ),
    "kb_op_destroy": (_c_int, [_vp]),
    "kb_workspace_bytes": (ctypes.c_size_t, [_vp]),
    "kb_op_info": (_c_int, [_vp, ctypes.POINTER(_c_int), _c_int]),
    "kb_apply": (_c_int, [_vp, _vp, _vp, _vp, _vp]),
    "kb_apply_adjoint": (_c_int, [_vp, _vp, _vp, _vp, _vp]),
    "kb_sfista_run": (
        _c_int,
        [_vp, _vp, _vp, _vp, _vp, _c_dp, _c_int, _c_int, _c_dp, _c_double, _c_int, _vp, _vp,
         _c_int, _vp],
    ),
    "kb_sfista_run_lams": (
        _c_int,
        [_vp, _vp, _vp, _vp, _vp, _c_dp, _c_int, _c_int, _c_dp, _c_dp, _c_int, _vp, _vp,
         _c_int, _vp],
    ),
    "kb_power_iter": (_c_int, [_vp, _vp, _vp, _vp, _c_int, _vp, _vp]),
    "kb_apply_block": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp]),
    "kb_block_residual": (_c_int, [_vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp]),
    "kb_fma_peak": (_c_int, [_c_int, ctypes.POINTER(ctypes.c_float), _vp]),
    "kb_resid_norms": (_c_int, [_c_int, _vp, _vp, _vp, _vp, ctypes.c_longlong, _vp, _vp, _vp]),
    "kb_blur_direct": (
        _c_int,
        [_vp, ctypes.c_longlong, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _c_int,
         _c_int, _vp],
    ),
    "kb_debug_trace": (_c_int, [ctypes.POINTER(ctypes.c_ulonglong), _c_int]),
    "kb_last_engines": (_c_int, [_vp, ctypes.POINTER(ctypes.c_int)]),
    "kb_time_passes": (
        _c_int,
        [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_dp, _c_double, _vp,
         ctypes.POINTER(ctypes.c_float), _vp],
    ),
    "kb_block_update": (
        _c_int,
        [_vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_double, _c_int, _c_double,
         _c_double, _c_int, _vp, _vp, _vp],
    ),
    "kb_inner2": (_c_int, [_c_int, _vp, _vp, ctypes.c_longlong, _vp, _vp, _vp]),
}


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the C-ABI library (no CUDA call is made). Raises if it has not been built."""
    global _lib
    with _lib_lock:
        if _lib is not None and path == LIB_PATH:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: the CUDA extension has not been built "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`)"
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path == LIB_PATH:
            _lib = lib
        return lib


def _check(rc: int, what: str) -> None:
    if rc == KB_OK:
        return
    msg = load_library().kb_last_error().decode(errors="replace")
    if rc == KB_ERR_ARGUMENT:
        raise ArgumentError(f"{what}: {msg}")
    if rc == KB_ERR_NUMERIC:
        raise NumericError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: CUDA failure: {msg}")


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the B200 path needs a CUDA device; no CPU fallback exists")
    return torch


def torch_dtype(dtype: str):
    torch = _torch()
    if dtype in ("float64", "f64", "double"):
        return torch.float64
    if dtype in ("float32", "f32", "float"):
        return torch.float32
    raise ArgumentError(f"unsupported dtype {dtype!r} (float64 or float32)")


def _code(dtype: str) -> int:
    return KB_F64 if dtype in ("float64", "f64", "double") else KB_F32


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _stream_handle():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


_PIECE_BYTES = 4 << 20  # host <-> device transfers move in 4 MiB pieces (tools/copy_bench.py)
_copy_pool = None


def _pool():
    """Host-copy workers: numpy releases the GIL for large contiguous copies, so the pieces'
    host copies (and dtype conversions) run in parallel with each other and with the DMAs."""
    global _copy_pool
    if _copy_pool is None:
        from concurrent.futures import ThreadPoolExecutor

        _copy_pool = ThreadPoolExecutor(max_workers=max(1, min(16, os.cpu_count() or 1)),
                                        thread_name_prefix="kb-copy")
    return _copy_pool


def upload_pieces(dst, src: np.ndarray, stage) -> None:
    """dst (device tensor) <- src (host array) through the pinned staging tensor `stage` (same
    element count). Pieces are copied (and converted) into `stage` by the copy workers; each
    piece's DMA is queued on the current stream as soon as its host copy is done. The caller
    keeps `stage` untouched until the stream has passed these copies (every public call
    synchronises before returning)."""
    flat = np.ascontiguousarray(src).reshape(-1)
    hs, hn, dflat = stage.view(-1), stage.view(-1).numpy(), dst.view(-1)
    step = max(1, _PIECE_BYTES // stage.element_size())
    spans = [(a, min(flat.size, a + step)) for a in range(0, flat.size, step)]
    if len(spans) == 1:  # small images: no worker hand-off
        hn[:flat.size] = flat
        dflat[:flat.size].copy_(hs[:flat.size], non_blocking=True)
        return

    def put(a, b):
        hn[a:b] = flat[a:b]

    futs = [_pool().submit(put, a, b) for a, b in spans]
    for (a, b), f in zip(spans, futs):
        f.result()
        dflat[a:b].copy_(hs[a:b], non_blocking=True)


def prefault(out: np.ndarray) -> list:
    """Touch every page of a freshly allocated host array on the copy workers and return their
    futures. The public solvers call it right after the (asynchronous) solve launch, so the
    first-touch page faults of the result array (2 GB at cfg5) are taken while the GPU iterates
    rather than inside download_pieces."""
    flat = out.reshape(-1)
    if flat.nbytes < (8 << 20):
        return []
    per_page = max(1, 4096 // flat.itemsize)
    step = max(per_page, (flat.size // 64 + per_page - 1) // per_page * per_page)

    def touch(a, b):
        flat[a:b:per_page] = 0

    return [_pool().submit(touch, a, min(flat.size, a + step)) for a in range(0, flat.size, step)]


def download_pieces(src, stage, out: np.ndarray, after=()) -> np.ndarray:
    """out (host array) <- src (device tensor) through the pinned `stage`: every piece's DMA is
    queued at once; the copy workers move (and convert) each piece into `out` once it landed.
    `after`: futures (prefault) to finish before the host copies start."""
    torch = _torch()
    for f in after:
        f.result()
    sflat, hs, hn = src.view(-1), stage.view(-1), stage.view(-1).numpy()
    oflat = out.reshape(-1)
    step = max(1, _PIECE_BYTES // stage.element_size())
    stream = torch.cuda.current_stream()
    if sflat.numel() <= step:  # small images: one DMA, converted by the caller
        hs.copy_(sflat, non_blocking=True)
        stream.synchronize()
        oflat[:] = hn
        return out
    marks = []
    for a in range(0, sflat.numel(), step):
        b = min(sflat.numel(), a + step)
        hs[a:b].copy_(sflat[a:b], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        marks.append((a, b, ev))

    def get(a, b, ev):
        ev.synchronize()
        oflat[a:b] = hn[a:b]

    for f in [_pool().submit(get, a, b, ev) for a, b, ev in marks]:
        f.result()
    return out


def _axis_bands(factors, tol: float):
    """Unified band (dlo, [batch*r, w] taps, kind) over one axis of all terms."""
    kinds = {kind_name(f) for f in factors}
    if "hankel" in kinds:
        raise ArgumentError("pure Hankel factors are not supported by the B200 operator")
    if len(kinds) != 1:
        raise ArgumentError(f"mixed factor kinds on one axis: {sorted(kinds)}")
    bands = [factor_band(f, tol) for f in factors]
    dlo = min(b[0] for b in bands)
    dhi = max(b[0] + b[1].size - 1 for b in bands)
    taps = np.zeros((len(bands), dhi - dlo + 1))
    for i, (lo, t) in enumerate(bands):
        taps[i, lo - dlo : lo - dlo + t.size] = t
    bc = KB_BC_REFLECTIVE if kinds == {"toeplitz_plus_hankel"} else KB_BC_ZERO
    return dlo, taps, bc


class DeviceOperator:
    """Immutable device copy of one KronOperator (or a batch of equal-shape operators).

    Holds the kb_op handle, the device workspace, and reusable pinned/device staging buffers for
    the host-facing API. Thread safety: the native handle is immutable (per-launch state lives in
    each call's context, kb_capi.cu ``Ctx``); the shared workspace and the staging buffers are
    guarded by ``self.lock`` (re-entrant), which every device-path method takes, so host threads
    sharing a cached operator serialise on it instead of racing on the workspace.
    """

    def __init__(self, ops, dtype: str = "float64", band_tol: float = BAND_REL_TOL):
        torch = _torch()
        ops = list(ops)
        if not ops:
            raise ArgumentError("no operator given")
        shape = tuple(int(s) for s in ops[0].shape)
        r = len(ops[0].terms)
        for op in ops:
            if tuple(int(s) for s in op.shape) != shape or len(op.terms) != r:
                raise ArgumentError("batched operators must share shape and term count")
        m, n = shape
        for op in ops:
            for t in op.terms:
                if int(t.H.n) != m or int(t.K.n) != n:
                    raise ArgumentError(f"factor orders {(t.H.n, t.K.n)} do not match shape {shape}")
        self.shape = shape
        self.m, self.n, self.r, self.batch = m, n, r, len(ops)
        self.dtype = "float64" if _code(dtype) == KB_F64 else "float32"
        self.tdtype = torch_dtype(self.dtype)
        self.device = torch.device("cuda", torch.cuda.current_device())
        Hs = [t.H for op in ops for t in op.terms]
        Ks = [t.K for op in ops for t in op.terms]
        a_dlo, a_taps, bc_a = _axis_bands(Hs, band_tol)
        b_dlo, b_taps, bc_b = _axis_bands(Ks, band_tol)
        self.bc = (bc_a, bc_b)
        self.bands = (a_dlo, a_taps.shape[1], b_dlo, b_taps.shape[1])
        self.half_widths = (max(abs(a_dlo), abs(a_dlo + a_taps.shape[1] - 1)),
                            max(abs(b_dlo), abs(b_dlo + b_taps.shape[1] - 1)))
        lib = load_library()
        a = np.ascontiguousarray(a_taps, dtype=np.float64)
        b = np.ascontiguousarray(b_taps, dtype=np.float64)
        handle = ctypes.c_void_p()
        rc = lib.kb_op_create(
            ctypes.byref(handle), _code(self.dtype), m, n, r, self.batch, bc_a, bc_b,
            a_dlo, a.shape[1], a.ctypes.data_as(_c_dp), b_dlo, b.shape[1], b.ctypes.data_as(_c_dp),
        )
        _check(rc, "kb_op_create")
        self._handle = handle
        self._finalizer = weakref.finalize(self, lib.kb_op_destroy, handle)
        nbytes = int(lib.kb_workspace_bytes(handle))
        self.work = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.lock = threading.RLock()
        self._stage = {}
        self._norm_work = None
        self._ws_event = None  # recorded after the latest launch that used the workspace

    @contextlib.contextmanager
    def exclusive(self):
        """Exclusive use of the shared workspace: the re-entrant host lock, plus stream ordering
        on the device - the caller's stream first waits for the previous user of the workspace
        (which may have run on another stream), and marks its own use when done."""
        torch = _torch()
        with self.lock:
            stream = torch.cuda.current_stream()
            if self._ws_event is not None:
                stream.wait_event(self._ws_event)
            try:
                yield
            finally:
                ev = torch.cuda.Event()
                ev.record(stream)
                self._ws_event = ev

    def info(self) -> dict:
        """Device layout facts (kb_op_info)."""
        vals = (_c_int * 9)()
        _check(load_library().kb_op_info(self._handle, vals, 9), "kb_op_info")
        keys = ("Ha", "Wpa", "Hb", "Wpb", "sym_a", "sym_b", "adj_groups", "gmax", "twin")
        return dict(zip(keys, (int(v) for v in vals)))

    # -- buffers ---------------------------------------------------------------------------
    def plane(self, batched: bool = False):
        torch = _torch()
        shape = (self.batch, self.m, self.n) if batched or self.batch > 1 else (self.m, self.n)
        return torch.empty(shape, dtype=self.tdtype, device=self.device)

    def staging(self, name: str, pinned: bool = False):
        """Reusable buffer (device, or pinned host) of one plane (or batch) of this dtype."""
        torch = _torch()
        key = (name, pinned)
        buf = self._stage.get(key)
        if buf is None:
            shape = (self.batch, self.m, self.n) if self.batch > 1 else (self.m, self.n)
            if pinned:
                buf = torch.empty(shape, dtype=self.tdtype, pin_memory=True)
            else:
                buf = torch.empty(shape, dtype=self.tdtype, device=self.device)
            self._stage[key] = buf
        return buf

    def _as_plane(self, t, what: str):
        torch = _torch()
        want = (self.batch, self.m, self.n) if self.batch > 1 else (self.m, self.n)
        if tuple(t.shape) != want:
            raise ArgumentError(f"{what} shape {tuple(t.shape)} does not match operator shape {want}")
        if t.dtype != self.tdtype or t.device != self.device or not t.is_contiguous():
            raise ArgumentError(f"{what} must be a contiguous {self.tdtype} tensor on {self.device}")
        return t

    # -- kernels ---------------------------------------------------------------------------
    def apply(self, X, out=None, adjoint: bool = False):
        """out = A X (or A^T X) for device planes X (kron.py:218-235)."""
        with self.exclusive():
            X = self._as_plane(X, "operand")
            out = self.plane() if out is None else self._as_plane(out, "output")
            fn = load_library().kb_apply_adjoint if adjoint else load_library().kb_apply
            _check(fn(self._handle, _ptr(X), _ptr(out), _ptr(self.work), _stream_handle()),
                   "kb_apply_adjoint" if adjoint else "kb_apply")
            return out

    def resid_norms(self, AX, B, X, truth, out2):
        """out2 (device double[2]) = ||AX - B||^2, ||X - truth||^2 (kb_resid_norms; truth may be None)."""
        with self.exclusive():
            torch = _torch()
            if self._norm_work is None:
                self._norm_work = torch.empty(KB_RESID_NORMS_WORK // 8, dtype=torch.float64, device=self.device)
            AX, B, X = self._as_plane(AX, "AX"), self._as_plane(B, "data"), self._as_plane(X, "x")
            if truth is not None:
                truth = self._as_plane(truth, "truth")
            rc = load_library().kb_resid_norms(
                _code(self.dtype), _ptr(AX), _ptr(B), _ptr(X), _ptr(truth) if truth is not None else None,
                int(AX.numel()), _ptr(out2), _ptr(self._norm_work), _stream_handle())
            _check(rc, "kb_resid_norms")

    def resid_norms_images(self, AX, B) -> np.ndarray:
        """||AX[k] - B[k]||^2 per image of a batched plane (kb_resid_norms per image)."""
        with self.exclusive():
            torch = _torch()
            AX, B = self._as_plane(AX, "AX"), self._as_plane(B, "data")
            if self._norm_work is None:
                self._norm_work = torch.empty(KB_RESID_NORMS_WORK // 8, dtype=torch.float64, device=self.device)
            out = torch.zeros((self.batch, 2), dtype=torch.float64, device=self.device)
            ax, bb = AX.reshape(self.batch, -1), B.reshape(self.batch, -1)
            lib = load_library()
            for k in range(self.batch):
                rc = lib.kb_resid_norms(_code(self.dtype), _ptr(ax[k]), _ptr(bb[k]), None, None,
                                        int(self.m * self.n), _ptr(out[k]), _ptr(self._norm_work),
                                        _stream_handle())
                _check(rc, "kb_resid_norms")
            return out[:, 0].cpu().numpy()

    def sfista_run(self, B, X, Y, beta: np.ndarray, k0: int, iters: int, L, lam: float,
                   project: bool, nonfinite, norms=None, use_graph: bool = False):
        """Native loop of `iters` sFISTA iterations (kb_sfista_run)."""
        with self.exclusive():
            B = self._as_plane(B, "data")
            X = self._as_plane(X, "x")
            Y = self._as_plane(Y, "y")
            beta = np.ascontiguousarray(beta, dtype=np.float64)
            Ls = np.ascontiguousarray(np.broadcast_to(np.asarray(L, dtype=np.float64), (self.batch,)))
            if beta.size < k0 + iters:
                raise ArgumentError("momentum table shorter than the iteration range")
            if np.ndim(lam) == 0:
                fn, lam_arg, what = load_library().kb_sfista_run, float(lam), "kb_sfista_run"
            else:  # one lambda per image (select_lambda's batched probes)
                lams = np.ascontiguousarray(lam, dtype=np.float64)
                if lams.shape != (self.batch,):
                    raise ArgumentError(f"{lams.size} lambdas for a batch of {self.batch}")
                fn, lam_arg, what = load_library().kb_sfista_run_lams, lams.ctypes.data_as(_c_dp), "kb_sfista_run_lams"
            rc = fn(
                self._handle, _ptr(B), _ptr(X), _ptr(Y), _ptr(self.work), beta.ctypes.data_as(_c_dp),
                int(k0), int(iters), Ls.ctypes.data_as(_c_dp), lam_arg, int(bool(project)),
                _ptr(nonfinite), _ptr(norms) if norms is not None else None, int(bool(use_graph)),
                _stream_handle(),
            )
            _check(rc, what)

    def time_passes(self, Y, B, L: float, lam: float, reps: int = 20) -> list:
        """Average device ms of the four kernels of one iteration (kb_time_passes)."""
        with self.exclusive():
            torch = _torch()
            Y = self._as_plane(Y, "y")
            B = self._as_plane(B, "data")
            R, X, Yio = torch.empty_like(Y), torch.zeros_like(Y), Y.clone()
            flag = torch.full((1,), INT_MAX, dtype=torch.int32, device=self.device)
            Ls = np.ascontiguousarray(np.broadcast_to(np.asarray(L, dtype=np.float64), (self.batch,)))
            ms = (ctypes.c_float * 4)()
            rc = load_library().kb_time_passes(self._handle, _ptr(Y), _ptr(B), _ptr(R), _ptr(X),
                                               _ptr(Yio), _ptr(self.work), int(reps),
                                               Ls.ctypes.data_as(_c_dp), float(lam), _ptr(flag), ms,
                                               _stream_handle())
            _check(rc, "kb_time_passes")
            return [float(v) for v in ms]

    def last_engines(self) -> list:
        """Engine names of the four phases {split fwd, sum fwd, split adj, sum adj} of the latest
        sfista_run or time_passes on this operator (kb_last_engines)."""
        out = (ctypes.c_int * 4)()
        _check(load_library().kb_last_engines(self._handle, out), "kb_last_engines")
        return [ENGINES.get(int(v), str(int(v))) for v in out]

    def power_iter(self, v, iters: int):
        """Device power iteration; returns the device history [iters][2][batch] (rho, ||w||^2)."""
        with self.exclusive():
            torch = _torch()
            v = self._as_plane(v, "start vector")
            w = torch.empty_like(v)
            hist = torch.zeros((iters, 2, self.batch), dtype=torch.float64, device=self.device)
            rc = load_library().kb_power_iter(self._handle, _ptr(v), _ptr(w), _ptr(self.work),
                                              int(iters), _ptr(hist), _stream_handle())
            _check(rc, "kb_power_iter")
            return hist


def fma_peak(dtype: str = "float64") -> float:
    """Measured tensor-instruction throughput (TFLOP/s) of the current GPU: "float64" DMMA,
    "float32" TF32 mma.sync, "tcgen05_tf32" tcgen05.mma kind::tf32."""
    out = ctypes.c_float()
    code = KB_PEAK_TC_TF32 if dtype == "tcgen05_tf32" else _code(dtype)
    _check(load_library().kb_fma_peak(code, ctypes.byref(out), _stream_handle()), "kb_fma_peak")
    return float(out.value)


_cache: dict = {}
_cache_lock = threading.Lock()


def device_operator(op, dtype: str = "float64") -> DeviceOperator:
    """Cached DeviceOperator for a KronOperator (keyed by id, evicted when the op dies).

    KronOperator is unhashable (ndarray fields) but weak-referenceable.
    """
    torch = _torch()
    key = (id(op), "float64" if _code(dtype) == KB_F64 else "float32", torch.cuda.current_device())
    with _cache_lock:
        dev = _cache.get(key)
        if dev is not None:
            return dev
    dev = DeviceOperator([op], dtype)
    with _cache_lock:
        _cache[key] = dev
    try:
        weakref.finalize(op, _cache.pop, key, None)
    except TypeError:  # not weak-referenceable: keep uncached
        with _cache_lock:
            _cache.pop(key, None)
    return dev
