"""eventscope-b200: B200-native GMM EM fitting, scoring and anomaly detection.

Python view of the C-ABI in include/eventscope_b200.h (the product is the
CUDA library paper_2506_02007_b200/lib/libeventscope_b200.so; this module is
a thin ctypes binding used by tests, bench.py and Python callers).  Names,
argument meaning and errors mirror the reference's operator interface
(SPEC.md gmm-core / anomaly-detect ops, errors.hpp ErrorKind + stable names):

    fit_em
    component_log_density
    mixture_density
    responsibilities
    select_k_bic
    detect
    calibrate_threshold
    score_samples / predict (batched log-density / argmax posterior)

There is no CPU fallback: if the extension is missing or no CUDA device is
present, calls raise EventscopeError(kind="Io", name="CudaError"/"NotBuilt").
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from ._build import LIB as _LIB_PATH

__all__ = [
    "EventscopeError", "Context", "Dataset", "GmmModel", "FitReport", "DetectionReport",
    "fit_em", "component_log_density", "mixture_density", "responsibilities", "select_k_bic",
    "score_samples", "predict", "detect", "calibrate_threshold", "default_context", "load_library",
    "ES_INIT_RANDOM", "ES_INIT_KMEANSPP", "ES_INIT_GIVEN",
]

ES_INIT_RANDOM, ES_INIT_KMEANSPP, ES_INIT_GIVEN = 0, 1, 2
_KIND = {1: "Data", 2: "Numeric", 3: "Io", 4: "Io"}


class EventscopeError(RuntimeError):
    """Mirror of eventscope::Error (errors.hpp:21-37): kind + stable name."""

    def __init__(self, kind: str, name: str, message: str):
        super().__init__(f"{name}: {message}")
        self.kind = kind
        self.name = name


class _Params(C.Structure):
    _fields_ = [("K", C.c_int32), ("D", C.c_int32), ("weights", C.c_void_p), ("means", C.c_void_p),
                ("covariances", C.c_void_p)]


class _FitOpts(C.Structure):
    _fields_ = [("init", C.c_int32), ("tol", C.c_double), ("max_iter", C.c_int32), ("reg", C.c_double),
                ("seed", C.c_uint64), ("covariance_type", C.c_int32)]


class _PipelineCfg(C.Structure):
    _fields_ = [("K", C.c_int32), ("train_window", C.c_double), ("quantile_q", C.c_double), ("delta", C.c_double),
                ("standardize", C.c_int32), ("mode", C.c_int32), ("fit", _FitOpts)]


class _FitReport(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("final_log_likelihood", C.c_double), ("converged", C.c_int32),
                ("seed", C.c_uint64), ("n_per_iter", C.c_int32), ("collapses", C.c_int32),
                ("reg_used", C.c_double)]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int)


class _Exchange(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allgather", ALLGATHER_FN), ("allreduce", ALLREDUCE_FN)]


_lib = None


def load_library() -> C.CDLL:
    """Load the in-tree CUDA library (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        # ES_LIB_OVERRIDE: an instrumented in-tree build of the same library (scripts/em_trace.sh)
        path = os.environ.get("ES_LIB_OVERRIDE") or _LIB_PATH
        if not os.path.exists(path):
            raise EventscopeError("Io", "NotBuilt",
                                  f"{path} missing; run __graft_entry__.build() (no CPU fallback exists)")
        lib = C.CDLL(path)
        lib.es_last_error_name.restype = C.c_char_p
        lib.es_last_error_message.restype = C.c_char_p
        lib.es_version.restype = C.c_char_p
        _lib = lib
    return _lib


def _check(status: int) -> None:
    if status != 0:
        lib = load_library()
        raise EventscopeError(_KIND.get(status, "Io"), lib.es_last_error_name().decode(),
                              lib.es_last_error_message().decode())


def _check_tensor(t, dtype: str, ndim: int) -> None:
    """A torch tensor handed to the library: its dtype must be what the C-ABI reads (no silent
    reinterpretation) and, on the GPU, the work that produced it must be complete - the library
    reads it on its own streams, so the caller's current stream is synchronised first."""
    if str(t.dtype).replace("torch.", "") != dtype:
        raise EventscopeError("Data", "InvalidDtype", f"expected a {dtype} tensor, got {t.dtype}")
    if t.dim() != ndim:
        raise EventscopeError("Data", "DimensionMismatch", f"expected a {ndim}-D tensor, got {t.dim()}-D")
    if t.is_cuda:
        import torch
        torch.cuda.current_stream(t.device).synchronize()


def _ptr(a) -> Optional[int]:
    """Address of a numpy array or torch tensor (host or device); None passes NULL."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


@dataclass
class FitReport:
    iterations: int = 0
    final_log_likelihood: float = 0.0
    per_iteration_log_likelihoods: np.ndarray = field(default_factory=lambda: np.zeros(0))
    converged: bool = False
    seed: int = 0
    collapses: int = 0
    reg: float = 0.0


@dataclass
class GmmModel:
    """weights (K), means (K,d), covariances (K,d,d)."""
    weights: np.ndarray
    means: np.ndarray
    covariances: np.ndarray
    fit_report: FitReport = field(default_factory=FitReport)

    @property
    def K(self) -> int:
        return int(self.weights.shape[0])

    @property
    def d(self) -> int:
        return int(self.means.shape[1])

    def _c(self):
        w = np.ascontiguousarray(self.weights, np.float64)
        m = np.ascontiguousarray(self.means, np.float64)
        c = np.ascontiguousarray(self.covariances, np.float64)
        if m.ndim != 2 or m.shape[0] != w.shape[0] or c.shape != (w.shape[0], m.shape[1], m.shape[1]):
            raise EventscopeError("Data", "InvalidModel", "weights/means/covariances shapes disagree")
        p = _Params(w.shape[0], m.shape[1], w.ctypes.data, m.ctypes.data, c.ctypes.data)
        return p, (w, m, c)


@dataclass
class DetectionReport:
    """SPEC.md:351-354."""
    flags: np.ndarray
    anomaly_indices: np.ndarray
    best_component: np.ndarray
    log_density: np.ndarray
    model: GmmModel
    delta: float
    log_delta: float
    n_flagged: int = 0


class Context:
    """One GPU (one process per GPU).  world>1 uses NCCL (nccl_id) or host
    exchange callbacks (exchange=(allgather_fn, allreduce_fn))."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 exchange=None, precision: str = "mixed"):
        lib = load_library()
        self._lib = lib
        h = C.c_void_p()
        self._keep = None
        if world > 1 and exchange is not None:
            ag, ar = exchange
            ex = _Exchange(None, ALLGATHER_FN(ag), ALLREDUCE_FN(ar))
            self._keep = ex
            _check(lib.es_ctx_create_exchange(device, rank, world, C.byref(ex), C.byref(h)))
        elif world > 1:
            idb = (C.c_ubyte * 128).from_buffer_copy(nccl_id)
            _check(lib.es_ctx_create_nccl(device, rank, world, idb, C.byref(h)))
        else:
            _check(lib.es_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device, self.rank, self.world = device, rank, world
        import weakref
        self._datasets = weakref.WeakSet()
        self.set_precision(os.environ.get("ES_PRECISION", precision))

    def set_precision(self, mode: str) -> None:
        """'mixed' (default: FP32 whitening, FP64 statistics) or 'fp64' (strict)."""
        _check(self._lib.es_ctx_set_precision(self.handle, {"mixed": 0, "fp64": 1}[mode]))
        self.precision = mode

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        _check(load_library().es_nccl_unique_id(buf))
        return bytes(buf)

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _check(self._lib.es_ctx_stream(self.handle, C.byref(s)))
        return s.value or 0

    @property
    def launch_count(self) -> int:
        n = C.c_int64()
        _check(self._lib.es_ctx_launch_count(self.handle, C.byref(n)))
        return n.value

    @property
    def collective_count(self) -> int:
        """NCCL collectives this context issued."""
        n = C.c_int64()
        _check(self._lib.es_ctx_collective_count(self.handle, C.byref(n)))
        return n.value

    def close(self) -> None:
        if getattr(self, "handle", None):
            for ds in list(getattr(self, "_datasets", ())):  # datasets first (the library detaches any left)
                ds.close()
            self._lib.es_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("ES_DEVICE", "0")))
    return _default_ctx


class Dataset:
    """This rank's event rows, resident in HBM (feature-planar FP64)."""

    def __init__(self, ctx: Context, handle: C.c_void_p):
        self.ctx = ctx
        self.handle = handle
        if hasattr(ctx, "_datasets"):
            ctx._datasets.add(self)
        nl, ng, off, d = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
        _check(ctx._lib.es_dataset_info(handle, C.byref(nl), C.byref(ng), C.byref(off), C.byref(d)))
        self.n_local, self.n_global, self.row_offset, self.D = nl.value, ng.value, off.value, d.value

    @classmethod
    def from_array(cls, X, ctx: Optional[Context] = None) -> "Dataset":
        """X: numpy (N,D) float64 (any strides) or a CUDA torch tensor (row- or column-major)."""
        ctx = ctx or default_context()
        if hasattr(X, "data_ptr"):
            _check_tensor(X, "float64", 2)
            n, d = X.shape
            rs, cs = X.stride()
            ptr = X.data_ptr()
        else:
            X = np.asarray(X, np.float64)
            if X.ndim == 1:
                X = X[:, None]
            n, d = X.shape
            rs, cs = X.strides[0] // 8, X.strides[1] // 8
            if X.strides[0] % 8 or X.strides[1] % 8:
                X = np.ascontiguousarray(X)
                rs, cs = d, 1
            ptr = X.ctypes.data
        h = C.c_void_p()
        _check(ctx._lib.es_dataset_create(ctx.handle, C.c_void_p(ptr), C.c_int64(n), C.c_int32(d),
                                          C.c_int64(rs), C.c_int64(cs), C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def generate(cls, seed: int, n_global: int, D: int, K_true: int, ctx: Optional[Context] = None,
                 row0: int = 0) -> "Dataset":
        """SYN-v1 synthetic events generated on the device (this rank's shard); row0 > 0
        selects rows [row0, row0 + n_global) of the same stream."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(ctx._lib.es_dataset_generate_range(ctx.handle, C.c_uint64(seed), C.c_int64(row0), C.c_int64(n_global),
                                                  C.c_int32(D), C.c_int32(K_true), C.byref(h)))
        return cls(ctx, h)

    def read_rows(self, row0: int = 0, n: Optional[int] = None, out=None):
        """Rows [row0, row0+n) row-major into `out` (numpy / pinned or CUDA tensor) or a new array."""
        n = self.n_local - row0 if n is None else n
        if out is None:
            out = np.empty((n, self.D))
        _check(self.ctx._lib.es_dataset_read_rows(self.handle, C.c_int64(row0), C.c_int64(n),
                                                  C.c_void_p(_ptr(out))))
        return out

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.ctx._lib.es_dataset_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _as_dataset(X, ctx: Optional[Context]) -> Dataset:
    return X if isinstance(X, Dataset) else Dataset.from_array(X, ctx)


def _seed(seed: Optional[int]) -> int:
    """An explicit seed wins; an omitted one (None) takes EACGM_SEED (the CLI-level
    override) or 0.  Applied identically by every seeded entry point (fits, BIC, pipeline,
    k-means baseline)."""
    if seed is not None:
        return int(seed)
    env = os.environ.get("EACGM_SEED")
    return int(env) if env is not None else 0


def _opts(init, tol, max_iter, reg, seed, covariance_type="full") -> _FitOpts:
    code = {"random": ES_INIT_RANDOM, "kmeans++": ES_INIT_KMEANSPP, "kmeanspp": ES_INIT_KMEANSPP,
            "given": ES_INIT_GIVEN}[init] if isinstance(init, str) else int(init)
    seed = _seed(seed)
    return _FitOpts(code, float(tol), int(max_iter), -1.0 if reg is None else float(reg), int(seed),
                    {"full": 0, "diag": 1}[covariance_type])


class EM:
    """Stepwise EM engine (es_gmm_em_begin/step/end): same semantics as fit_em."""

    def __init__(self, X, K: int, init="kmeans++", tol=1e-6, max_iter=200, reg=None, seed=None,
                 init_params: Optional[GmmModel] = None, ctx: Optional[Context] = None, covariance_type="full"):
        self.ds = _as_dataset(X, ctx)
        self.ctx = self.ds.ctx
        self.K = K
        o = _opts("given" if init_params is not None else init, tol, max_iter, reg, seed, covariance_type)
        self.max_iter = o.max_iter
        keep = None
        pp = None
        if init_params is not None:
            p, keep = init_params._c()
            pp = C.byref(p)
        h = C.c_void_p()
        _check(self.ctx._lib.es_gmm_em_begin(self.ctx.handle, self.ds.handle, C.c_int32(K), C.byref(o), pp,
                                             C.byref(h)))
        del keep
        self.handle = h
        self.done = False

    def step(self, n: int = 1) -> bool:
        d = C.c_int32()
        _check(self.ctx._lib.es_gmm_em_step(self.handle, C.c_int32(n), C.byref(d)))
        self.done = bool(d.value)
        return self.done


    @property
    def record_passes(self) -> int:
        """Record precision of the last fused tcgen05 E+M pass (1 or 2; 0 = another kernel)."""
        v = C.c_int32()
        _check(self.ctx._lib.es_gmm_em_record_passes(self.handle, C.byref(v)))
        return v.value
    @property
    def last_kernel(self) -> str:
        """EM pass kernel of the last iteration (e.g. 'k_em_mma<1>', 'k_em_diag_mixed')."""
        v = C.c_char_p()
        _check(self.ctx._lib.es_gmm_em_last_kernel(self.handle, C.byref(v)))
        return v.value.decode()

    def finish(self) -> GmmModel:
        K, D = self.K, self.ds.D
        w, m, c = np.empty(K), np.empty((K, D)), np.empty((K, D, D))
        out = _Params(K, D, w.ctypes.data, m.ctypes.data, c.ctypes.data)
        rep = _FitReport()
        per = np.empty(self.max_iter + 1)
        _check(self.ctx._lib.es_gmm_em_end(self.handle, C.byref(out), C.byref(rep), C.c_void_p(per.ctypes.data)))
        fr = FitReport(rep.iterations, rep.final_log_likelihood, per[:rep.n_per_iter].copy(), bool(rep.converged),
                       rep.seed, rep.collapses, rep.reg_used)
        return GmmModel(w, m, c, fr)

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.ctx._lib.es_gmm_em_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fit_em(X, K: int, init="kmeans++", tol: float = 1e-6, max_iter: int = 200, reg: Optional[float] = None,
           seed: Optional[int] = None, init_params: Optional[GmmModel] = None, ctx: Optional[Context] = None,
           covariance_type: str = "full") -> GmmModel:
    """EM fit.  Defaults per SPEC.md:319-321.  covariance_type "diag" is an
    extension (diagonal covariances, not in the reference)."""
    em = EM(X, K, init, tol, max_iter, reg, seed, init_params, ctx, covariance_type)
    try:
        em.step(max(max_iter, 0))
        return em.finish()
    finally:
        em.close()


def score(model: GmmModel, X, ctx: Optional[Context] = None, ll=None, predict=None, best_k=None,
          best_logdens=None) -> float:
    """Batched scoring into caller buffers (numpy or CUDA tensors); returns global sum of ll."""
    ds = _as_dataset(X, ctx)
    p, keep = model._c()
    tot = C.c_double()
    _check(ds.ctx._lib.es_gmm_score(ds.ctx.handle, ds.handle, C.byref(p), C.c_void_p(_ptr(ll)),
                                    C.c_void_p(_ptr(predict)), C.c_void_p(_ptr(best_k)),
                                    C.c_void_p(_ptr(best_logdens)), C.byref(tot)))
    del keep
    return tot.value


def score_samples(model: GmmModel, X, ctx: Optional[Context] = None) -> np.ndarray:
    ds = _as_dataset(X, ctx)
    ll = np.empty(ds.n_local)
    score(model, ds, ll=ll)
    return ll


def predict(model: GmmModel, X, ctx: Optional[Context] = None) -> np.ndarray:
    ds = _as_dataset(X, ctx)
    pr = np.empty(ds.n_local, np.int32)
    score(model, ds, predict=pr)
    return pr


def responsibilities(model: GmmModel, X, ctx: Optional[Context] = None) -> np.ndarray:
    ds = _as_dataset(X, ctx)
    p, keep = model._c()
    g = np.empty((ds.n_local, model.K))
    _check(ds.ctx._lib.es_gmm_responsibilities(ds.ctx.handle, ds.handle, C.byref(p), C.c_void_p(g.ctypes.data)))
    del keep
    return g


def component_log_density(model: GmmModel, x, k: int, ctx: Optional[Context] = None) -> float:
    ctx = ctx or default_context()
    x = np.ascontiguousarray(x, np.float64).reshape(-1)
    if x.shape[0] != model.d:
        raise EventscopeError("Data", "DimensionMismatch", "x has the wrong dimension")
    p, keep = model._c()
    out = C.c_double()
    _check(ctx._lib.es_gmm_component_log_density(ctx.handle, C.byref(p), C.c_void_p(x.ctypes.data),
                                                 C.c_int32(k), C.byref(out)))
    del keep
    return out.value


def mixture_density(model: GmmModel, x, ctx: Optional[Context] = None) -> float:
    ctx = ctx or default_context()
    x = np.ascontiguousarray(x, np.float64).reshape(-1)
    if x.shape[0] != model.d:
        raise EventscopeError("Data", "DimensionMismatch", "x has the wrong dimension")
    p, keep = model._c()
    out = C.c_double()
    _check(ctx._lib.es_gmm_mixture_log_density(ctx.handle, C.byref(p), C.c_void_p(x.ctypes.data), C.byref(out)))
    del keep
    return float(np.exp(out.value))


def detect(model: GmmModel, X, delta: Optional[float] = None, mode: str = "component",
           log_delta: Optional[float] = None, ctx: Optional[Context] = None, flags=None, best_k=None,
           best_logdens=None, indices=True) -> DetectionReport:
    """Def. 1 / Alg. 2: flag iff log p < log delta (strict).
    flags / best_k / best_logdens / indices may be caller buffers (numpy or CUDA tensors; a
    device buffer keeps that output in HBM); indices=False skips the anomaly-index list."""
    if log_delta is None:
        if delta is None or not delta > 0:
            raise EventscopeError("Data", "RangeViolation", "delta must be > 0")
        log_delta = float(np.log(delta)) if np.isfinite(delta) else float("inf")
    ds = _as_dataset(X, ctx)
    p, keep = model._c()
    n = ds.n_local
    fl = np.empty(n, np.uint8) if flags is None else flags
    bk = np.empty(n, np.int32) if best_k is None else best_k
    bl = np.empty(n) if best_logdens is None else best_logdens
    if indices is True:
        idx = np.empty(max(n, 1), np.int64)
    elif indices is False or indices is None:
        idx = None
    else:
        idx = indices  # caller buffer, capacity >= n_local
    nloc, ng = C.c_int64(), C.c_int64()
    m = {"component": 0, "mixture": 1}[mode]
    _check(ds.ctx._lib.es_gmm_detect(ds.ctx.handle, ds.handle, C.byref(p), C.c_double(log_delta), C.c_int32(m),
                                     C.c_void_p(_ptr(fl)), C.c_void_p(_ptr(bk)), C.c_void_p(_ptr(bl)),
                                     C.c_void_p(_ptr(idx)), C.byref(nloc), C.byref(ng)))
    del keep
    A = np.zeros(0, np.int64) if idx is None else (idx[:nloc.value].copy() if indices is True else idx[:nloc.value])
    d = float(np.exp(log_delta)) if delta is None else float(delta)
    return DetectionReport(fl, A, bk, bl, model, d, float(log_delta), ng.value)


def calibrate_threshold(model: GmmModel, X_train, q: float, mode: str = "component", n_train: Optional[int] = None,
                        ctx: Optional[Context] = None, return_log: bool = False):
    """delta = q-quantile of best-component densities over the train rows."""
    ds = _as_dataset(X_train, ctx)
    nt = ds.n_global if n_train is None else n_train
    p, keep = model._c()
    d, ld = C.c_double(), C.c_double()
    m = {"component": 0, "mixture": 1}[mode]
    _check(ds.ctx._lib.es_gmm_calibrate(ds.ctx.handle, ds.handle, C.byref(p), C.c_int64(nt), C.c_double(q),
                                        C.c_int32(m), C.byref(d), C.byref(ld)))
    del keep
    return (d.value, ld.value) if return_log else d.value


def select_k_bic(X, k_range: Sequence[int], init="kmeans++", tol=1e-6, max_iter=200, reg=None, seed=None,
                 ctx: Optional[Context] = None, covariance_type: str = "full"):
    """(best_K, bic_values); failed K -> NaN."""
    ds = _as_dataset(X, ctx)
    kr = np.ascontiguousarray(list(k_range), np.int32)
    bic = np.empty(len(kr))
    best = C.c_int32()
    o = _opts(init, tol, max_iter, reg, seed, covariance_type)
    _check(ds.ctx._lib.es_gmm_select_k_bic(ds.ctx.handle, ds.handle, C.c_void_p(kr.ctypes.data),
                                           C.c_int32(len(kr)), C.byref(o), C.byref(best),
                                           C.c_void_p(bic.ctypes.data)))
    return best.value, bic


@dataclass
class PipelineResult:
    """run_pipeline: the model (standardized space), the standardization
    (per-column mean, scale; scale 1 for a zero-variance column), the threshold and the
    DetectionReport over ALL events."""
    model: GmmModel
    report: DetectionReport
    mean: np.ndarray
    scale: np.ndarray
    n_train: int


def run_pipeline(X, K: int, train_window: float = 0.5, quantile_q: Optional[float] = 0.01,
                 delta: Optional[float] = None, standardize: bool = True, mode: str = "component",
                 init="kmeans++", tol: float = 1e-6, max_iter: int = 200, reg: Optional[float] = None,
                 seed: Optional[int] = None,
                 ctx: Optional[Context] = None) -> PipelineResult:
    """run_pipeline over a time-ordered feature matrix: fit on the standardized
    first train_window fraction, calibrate delta as the quantile_q-quantile there (or use delta),
    detect over every event.  Runs on the device end to end (es_run_pipeline)."""
    ds = _as_dataset(X, ctx)
    D, n = ds.D, ds.n_local
    q = float(quantile_q) if quantile_q is not None and delta is None else 0.0
    cfg = _PipelineCfg(int(K), float(train_window), q, float(delta) if delta is not None else 0.0,
                       1 if standardize else 0, {"component": 0, "mixture": 1}[mode],
                       _opts(init, tol, max_iter, reg, seed))
    w, mu, cov = np.empty(K), np.empty((K, D)), np.empty((K, D, D))
    p = _Params(K, D, w.ctypes.data, mu.ctypes.data, cov.ctypes.data)
    rep = _FitReport()
    mean, scale = np.empty(D), np.empty(D)
    d, ld = C.c_double(), C.c_double()
    fl, bk, bl = np.empty(n, np.uint8), np.empty(n, np.int32), np.empty(n)
    idx = np.empty(max(n, 1), np.int64)
    nloc, ng = C.c_int64(), C.c_int64()
    _check(ds.ctx._lib.es_run_pipeline(ds.ctx.handle, ds.handle, C.byref(cfg), C.byref(p), C.byref(rep),
                                       mean.ctypes.data_as(C.c_void_p), scale.ctypes.data_as(C.c_void_p),
                                       C.byref(d), C.byref(ld), C.c_void_p(_ptr(fl)), C.c_void_p(_ptr(bk)),
                                       C.c_void_p(_ptr(bl)), C.c_void_p(_ptr(idx)), C.byref(nloc), C.byref(ng)))
    fr = FitReport(rep.iterations, rep.final_log_likelihood, np.zeros(0), bool(rep.converged), rep.seed,
                   rep.collapses, rep.reg_used)
    model = GmmModel(w, mu, cov, fr)
    report = DetectionReport(fl, idx[:nloc.value].copy(), bk, bl, model, d.value, ld.value, ng.value)
    return PipelineResult(model, report, mean, scale, int(np.floor(train_window * ds.n_global)))


# ------------------------------------------------------------------ eval-bench
@dataclass
class KMeansResult:
    """kmeans_baseline: centroids fitted on the train split, the
    (1-q)-quantile threshold of the train distances, per-event distances and flags."""
    centroids: np.ndarray
    threshold: float
    flags: np.ndarray
    scores: np.ndarray
    n_flagged: int
    iterations: int


def kmeans_baseline(X, K: int, q: float = 0.01, train_window: float = 0.5, seed: Optional[int] = None,
                    max_iter: int = 100,
                    ctx: Optional[Context] = None) -> KMeansResult:
    """KMeans baseline on the device (es_kmeans_baseline): k-means++ seeding and Lloyd's
    algorithm on the first train_window fraction of the events; flag iff the distance to
    the nearest centroid exceeds the (1-q)-quantile of the train distances."""
    ds = _as_dataset(X, ctx)
    D, n = ds.D, ds.n_local
    cen = np.empty((K, D))
    fl, sc = np.empty(n, np.uint8), np.empty(n)
    thr, nf, it = C.c_double(), C.c_int64(), C.c_int32()
    _check(ds.ctx._lib.es_kmeans_baseline(ds.ctx.handle, ds.handle, C.c_int32(K), C.c_double(q),
                                          C.c_double(train_window), C.c_uint64(_seed(seed)), C.c_int32(max_iter),
                                          C.c_void_p(cen.ctypes.data), C.byref(thr), C.c_void_p(_ptr(fl)),
                                          C.c_void_p(_ptr(sc)), C.byref(nf), C.byref(it)))
    return KMeansResult(cen, thr.value, fl, sc, nf.value, it.value)


@dataclass
class ConfusionMatrix:
    """counts with anomaly as the positive class."""
    tp: int
    fp: int
    tn: int
    fn: int


def confusion(labels, flags, ctx: Optional[Context] = None) -> ConfusionMatrix:
    """confusion(labels, flags), counted on the device (es_confusion);
    labels / flags may be host arrays or device tensors of equal length."""
    c = ctx or default_context()
    nl, nf = len(labels), len(flags)
    if nl != nf:
        raise EventscopeError("Data", "LengthMismatch", f"labels ({nl}) and flags ({nf}) differ in length")
    for t in (labels, flags):
        if hasattr(t, "data_ptr"):
            _check_tensor(t, "uint8", 1)
    lab = labels if hasattr(labels, "data_ptr") else np.ascontiguousarray(labels, np.uint8)
    fl = flags if hasattr(flags, "data_ptr") else np.ascontiguousarray(flags, np.uint8)
    out = np.zeros(4, np.int64)
    _check(c._lib.es_confusion(c.handle, C.c_void_p(_ptr(lab)), C.c_void_p(_ptr(fl)), C.c_int64(nl),
                               C.c_void_p(out.ctypes.data)))
    return ConfusionMatrix(*(int(v) for v in out))


@dataclass
class EvalSummary:
    """SPEC.md:424-428."""
    accuracy: float
    precision: float
    recall: float
    f1: float
    cm: ConfusionMatrix
    method: str = "gmm"
    params: tuple = ()


def metrics(cm: ConfusionMatrix, method: str = "gmm", params: tuple = ()) -> EvalSummary:
    """metrics(cm): zero-division conventions fixed to 0."""
    n = cm.tp + cm.fp + cm.tn + cm.fn
    if n <= 0:
        raise EventscopeError("Data", "EmptyMatrix", "confusion matrix has no events")
    precision = cm.tp / (cm.tp + cm.fp) if cm.tp + cm.fp else 0.0
    recall = cm.tp / (cm.tp + cm.fn) if cm.tp + cm.fn else 0.0
    f1 = 2 * precision * recall / (precision + recall) if precision + recall else 0.0
    return EvalSummary((cm.tp + cm.tn) / n, precision, recall, f1, cm, method, params)


def sensitivity_sweep(X, labels, K_range: Sequence[int], q_range: Sequence[float], seeds: Sequence[int] = (0,),
                      layer: str = "all", csv_path: Optional[str] = None, ctx: Optional[Context] = None,
                      **pipeline_kw):
    """sensitivity_sweep: the full K x q grid of run_pipeline cells, each
    averaged over seeds; a failing cell is recorded in the grid (status = error name), not
    raised.  The feature matrix is uploaded once and shared by every cell.  Returns rows
    with the CSV columns layer, K, q, seed_count, accuracy, precision, recall, f1, status
    (and writes them to csv_path when given)."""
    if not len(K_range) or not len(q_range) or not len(seeds):
        raise EventscopeError("Data", "EmptyRange", "K_range, q_range and seeds must be nonempty")
    ds = _as_dataset(X, ctx)
    lab = np.ascontiguousarray(labels, np.uint8)
    rows = []
    for K in K_range:
        for q in q_range:
            acc = []
            status = "ok"
            for sd in seeds:
                try:
                    r = run_pipeline(ds, int(K), quantile_q=float(q), seed=int(sd), **pipeline_kw)
                    acc.append(metrics(confusion(lab, r.report.flags, ds.ctx), "gmm", (int(K), float(q))))
                except EventscopeError as e:
                    status = e.name
            if acc:
                m = [float(np.mean([getattr(a, f) for a in acc])) for f in ("accuracy", "precision", "recall", "f1")]
            else:
                m = [float("nan")] * 4
            rows.append({"layer": layer, "K": int(K), "q": float(q), "seed_count": len(acc), "accuracy": m[0],
                         "precision": m[1], "recall": m[2], "f1": m[3], "status": status})
    if csv_path:
        import csv as _csv
        with open(csv_path, "w", newline="") as fh:
            w = _csv.DictWriter(fh, fieldnames=["layer", "K", "q", "seed_count", "accuracy", "precision", "recall",
                                                "f1", "status"])
            w.writeheader()
            w.writerows(rows)
    return rows


from .events import (EventColumns, extract_features, from_records, read_columnar, read_trace_jsonl,  # noqa: E402
                     write_columnar)
