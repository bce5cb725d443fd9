"""ctypes view of the CPU oracle (oracle/build/libes_oracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py — never by the product
package.  See es_oracle.h for the algorithm sources (SPEC.md file:line).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libes_oracle.so")

_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, status: int, name: str, message: str):
        super().__init__(f"{name}: {message}")
        self.status = status
        self.name = name


class FitOpts(C.Structure):
    _fields_ = [("init", C.c_int), ("tol", C.c_double), ("max_iter", C.c_int),
                ("reg", C.c_double), ("seed", C.c_uint64), ("nthreads", C.c_int), ("cov_type", C.c_int)]


class FitReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("final_log_likelihood", C.c_double),
                ("converged", C.c_int), ("seed", C.c_uint64), ("n_per_iter", C.c_int),
                ("collapses", C.c_int), ("reg_used", C.c_double)]


def build() -> str:
    """Compile the oracle with its committed Makefile (checker, not product)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.eso_last_error_name.restype = C.c_char_p
        _lib.eso_last_error_message.restype = C.c_char_p
    return _lib


def _check(status: int) -> None:
    if status != 0:
        L = lib()
        raise OracleError(status, L.eso_last_error_name().decode(), L.eso_last_error_message().decode())


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _params(pi, mu, cov):
    pi = np.ascontiguousarray(pi, np.float64)
    mu = np.ascontiguousarray(mu, np.float64)
    cov = np.ascontiguousarray(cov, np.float64)
    K = pi.shape[0]
    D = mu.shape[1]
    assert mu.shape == (K, D) and cov.shape == (K, D, D)
    return pi, mu, cov, K, D


def component_log_density(pi, mu, cov, x, k) -> float:
    pi, mu, cov, K, D = _params(pi, mu, cov)
    x = np.ascontiguousarray(x, np.float64).reshape(-1)
    if x.shape[0] != D:
        raise OracleError(1, "DimensionMismatch", "x has wrong dimension")
    out = C.c_double()
    _check(lib().eso_component_log_density(_p(pi), _p(mu), _p(cov), K, D, _p(x), int(k), C.byref(out)))
    return out.value


def mixture_log_density(pi, mu, cov, x) -> float:
    pi, mu, cov, K, D = _params(pi, mu, cov)
    x = np.ascontiguousarray(x, np.float64).reshape(-1)
    out = C.c_double()
    _check(lib().eso_mixture_log_density(_p(pi), _p(mu), _p(cov), K, D, _p(x), C.byref(out)))
    return out.value


def score(X, pi, mu, cov, gamma=False, nthreads=0):
    """Returns dict(ll, predict, best_k, best_logdens[, gamma])."""
    pi, mu, cov, K, D = _params(pi, mu, cov)
    X = np.ascontiguousarray(X, np.float64)
    N = X.shape[0]
    ll = np.empty(N)
    pred = np.empty(N, np.int32)
    bk = np.empty(N, np.int32)
    bl = np.empty(N)
    g = np.empty((N, K)) if gamma else None
    _check(lib().eso_score(_p(X), C.c_int64(N), D, _p(pi), _p(mu), _p(cov), K, _p(ll), _p(pred), _p(bk),
                           _p(bl), _p(g), nthreads))
    out = dict(ll=ll, predict=pred, best_k=bk, best_logdens=bl)
    if gamma:
        out["gamma"] = g
    return out


def data_stats(X, nthreads=0):
    X = np.ascontiguousarray(X, np.float64)
    N, D = X.shape
    mean, S, mn, mx = np.empty(D), np.empty((D, D)), np.empty(D), np.empty(D)
    _check(lib().eso_data_stats(_p(X), C.c_int64(N), D, _p(mean), _p(S), _p(mn), _p(mx), nthreads))
    return mean, S, mn, mx


def random_init(X, K, seed, reg=-1.0):
    X = np.ascontiguousarray(X, np.float64)
    N, D = X.shape
    pi, mu, cov = np.empty(K), np.empty((K, D)), np.empty((K, D, D))
    reg_used = C.c_double()
    _check(lib().eso_random_init(_p(X), C.c_int64(N), D, K, C.c_uint64(seed), C.c_double(reg), _p(pi), _p(mu),
                                 _p(cov), C.byref(reg_used)))
    return pi, mu, cov, reg_used.value


INIT_RANDOM, INIT_KMEANSPP, INIT_GIVEN = 0, 1, 2


def fit_em(X, K, init="kmeans++", tol=1e-6, max_iter=200, reg=None, seed=0, init_params=None, nthreads=0,
           covariance_type="full"):
    X = np.ascontiguousarray(X, np.float64)
    N, D = X.shape
    code = {"random": INIT_RANDOM, "kmeans++": INIT_KMEANSPP, "given": INIT_GIVEN}[init]
    if init_params is not None:
        code = INIT_GIVEN
    opts = FitOpts(code, tol, max_iter, -1.0 if reg is None else float(reg), seed, nthreads,
                   {"full": 0, "diag": 1}[covariance_type])
    pi, mu, cov = np.empty(K), np.empty((K, D)), np.empty((K, D, D))
    per = np.empty(max_iter + 1)
    rep = FitReport()
    ip = im = ic = None
    if code == INIT_GIVEN:
        ip, im, ic, _, _ = _params(*init_params)
    _check(lib().eso_fit_em(_p(X), C.c_int64(N), D, K, C.byref(opts), _p(ip), _p(im), _p(ic), _p(pi), _p(mu),
                            _p(cov), C.byref(rep), _p(per)))
    report = dict(iterations=rep.iterations, final_log_likelihood=rep.final_log_likelihood,
                  converged=bool(rep.converged), seed=rep.seed, collapses=rep.collapses, reg=rep.reg_used,
                  per_iteration_log_likelihoods=per[:rep.n_per_iter].copy())
    return pi, mu, cov, report


def em_step(X, pi, mu, cov, reg, nthreads=0, covariance_type="full"):
    """One EM iteration in place on (pi, mu, cov) (C-contiguous float64 arrays, updated);
    returns (logL of the entry parameters, number of components with N_k < 1)."""
    X = np.ascontiguousarray(X, np.float64)
    N, D = X.shape
    K = pi.shape[0]
    for a in (pi, mu, cov):
        assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    ll, nc = C.c_double(), C.c_int()
    _check(lib().eso_em_step(_p(X), C.c_int64(N), D, K, C.c_double(reg), {"full": 0, "diag": 1}[covariance_type],
                             _p(pi), _p(mu), _p(cov), C.byref(ll), C.byref(nc), nthreads))
    return ll.value, nc.value


def detect(X, pi, mu, cov, log_delta, mode=0, nthreads=0):
    pi, mu, cov, K, D = _params(pi, mu, cov)
    X = np.ascontiguousarray(X, np.float64)
    N = X.shape[0]
    flags = np.empty(N, np.uint8)
    bk = np.empty(N, np.int32)
    bl = np.empty(N)
    n = C.c_int64()
    _check(lib().eso_detect(_p(X), C.c_int64(N), D, _p(pi), _p(mu), _p(cov), K, C.c_double(log_delta), mode,
                            _p(flags), _p(bk), _p(bl), C.byref(n), nthreads))
    return flags, bk, bl, n.value


def calibrate(X_train, pi, mu, cov, q, mode=0, nthreads=0):
    pi, mu, cov, K, D = _params(pi, mu, cov)
    X = np.ascontiguousarray(X_train, np.float64)
    d, ld = C.c_double(), C.c_double()
    _check(lib().eso_calibrate(_p(X), C.c_int64(X.shape[0]), D, _p(pi), _p(mu), _p(cov), K, C.c_double(q), mode,
                               C.byref(d), C.byref(ld), nthreads))
    return d.value, ld.value


def kmeans_baseline(X, K, q=0.01, train_window=0.5, seed=0, max_iter=100, nthreads=0):
    """SPEC.md:451-458 restated (es_oracle.cpp eso_kmeans_baseline)."""
    X = np.ascontiguousarray(X, np.float64)
    N, D = X.shape
    cen = np.empty((K, D))
    flags = np.empty(N, np.uint8)
    scores = np.empty(N)
    thr, nf, it = C.c_double(), C.c_int64(), C.c_int()
    _check(lib().eso_kmeans_baseline(_p(X), C.c_int64(N), D, K, C.c_double(q), C.c_double(train_window),
                                     C.c_uint64(seed), max_iter, _p(cen), C.byref(thr), _p(flags), _p(scores),
                                     C.byref(nf), C.byref(it), nthreads))
    return cen, thr.value, flags, scores, nf.value, it.value


def lloyd(X, centroids, max_iter=300):
    """Lloyd's iterations from given centroids (the kmeans_baseline inner loop)."""
    X = np.ascontiguousarray(X, np.float64)
    cen = np.array(centroids, np.float64, order="C", copy=True)
    it = C.c_int()
    _check(lib().eso_lloyd(_p(X), C.c_int64(X.shape[0]), X.shape[1], cen.shape[0], _p(cen), max_iter,
                           C.byref(it)))
    return cen, it.value


def confusion(labels, flags):
    """(tp, fp, tn, fn), anomaly = positive class."""
    lab = np.ascontiguousarray(labels, np.uint8)
    fl = np.ascontiguousarray(flags, np.uint8)
    if lab.shape != fl.shape:
        raise OracleError(1, "LengthMismatch", "labels and flags differ in length")
    out = np.zeros(4, np.int64)
    _check(lib().eso_confusion(_p(lab), _p(fl), C.c_int64(lab.size), _p(out)))
    return tuple(int(v) for v in out)


def select_k_bic(X, k_range, init="kmeans++", tol=1e-6, max_iter=200, reg=None, seed=0, nthreads=0,
                 covariance_type="full"):
    X = np.ascontiguousarray(X, np.float64)
    N, D = X.shape
    kr = np.ascontiguousarray(k_range, np.int32)
    code = {"random": INIT_RANDOM, "kmeans++": INIT_KMEANSPP}[init]
    opts = FitOpts(code, tol, max_iter, -1.0 if reg is None else float(reg), seed, nthreads,
                   {"full": 0, "diag": 1}[covariance_type])
    bic = np.empty(len(kr))
    best = C.c_int()
    _check(lib().eso_select_k_bic(_p(X), C.c_int64(N), D, _p(kr), len(kr), C.byref(opts), C.byref(best), _p(bic)))
    return best.value, bic


def syn_model(seed, D, K):
    pi, mu, ch = np.empty(K), np.empty((K, D)), np.empty((K, D, D))
    _check(lib().eso_syn_model(C.c_uint64(seed), D, K, _p(pi), _p(mu), _p(ch)))
    return pi, mu, ch


def syn_rows(seed, D, K, model, row0, n, nthreads=0):
    pi, mu, ch = model
    X = np.empty((n, D))
    comp = np.empty(n, np.int32)
    anom = np.empty(n, np.uint8)
    _check(lib().eso_syn_rows(C.c_uint64(seed), D, K, _p(pi), _p(mu), _p(ch), C.c_int64(row0), C.c_int64(n),
                              _p(X), _p(comp), _p(anom), nthreads))
    return X, comp, anom


def philox4x32(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().eso_philox4x32(c, k, o)
    return list(o)
