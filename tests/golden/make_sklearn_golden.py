"""Generates tests/golden/sklearn_*.npz: independent cross-check fixtures for
the CPU oracle (scikit-learn 1.9.0 GaussianMixture, full covariance).

sklearn is NOT a dependency of the reference; it is an independent
implementation of the same M-step (Sigma_k = sum gamma (x-mu)(x-mu)^T / N_k
+ reg I, sklearn/mixture/_gaussian_mixture.py:195-196) used to pin the oracle
where the reference ships no vectors (SPEC has only closed-form examples).
Run:  python tests/golden/make_sklearn_golden.py
"""
import os

import numpy as np
import sklearn
from sklearn.mixture import GaussianMixture

HERE = os.path.dirname(os.path.abspath(__file__))


def make(name, N, D, K, iters, seed, covariance_type="full"):
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-4, 4, size=(K, D))
    comp = rng.integers(0, K, size=N)
    A = rng.normal(size=(K, D, D)) / np.sqrt(D)
    X = centers[comp] + np.einsum("nij,nj->ni", A[comp], rng.normal(size=(N, D))) + 0.2 * rng.normal(size=(N, D))
    S = np.cov(X.T, bias=True).reshape(D, D)
    reg = 1e-6 * np.trace(S) / D
    rows = rng.choice(N, size=K, replace=False)
    w0 = np.full(K, 1.0 / K)
    mu0 = X[rows].copy()
    cov0 = np.repeat((S + reg * np.eye(D))[None], K, axis=0)
    if covariance_type == "diag":
        cov0 = np.repeat(np.diag(np.diag(S) + reg)[None], K, axis=0)
        prec0 = 1.0 / np.diagonal(cov0, axis1=1, axis2=2)
    else:
        prec0 = np.linalg.inv(cov0)
    gm = GaussianMixture(n_components=K, covariance_type=covariance_type, tol=0.0, max_iter=iters, reg_covar=reg,
                         weights_init=w0, means_init=mu0, precisions_init=prec0, n_init=1)
    gm.fit(X)
    np.savez_compressed(os.path.join(HERE, name), X=X, w0=w0, mu0=mu0, cov0=cov0, reg=reg, iters=iters,
                        weights=gm.weights_, means=gm.means_,
                        covariances=(np.array([np.diag(c) for c in gm.covariances_]) if covariance_type == "diag"
                                     else gm.covariances_), covariance_type=covariance_type,
                        lower_bounds=np.array(gm.lower_bounds_), score=gm.score_samples(X),
                        predict=gm.predict(X), sklearn_version=sklearn.__version__)


if __name__ == "__main__":
    make("sklearn_d3k3.npz", 3000, 3, 3, 25, 11)
    make("sklearn_d8k4.npz", 2000, 8, 4, 15, 12)
    make("sklearn_diag_d6k5.npz", 3000, 6, 5, 20, 13, covariance_type="diag")
    print("ok")
