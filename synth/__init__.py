"""Seeded synthetic input generators shared by the oracle tests, the GPU parity tests and
bench.py.  This module holds NONE of the method's arithmetic (no binning, sampling, fixed
point, histogram or split logic) — only data shaped like the paper's workloads.

Recipe: the paper's synthetic data is "generated using Scikit-learn"
(Table 1, 500 columns); we use ``sklearn.datasets.make_classification`` with
its defaults (n_informative=2, n_redundant=2, n_clusters_per_class=2, flip_y=0.01,
class_sep=1.0, shuffle=True), float32 features, {0,1} labels.  The "stress" variant replaces
25% of the columns by low-cardinality features (2..8 distinct values) to exercise atomic
contention and the D_j <= max_bin cut rule.
"""
from __future__ import annotations

import numpy as np


def make_classification(n_rows: int, n_features: int, seed: int = 0, stress: bool = False,
                        dtype=np.float32):
    """Returns (X float32 [n, m] C-contiguous, y float32 [n])."""
    from sklearn.datasets import make_classification as _mc

    n_inf = min(2, n_features)
    n_red = min(2, max(0, n_features - n_inf))
    X, y = _mc(n_samples=n_rows, n_features=n_features, n_informative=n_inf,
               n_redundant=n_red, n_repeated=0, n_classes=2, n_clusters_per_class=min(2, 2 ** n_inf // 2),
               flip_y=0.01, class_sep=1.0, shuffle=True, random_state=seed)
    X = np.ascontiguousarray(X, dtype=dtype)
    if stress:
        rng = np.random.default_rng(seed + 1000)
        cols = rng.choice(n_features, size=max(1, n_features // 4), replace=False)
        for c in cols:
            k = int(rng.integers(2, 9))
            levels = np.sort(rng.normal(size=k)).astype(dtype)
            X[:, c] = levels[rng.integers(0, k, size=n_rows)]
    return X, np.ascontiguousarray(y, dtype=np.float32)


def fast_classification(n_rows: int, n_features: int, seed: int = 0):
    """A make_classification-shaped generator that is cheap at 10^6-10^7 rows (numpy
    vectorised, float32 throughout): 4 Gaussian clusters at the vertices of {+-1}^2 in the
    2 informative columns, 2 redundant linear combinations, the rest N(0,1) noise, 1% label
    flips, a fixed column permutation.  Same structure as sklearn's defaults (SURVEY.md
    §8(d) 'GPU generator'); used by bench.py for the 1M x 500 workload."""
    rng = np.random.default_rng(seed)
    n_inf = 2
    cluster = rng.integers(0, 4, size=n_rows)
    centroids = np.array([[-1, -1], [1, -1], [-1, 1], [1, 1]], np.float32)
    A = rng.uniform(-1, 1, size=(4, n_inf, n_inf)).astype(np.float32)
    z = rng.standard_normal((n_rows, n_inf), dtype=np.float32)
    x_inf = np.einsum("ni,nij->nj", z, A[cluster]) + centroids[cluster]
    B = rng.uniform(-1, 1, size=(n_inf, 2)).astype(np.float32)
    X = np.empty((n_rows, n_features), np.float32)
    X[:, 0:2] = x_inf
    if n_features > 2:
        X[:, 2:4] = (x_inf @ B)[:, : max(0, min(2, n_features - 2))]
    if n_features > 4:
        X[:, 4:] = rng.standard_normal((n_rows, n_features - 4), dtype=np.float32)
    y = (cluster % 2).astype(np.float32)
    flip = rng.random(n_rows) < 0.01
    y[flip] = rng.integers(0, 2, size=int(flip.sum())).astype(np.float32)
    perm = rng.permutation(n_features)
    X = np.ascontiguousarray(X[:, perm])
    return X, y


def gradient_pairs(n: int, seed: int = 0, kind: str = "logistic"):
    """Seeded (g, h) float32 vectors shaped like binary:logistic gradients at a random
    margin: g in (-1, 1), h in (0, 1/4].  kind='wide' draws heavy-tailed g (for MVS tests),
    kind='ties' draws from a handful of values (exercises equal-key handling)."""
    rng = np.random.default_rng(seed)
    if kind == "logistic":
        p = rng.uniform(0.02, 0.98, size=n)
        y = (rng.random(n) < 0.5).astype(np.float64)
        g = (p - y).astype(np.float32)
        h = (p * (1 - p)).astype(np.float32)
    elif kind == "wide":
        g = (rng.standard_cauchy(n) * 0.1).clip(-50, 50).astype(np.float32)
        h = rng.uniform(0.01, 1.0, size=n).astype(np.float32)
    elif kind == "ties":
        g = rng.choice(np.array([-0.5, -0.25, 0.0, 0.25, 0.5], np.float32), size=n)
        h = rng.choice(np.array([0.0, 0.125, 0.25], np.float32), size=n)
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(g), np.ascontiguousarray(h)


def labels_like(n: int, seed: int = 0):
    rng = np.random.default_rng(seed)
    return (rng.random(n) < 0.5).astype(np.float32)


def torch_classification_chunk(row0: int, n_rows: int, n_features: int, seed: int = 0, device="cuda"):
    """make_classification-shaped rows [row0, row0 + n_rows) generated on the GPU with torch, for
    the 10^7..10^8-row configurations (3, 4) where X is never materialised on the host.  The
    chunk's values depend only on (seed, row0, n_rows): regenerating a chunk gives identical
    data, so the two quantise passes (sketch, pages) see the same rows.  Structure as
    fast_classification: 4 clusters on {+-1}^2, 2 redundant combinations, N(0,1) noise,
    1% label flips, a fixed column permutation.  Returns (X float32 [n, m], y float32 [n])."""
    import torch

    g = torch.Generator(device="cpu").manual_seed(seed)
    A = torch.rand((4, 2, 2), generator=g) * 2 - 1
    Bm = torch.rand((2, 2), generator=g) * 2 - 1
    perm = torch.randperm(n_features, generator=g)
    gc = torch.Generator(device=device).manual_seed((seed * 1_000_003 + row0) % (2**63 - 1))
    cluster = torch.randint(0, 4, (n_rows,), generator=gc, device=device)
    centroids = torch.tensor([[-1, -1], [1, -1], [-1, 1], [1, 1]], dtype=torch.float32, device=device)
    z = torch.randn((n_rows, 2), generator=gc, device=device)
    x_inf = torch.einsum("ni,nij->nj", z, A.to(device)[cluster]) + centroids[cluster]
    X = torch.randn((n_rows, n_features), generator=gc, device=device)
    X[:, 0:2] = x_inf
    if n_features > 2:
        X[:, 2:4] = (x_inf @ Bm.to(device))[:, : max(0, min(2, n_features - 2))]
    y = (cluster % 2).to(torch.float32)
    flip = torch.rand((n_rows,), generator=gc, device=device) < 0.01
    y[flip] = torch.randint(0, 2, (int(flip.sum().item()),), generator=gc, device=device).to(torch.float32)
    X = X[:, perm.to(device)].contiguous()
    return X, y
