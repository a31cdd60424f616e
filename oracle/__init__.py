"""ctypes wrapper of the CPU ORACLE (oracle/oocgb_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this module.  The product package
(paper_2005_09148_b200/) never imports it and shares no code with it.

Every function below is argument marshalling around the C definitions; the arithmetic
lives in the C file, each function there citing PAPER.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oocgb_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboocgb_oracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=gnu11"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, -O2 -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _declare(_lib)
    return _lib


class OrcNode(ctypes.Structure):
    _fields_ = [
        ("feature", ctypes.c_int32),
        ("split_bin", ctypes.c_int32),
        ("split_value", ctypes.c_float),
        ("leaf_value", ctypes.c_float),
        ("gain", ctypes.c_double),
        ("sum_g", ctypes.c_double),
        ("sum_h", ctypes.c_double),
        ("n_rows", ctypes.c_int64),
        ("default_left", ctypes.c_int32),
        ("pad", ctypes.c_int32),
    ]


NODE_DTYPE = np.dtype([
    ("feature", np.int32), ("split_bin", np.int32), ("split_value", np.float32),
    ("leaf_value", np.float32), ("gain", np.float64), ("sum_g", np.float64),
    ("sum_h", np.float64), ("n_rows", np.int64), ("default_left", np.int32), ("pad", np.int32),
])
assert NODE_DTYPE.itemsize == ctypes.sizeof(OrcNode)

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_u64 = ctypes.c_uint64
_d = ctypes.c_double


def _declare(L):
    L.orc_philox4x64_10.argtypes = [_p, _p, _p]
    L.orc_philox4x64_10.restype = None
    L.orc_uniform.argtypes = [_u64, _u64, _u64, _u64]
    L.orc_uniform.restype = _d
    L.orc_sketch_row_selected.argtypes = [_i64, _u64, _i64]
    L.orc_sketch_row_selected.restype = ctypes.c_int
    L.orc_cuts.argtypes = [_p, _i64, _i32, _i32, _i64, _i64, _u64, _p, _p]
    L.orc_cuts.restype = ctypes.c_int
    L.orc_bins.argtypes = [_p, _i64, _i32, _p, _p, _i32, _p]
    L.orc_bins.restype = ctypes.c_int
    L.orc_sample.argtypes = [_p, _p, _i64, _i32, _d, _d, _u64, _u64, _p, _p, _p, _p, _p]
    L.orc_sample.restype = ctypes.c_int
    L.orc_sample_goss.argtypes = [_p, _p, _i64, _d, _d, _u64, _u64, _p, _p, _p, _p, _p]
    L.orc_sample_goss.restype = ctypes.c_int
    L.orc_quantise.argtypes = [_p, _i64, _i32, _p]
    L.orc_quantise.restype = ctypes.c_int
    L.orc_histogram.argtypes = [_p, _i32, _i32, _p, _i64, _p, _p, _p]
    L.orc_histogram.restype = None
    L.orc_build_tree.argtypes = [_p, _i32, _i32, _p, _p, _i64, _p, _p, _i32, _i32, _i32,
                                 _d, _d, _d, _d, _i32, _p, _p, _p]
    L.orc_build_tree.restype = ctypes.c_int
    L.orc_predict.argtypes = [_p, _i32, _i64, _p, _i32, _p]
    L.orc_predict.restype = None
    L.orc_logistic_grad.argtypes = [_p, _p, _i64, _p, _p]
    L.orc_logistic_grad.restype = None
    L.orc_auc_bruteforce.argtypes = [_p, _p, _i64]
    L.orc_auc_bruteforce.restype = _d


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class OracleError(RuntimeError):
    pass


# ---------------------------------------------------------------------------------------- O3
def philox4x64_10(ctr, key) -> np.ndarray:
    c = _c(ctr, np.uint64)
    k = _c(key, np.uint64)
    out = np.zeros(4, np.uint64)
    lib().orc_philox4x64_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def uniform(seed: int, round_: int, row: int, stream: int) -> float:
    return lib().orc_uniform(seed, round_, row, stream)


# ---------------------------------------------------------------------------------------- O1
def cuts(X: np.ndarray, max_bin: int = 256, seed: int = 2, row0: int = 0, n_global: int | None = None):
    """O1: returns (cut_values float32 [sum B_j], cut_ptrs int32 [m+1])."""
    X = _c(X, np.float32)
    n, m = X.shape
    if n_global is None:
        n_global = n
    vals = np.zeros(max(1, m * max_bin), np.float32)
    ptrs = np.zeros(m + 1, np.int32)
    rc = lib().orc_cuts(_ptr(X), n, m, max_bin, row0, n_global, seed, _ptr(vals), _ptr(ptrs))
    if rc != 0:
        raise OracleError(f"orc_cuts rc={rc}")
    return vals[: ptrs[-1]].copy(), ptrs


def stride_of(m: int) -> int:
    """R5: bytes per ELLPACK row = 32 * ceil(m / 32) (feature groups of 32), pad bytes 0."""
    return (m + 31) // 32 * 32


# ---------------------------------------------------------------------------------------- O2
def bins(X: np.ndarray, cut_values: np.ndarray, cut_ptrs: np.ndarray) -> np.ndarray:
    """O2: uint8 ELLPACK rows [n][stride]."""
    X = _c(X, np.float32)
    n, m = X.shape
    s = stride_of(m)
    out = np.zeros((n, s), np.uint8)
    cv = _c(cut_values, np.float32)
    cp = _c(cut_ptrs, np.int32)
    rc = lib().orc_bins(_ptr(X), n, m, _ptr(cv), _ptr(cp), s, _ptr(out))
    if rc != 0:
        raise OracleError(f"orc_bins rc={rc}")
    return out


# ---------------------------------------------------------------------------------------- O4
SAMPLE_NONE, SAMPLE_UNIFORM, SAMPLE_MVS = 0, 1, 2


def sample(g, h, mode: int, ratio: float, mvs_lambda: float = 1.0, seed: int = 1, round_: int = 0):
    """O4: returns dict(selected uint8[n], p f64[n], gs f64[n], hs f64[n], n_selected, k_star, mu, e_prime)."""
    g = _c(g, np.float32)
    h = _c(h, np.float32)
    n = g.shape[0]
    sel = np.zeros(n, np.uint8)
    p = np.zeros(n, np.float64)
    gs = np.zeros(n, np.float64)
    hs = np.zeros(n, np.float64)
    info = np.zeros(4, np.float64)
    rc = lib().orc_sample(_ptr(g), _ptr(h), n, mode, ratio, mvs_lambda, seed, round_,
                          _ptr(sel), _ptr(p), _ptr(gs), _ptr(hs), _ptr(info))
    if rc != 0:
        raise OracleError(f"orc_sample rc={rc}")
    return dict(selected=sel, p=p, gs=gs, hs=hs, n_selected=int(info[0]), k_star=int(info[1]),
                mu=float(info[2]), e_prime=int(info[3]))


def sample_goss(g, h, a: float, b: float, seed: int = 1, round_: int = 0):
    """O4b GOSS: returns dict(selected, p, gs, hs, n_selected, k_a, t, e_prime)."""
    g = _c(g, np.float32)
    h = _c(h, np.float32)
    n = g.shape[0]
    sel = np.zeros(n, np.uint8)
    p = np.zeros(n, np.float64)
    gs = np.zeros(n, np.float64)
    hs = np.zeros(n, np.float64)
    info = np.zeros(4, np.float64)
    rc = lib().orc_sample_goss(_ptr(g), _ptr(h), n, a, b, seed, round_, _ptr(sel), _ptr(p), _ptr(gs), _ptr(hs),
                               _ptr(info))
    if rc != 0:
        raise OracleError(f"orc_sample_goss rc={rc}")
    return dict(selected=sel, p=p, gs=gs, hs=hs, n_selected=int(info[0]), k_a=int(info[1]), t=float(info[2]),
                e_prime=int(info[3]))


# ---------------------------------------------------------------------------------------- O5
def quantise(x, P: int = 16):
    """O5: returns (q int64[n], e)."""
    x = _c(x, np.float64)
    q = np.zeros(x.shape[0], np.int64)
    e = lib().orc_quantise(_ptr(x), x.shape[0], P, _ptr(q))
    return q, int(e)


# ---------------------------------------------------------------------------------------- O6
def histogram(bins_: np.ndarray, m: int, rows, qg, qh) -> np.ndarray:
    """O6: int64 [m][256][2] over the listed rows."""
    b = _c(bins_, np.uint8)
    rows = _c(rows, np.int64)
    qg = _c(qg, np.int64)
    qh = _c(qh, np.int64)
    out = np.zeros((m, 256, 2), np.int64)
    lib().orc_histogram(_ptr(b), b.shape[1], m, _ptr(rows), rows.shape[0], _ptr(qg), _ptr(qh), _ptr(out))
    return out


# ---------------------------------------------------------------------------------------- O7-O10
def build_tree(bins_: np.ndarray, m: int, cut_values, cut_ptrs, qg, qh, e_g: int, e_h: int,
               max_depth: int = 6, lam: float = 1.0, gamma: float = 0.0, mcw: float = 1.0,
               eta: float = 0.1, want_hist: bool = False, has_missing: bool = False):
    """O6-O10 on the selected rows (bins_ holds only the selected rows, in ascending global
    order).  has_missing (R27): symbol 255 is a missing value and every candidate is tried with
    the missing rows on either side.  Returns (nodes, leaf_of_row int32[n_sel], hist or None)."""
    b = _c(bins_, np.uint8)
    n_sel = b.shape[0]
    cv = _c(cut_values, np.float32)
    cp = _c(cut_ptrs, np.int32)
    qg = _c(qg, np.int64)
    qh = _c(qh, np.int64)
    n_nodes = (1 << (max_depth + 1)) - 1
    nodes = np.zeros(n_nodes, NODE_DTYPE)
    lor = np.full(n_sel, -1, np.int32)
    hist = np.zeros(((1 << max_depth) - 1, m, 256, 2), np.int64) if want_hist else None
    rc = lib().orc_build_tree(_ptr(b), b.shape[1], m, _ptr(cp), _ptr(cv), n_sel, _ptr(qg), _ptr(qh),
                              e_g, e_h, max_depth, lam, gamma, mcw, eta, int(has_missing), _ptr(nodes), _ptr(lor),
                              _ptr(hist) if want_hist else None)
    if rc != 0:
        raise OracleError(f"orc_build_tree rc={rc}")
    return nodes, lor, hist


# ---------------------------------------------------------------------------------------- O11-O12
def predict(bins_: np.ndarray, nodes: np.ndarray, margin: np.ndarray, has_missing: bool = False) -> np.ndarray:
    b = _c(bins_, np.uint8)
    out = _c(margin, np.float32).copy()
    nd = np.ascontiguousarray(nodes, dtype=NODE_DTYPE)
    lib().orc_predict(_ptr(b), b.shape[1], b.shape[0], _ptr(nd), int(has_missing), _ptr(out))
    return out


def logistic_grad(margin, y):
    margin = _c(margin, np.float32)
    y = _c(y, np.float32)
    g = np.zeros_like(margin)
    h = np.zeros_like(margin)
    lib().orc_logistic_grad(_ptr(margin), _ptr(y), margin.shape[0], _ptr(g), _ptr(h))
    return g, h


def auc_bruteforce(score, y) -> float:
    s = _c(score, np.float32)
    y = _c(y, np.float32)
    return lib().orc_auc_bruteforce(_ptr(s), _ptr(y), s.shape[0])


# ---------------------------------------------------------------------------------------- one round
def boosting_round(bins_: np.ndarray, m: int, cut_values, cut_ptrs, margin, y, *, mode=SAMPLE_NONE,
                   ratio=1.0, mvs_lambda=1.0, seed=1, round_=0, max_depth=8, lam=1.0, gamma=0.0,
                   mcw=1.0, eta=0.1, quant_bits=16, prev_tree=None, has_missing=False):
    """One boosting round exactly as the product path runs it (SURVEY.md §3 stack 2):
    predict(tree_{t-1}) -> logistic gradients -> Sample -> fixed point -> BuildTree.
    Returns (tree nodes, new margin, sample dict)."""
    if prev_tree is not None:
        margin = predict(bins_, prev_tree, margin, has_missing)
    g, h = logistic_grad(margin, y)
    s = sample(g, h, mode, ratio, mvs_lambda, seed, round_)
    sel = s["selected"].astype(bool)
    qg, e_g = quantise(s["gs"][sel], quant_bits)
    qh, e_h = quantise(s["hs"][sel], quant_bits)
    nodes, lor, _ = build_tree(bins_[sel], m, cut_values, cut_ptrs, qg, qh, e_g, e_h, max_depth,
                               lam, gamma, mcw, eta, has_missing=has_missing)
    return nodes, margin, dict(s, e_g=e_g, e_h=e_h, qg=qg, qh=qh, leaf_of_row=lor)
