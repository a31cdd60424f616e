"""paper_2005_09148_b200 — Python binding of liboocgb.so, the B200 (sm_100a) hot path of
"Out-of-Core GPU Gradient Boosting" (R. Ou, arXiv 2005.09148).

Argument marshalling only: every step of the path runs in the CUDA library behind the C ABI
declared in include/oocgb.h.  Names follow that header:
  Context.quantise / Data.set_gradients / Data.sample / Data.build_tree / Data.predict ...
Arrays may be numpy arrays (host) or torch tensors (host or CUDA); CUDA tensors are passed
as device pointers without copies.  There is NO CPU fallback: importing this package on a
machine where liboocgb.so is missing raises, and every call on a box without a GPU fails
with OocgbError(ERR_DEVICE).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboocgb.so")

OK, ERR_ARG, ERR_NOMEM, ERR_DEVICE, ERR_STATE = 0, 2, 3, 4, 5
PLACE_DEVICE, PLACE_PINNED_HOST = 0, 1
SAMPLE_NONE, SAMPLE_UNIFORM, SAMPLE_MVS, SAMPLE_GOSS = 0, 1, 2, 3

# Every symbol include/oocgb.h declares (tests check the library exports all of them).
ABI_SYMBOLS = (
    "oocgb_nccl_unique_id", "oocgb_ctx_create", "oocgb_ctx_destroy", "oocgb_quantise",
    "oocgb_sketch_begin", "oocgb_sketch_push", "oocgb_cuts_finalize", "oocgb_pages_push",
    "oocgb_quantise_like", "oocgb_data_info", "oocgb_data_destroy", "oocgb_set_gradients",
    "oocgb_set_logistic_gradients", "oocgb_sample", "oocgb_build_tree", "oocgb_tree_export",
    "oocgb_tree_destroy", "oocgb_predict", "oocgb_update_margin", "oocgb_get_cuts",
    "oocgb_get_bins", "oocgb_get_sample", "oocgb_get_histogram", "oocgb_get_partition", "oocgb_get_row_order",
    "oocgb_get_timings", "oocgb_set_profiling", "oocgb_last_error", "oocgb_abi_version",
    "oocgb_ctx_create_hostcomm", "oocgb_sample_goss", "oocgb_set_streaming", "oocgb_quantise_csr",
)

COLLECTIVE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64,
                                 ctypes.c_void_p)


class OocgbError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[oocgb status {status}] {msg}")
        self.status = status


class Node(ctypes.Structure):
    _fields_ = [("feature", ctypes.c_int32), ("split_bin", ctypes.c_int32),
                ("split_value", ctypes.c_float), ("leaf_value", ctypes.c_float),
                ("gain", ctypes.c_double), ("sum_g", ctypes.c_double), ("sum_h", ctypes.c_double),
                ("n_rows", ctypes.c_int64), ("default_left", ctypes.c_int32), ("pad", ctypes.c_int32)]


NODE_DTYPE = np.dtype([("feature", np.int32), ("split_bin", np.int32), ("split_value", np.float32),
                       ("leaf_value", np.float32), ("gain", np.float64), ("sum_g", np.float64),
                       ("sum_h", np.float64), ("n_rows", np.int64), ("default_left", np.int32),
                       ("pad", np.int32)])


class Info(ctypes.Structure):
    _fields_ = [("n_rows_local", ctypes.c_int64), ("n_rows_global", ctypes.c_int64),
                ("row0_global", ctypes.c_int64), ("n_features", ctypes.c_int32),
                ("row_stride", ctypes.c_int32), ("max_bin", ctypes.c_int32),
                ("placement", ctypes.c_int32), ("n_pages", ctypes.c_int64),
                ("rows_per_page", ctypes.c_int64), ("total_cuts", ctypes.c_int64),
                ("has_missing", ctypes.c_int32), ("pad", ctypes.c_int32)]


class SampleInfo(ctypes.Structure):
    _fields_ = [("n_selected_local", ctypes.c_int64), ("n_selected_global", ctypes.c_int64),
                ("k_star", ctypes.c_int64), ("mu", ctypes.c_double), ("e_g", ctypes.c_int32),
                ("e_h", ctypes.c_int32), ("e_prime", ctypes.c_int32),
                ("fallback_uniform", ctypes.c_int32)]


_lib = None


def load_library():
    """Load liboocgb.so (built by __graft_entry__.build()).  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                          " — there is no CPU fallback")
    try:  # torch first: the library dlopen()s libnccl.so.2 and must bind to torch's copy (a system
        import torch  # noqa: F401  NCCL loaded first would shadow torch's bundled one)
    except ImportError:
        pass
    L = ctypes.CDLL(LIB_PATH)
    p, i32, i64, u64, d = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
    sig = {
        "oocgb_nccl_unique_id": [p],
        "oocgb_ctx_create": [i32, i32, i32, p, u64, p],
        "oocgb_ctx_destroy": [p],
        "oocgb_quantise": [p, p, i64, i64, i64, i32, i32, i64, i32, u64, p],
        "oocgb_sketch_begin": [p, i32, i32, i64, i64, i64, i64, i32, u64, p],
        "oocgb_sketch_push": [p, p, i64, i64],
        "oocgb_cuts_finalize": [p],
        "oocgb_pages_push": [p, p, i64, i64],
        "oocgb_quantise_like": [p, p, i64, i32, p],
        "oocgb_data_info": [p, p],
        "oocgb_data_destroy": [p],
        "oocgb_set_gradients": [p, p, p, i64],
        "oocgb_set_logistic_gradients": [p, p, p, i64],
        "oocgb_sample": [p, i32, d, d, u64, u64, i32, p],
        "oocgb_build_tree": [p, i32, d, d, d, d, i32, p],
        "oocgb_tree_export": [p, p, i32, p],
        "oocgb_tree_destroy": [p],
        "oocgb_predict": [p, p, i32, p],
        "oocgb_update_margin": [p, p, p],
        "oocgb_get_cuts": [p, p, p],
        "oocgb_get_bins": [p, i64, i64, p],
        "oocgb_get_sample": [p, p, p, p],
        "oocgb_get_histogram": [p, i32, p],
        "oocgb_get_partition": [p, p],
        "oocgb_get_row_order": [p, p],
        "oocgb_get_timings": [p, p, i32],
        "oocgb_set_profiling": [p, i32],
        "oocgb_ctx_create_hostcomm": [i32, i32, i32, COLLECTIVE_FN, p, u64, p],
        "oocgb_sample_goss": [p, d, d, u64, u64, i32, p],
        "oocgb_set_streaming": [p, i32],
        "oocgb_quantise_csr": [p, p, p, p, i64, i64, i64, i32, i32, i64, i32, u64, p],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.oocgb_last_error.argtypes = []
    L.oocgb_last_error.restype = ctypes.c_char_p
    L.oocgb_abi_version.argtypes = []
    L.oocgb_abi_version.restype = ctypes.c_int32
    _lib = L
    return L


def _check(rc: int):
    if rc != OK:
        raise OocgbError(rc, load_library().oocgb_last_error().decode(errors="replace"))


def _ptr(a, dtype=None):
    """(pointer, keepalive) of a numpy array or torch tensor (host or device, contiguous)."""
    if a is None:
        return None, None
    mod = type(a).__module__
    if mod.startswith("torch"):
        if not a.is_contiguous():
            a = a.contiguous()
        return ctypes.c_void_p(a.data_ptr()), a
    arr = np.ascontiguousarray(a, dtype=dtype) if dtype is not None else np.ascontiguousarray(a)
    return arr.ctypes.data_as(ctypes.c_void_p), arr


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(load_library().oocgb_nccl_unique_id(buf))
    return bytes(buf)


class Context:
    """One per process == one GPU (oocgb_ctx_create)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 stream: int = 0, host_collective=None):
        """host_collective: optional Python callable(op, np_array) performing the exchange in place
        (test transport, see oocgb_ctx_create_hostcomm); otherwise NCCL when world > 1."""
        L = load_library()
        h = ctypes.c_void_p()
        self._cb = None
        if host_collective is not None:
            dtypes = {0: np.int64, 1: np.uint64, 2: np.uint32}

            def _cb(op, dtype, buf, count, user):
                try:
                    n = count * (world if op == 2 else 1)
                    arr = np.ctypeslib.as_array(ctypes.cast(buf, ctypes.POINTER(ctypes.c_uint8)),
                                                shape=(n * np.dtype(dtypes[dtype]).itemsize,)).view(dtypes[dtype])
                    host_collective(op, arr)
                    return 0
                except Exception as e:  # pragma: no cover - reported through the status code
                    print("host collective failed:", e)
                    return 1

            self._cb = COLLECTIVE_FN(_cb)
            _check(L.oocgb_ctx_create_hostcomm(device, rank, world, self._cb, None, stream, ctypes.byref(h)))
        else:
            idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id is not None else None
            _check(L.oocgb_ctx_create(device, rank, world, idbuf, stream, ctypes.byref(h)))
        self._h = h
        self.device, self.rank, self.world = device, rank, world

    def close(self):
        if getattr(self, "_h", None):
            _check(load_library().oocgb_ctx_destroy(self._h))
            self._h = None

    # Alg. 2 + Alg. 4/5
    def quantise(self, X, max_bin: int = 256, *, row0_global: int = 0, n_rows_global: int | None = None,
                 page_bytes: int = 0, placement: int = PLACE_DEVICE, seed: int = 2) -> "Data":
        n, m = int(X.shape[0]), int(X.shape[1])
        px, keep = _ptr(X, np.float32)
        h = ctypes.c_void_p()
        _check(load_library().oocgb_quantise(self._h, px, n, row0_global,
                                              n if n_rows_global is None else n_rows_global, m, max_bin,
                                              page_bytes, placement, seed, ctypes.byref(h)))
        return Data(self, h)

    def quantise_csr(self, indptr, indices, values, n_features: int, max_bin: int = 255, *, row0_global: int = 0,
                     n_rows_global: int | None = None, page_bytes: int = 0, placement: int = PLACE_DEVICE,
                     seed: int = 2) -> "Data":
        """Sparse CSR rows (R27): absent entries are missing values (symbol 255, max_bin <= 255)."""
        pp, k1 = _ptr(indptr, np.int64)
        pi, k2 = _ptr(indices, np.int32)
        pv, k3 = _ptr(values, np.float32)
        n = int(indptr.shape[0]) - 1
        h = ctypes.c_void_p()
        _check(load_library().oocgb_quantise_csr(self._h, pp, pi, pv, n, row0_global,
                                                  n if n_rows_global is None else n_rows_global, n_features,
                                                  max_bin, page_bytes, placement, seed, ctypes.byref(h)))
        return Data(self, h)

    # Alg. 3 + Alg. 5, streamed
    def sketch_begin(self, n_features: int, max_bin: int, n_rows: int, *, row0_global: int = 0,
                     n_rows_global: int | None = None, page_bytes: int = 0, placement: int = PLACE_DEVICE,
                     seed: int = 2) -> "Data":
        h = ctypes.c_void_p()
        _check(load_library().oocgb_sketch_begin(self._h, n_features, max_bin, n_rows, row0_global,
                                                  n_rows if n_rows_global is None else n_rows_global,
                                                  page_bytes, placement, seed, ctypes.byref(h)))
        return Data(self, h)

    def set_profiling(self, enable: bool):
        _check(load_library().oocgb_set_profiling(self._h, int(enable)))

    def get_timings(self) -> dict:
        out = (ctypes.c_double * 16)()
        _check(load_library().oocgb_get_timings(self._h, out, 16))
        keys = ["hist_ms", "eval_ms", "partition_ms", "sample_ms", "predict_ms", "h2d_ms", "build_ms",
                "hist_launches", "hist_bytes", "graph_captures"]
        return {k: out[i] for i, k in enumerate(keys)}


class Data:
    """Cuts + ELLPACK pages + per-round row state (oocgb_data)."""

    def __init__(self, ctx: Context, h):
        self.ctx = ctx
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _check(load_library().oocgb_data_destroy(self._h))
            self._h = None

    def info(self) -> dict:
        i = Info()
        _check(load_library().oocgb_data_info(self._h, ctypes.byref(i)))
        return {k: getattr(i, k) for k, _ in Info._fields_}

    def sketch_push(self, X, row0_global: int):
        px, keep = _ptr(X, np.float32)
        _check(load_library().oocgb_sketch_push(self._h, px, row0_global, int(X.shape[0])))

    def cuts_finalize(self):
        _check(load_library().oocgb_cuts_finalize(self._h))

    def pages_push(self, X, row0_global: int):
        px, keep = _ptr(X, np.float32)
        _check(load_library().oocgb_pages_push(self._h, px, row0_global, int(X.shape[0])))

    def quantise_like(self, X, placement: int = PLACE_DEVICE) -> "Data":
        px, keep = _ptr(X, np.float32)
        h = ctypes.c_void_p()
        _check(load_library().oocgb_quantise_like(self._h, px, int(X.shape[0]), placement, ctypes.byref(h)))
        return Data(self.ctx, h)

    def set_gradients(self, g, h):
        pg, kg = _ptr(g, np.float32)
        ph, kh = _ptr(h, np.float32)
        _check(load_library().oocgb_set_gradients(self._h, pg, ph, int(g.shape[0])))

    def set_logistic_gradients(self, margin, labels):
        pm, km = _ptr(margin, np.float32)
        py, ky = _ptr(labels, np.float32)
        _check(load_library().oocgb_set_logistic_gradients(self._h, pm, py, int(margin.shape[0])))

    def sample(self, mode: int = SAMPLE_NONE, ratio: float = 1.0, mvs_lambda: float = 1.0, seed: int = 1,
               round: int = 0, quant_bits: int = 16, want_info: bool = True):
        """Sample(g) + fixed point.  want_info=False skips the host synchronisation (returns None)."""
        if not want_info:
            _check(load_library().oocgb_sample(self._h, mode, ratio, mvs_lambda, seed, round, quant_bits, None))
            return None
        si = SampleInfo()
        _check(load_library().oocgb_sample(self._h, mode, ratio, mvs_lambda, seed, round, quant_bits,
                                            ctypes.byref(si)))
        return {k: getattr(si, k) for k, _ in SampleInfo._fields_}

    def set_streaming(self, enable: bool = True):
        """Alg. 6: build f = 1 trees by streaming the pinned pages once per level (PINNED_HOST)."""
        _check(load_library().oocgb_set_streaming(self._h, int(enable)))

    def sample_goss(self, a: float, b: float, seed: int = 1, round: int = 0, quant_bits: int = 16) -> dict:
        """GOSS: top round(a n) by |g| with p = 1, the rest Bernoulli(b / (1 - a)), scale 1/p."""
        si = SampleInfo()
        _check(load_library().oocgb_sample_goss(self._h, a, b, seed, round, quant_bits, ctypes.byref(si)))
        return {k: getattr(si, k) for k, _ in SampleInfo._fields_}

    def build_tree(self, max_depth: int = 8, lam: float = 1.0, gamma: float = 0.0,
                   min_child_weight: float = 1.0, eta: float = 0.1, keep_debug: bool = False) -> "Tree":
        h = ctypes.c_void_p()
        _check(load_library().oocgb_build_tree(self._h, max_depth, lam, gamma, min_child_weight, eta,
                                                int(keep_debug), ctypes.byref(h)))
        return Tree(self, h, max_depth)

    def predict(self, trees, margin):
        """margin (float32 [n_local], numpy or torch, host or CUDA) += sum of tree leaves; in place."""
        trees = list(trees)
        arr = (ctypes.c_void_p * max(1, len(trees)))(*[t._h for t in trees])
        pm, km = _ptr(margin, np.float32)
        _check(load_library().oocgb_predict(self._h, arr, len(trees), pm))
        if km is not margin and isinstance(margin, np.ndarray):
            margin[...] = km
        return margin

    def update_margin(self, tree: "Tree", margin):
        pm, km = _ptr(margin, np.float32)
        _check(load_library().oocgb_update_margin(self._h, tree._h, pm))
        if km is not margin and isinstance(margin, np.ndarray):
            margin[...] = km
        return margin

    def get_cuts(self):
        info = self.info()
        vals = np.zeros(max(1, info["total_cuts"]), np.float32)
        ptrs = np.zeros(info["n_features"] + 1, np.int32)
        _check(load_library().oocgb_get_cuts(self._h, vals.ctypes.data_as(ctypes.c_void_p),
                                              ptrs.ctypes.data_as(ctypes.c_void_p)))
        return vals[: info["total_cuts"]], ptrs

    def get_bins(self, row0: int = 0, n: int | None = None) -> np.ndarray:
        info = self.info()
        if n is None:
            n = info["n_rows_local"] - row0
        out = np.zeros((n, info["row_stride"]), np.uint8)
        _check(load_library().oocgb_get_bins(self._h, row0, n, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def get_sample(self, n_selected_local: int):
        gid = np.zeros(n_selected_local, np.int64)
        qg = np.zeros(n_selected_local, np.int64)
        qh = np.zeros(n_selected_local, np.int64)
        _check(load_library().oocgb_get_sample(self._h, gid.ctypes.data_as(ctypes.c_void_p),
                                                qg.ctypes.data_as(ctypes.c_void_p),
                                                qh.ctypes.data_as(ctypes.c_void_p)))
        return gid, qg, qh


class Tree:
    def __init__(self, data: Data, h, max_depth: int):
        self.data = data
        self._h = h
        self.max_depth = max_depth

    def close(self):
        if getattr(self, "_h", None):
            _check(load_library().oocgb_tree_destroy(self._h))
            self._h = None

    def export(self) -> np.ndarray:
        n = ctypes.c_int32()
        _check(load_library().oocgb_tree_export(self._h, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value, NODE_DTYPE)
        _check(load_library().oocgb_tree_export(self._h, out.ctypes.data_as(ctypes.c_void_p), n.value,
                                                 ctypes.byref(n)))
        return out

    def get_histogram(self, node: int) -> np.ndarray:
        m = self.data.info()["n_features"]
        out = np.zeros((m, 256, 2), np.int64)
        _check(load_library().oocgb_get_histogram(self._h, node, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def get_row_order(self, n_selected_local: int) -> np.ndarray:
        """Final partition, position -> selected-row index (stable: ascending inside each leaf)."""
        out = np.zeros(n_selected_local, np.int32)
        _check(load_library().oocgb_get_row_order(self._h, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def get_partition(self, n_selected_local: int) -> np.ndarray:
        out = np.zeros(n_selected_local, np.int32)
        _check(load_library().oocgb_get_partition(self._h, out.ctypes.data_as(ctypes.c_void_p)))
        return out
