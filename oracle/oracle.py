"""TEST INFRASTRUCTURE — ctypes bindings for the two CPU checkers.

* ``Oracle``: the C restatement (oracle/sgnn_oracle.c -> oracle/liboracle.so).
* ``RefEngine``: the unmodified reference engine compiled from /root/reference
  (oracle/ref.mk -> oracle/_ref/libstreamgnn_ref.so), when it was built.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module. The product never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import model_io

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libstreamgnn_ref.so")

COUNTERS = ["events", "targets", "user_targets", "no_deletion", "deletion_no_effect",
            "covered_reset", "exposed_reset", "recomputes", "dirty", "fetch_rows"]

_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")


class _OrcOp(C.Structure):
    _fields_ = [("kind", C.c_int), ("w", C.c_void_p), ("rows", C.c_uint32), ("cols", C.c_uint32),
                ("bias", C.c_void_p), ("eps", C.c_float)]


def _load(path):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built (run python -c 'import __graft_entry__ as g; g.build()')")
    return C.CDLL(path)


_orc = None


def orc_lib():
    global _orc
    if _orc is None:
        lib = _load(ORACLE_SO)
        lib.orc_create.restype = C.c_void_p
        lib.orc_create.argtypes = [C.c_uint32, _u32p, _u32p, C.c_uint64, _f32p, C.c_uint32, C.c_void_p, C.c_int,
                                   C.c_int, C.POINTER(C.c_int)]
        lib.orc_destroy.argtypes = [C.c_void_p]
        lib.orc_set_option.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        lib.orc_num_layers.argtypes = [C.c_void_p]
        lib.orc_apply.argtypes = [C.c_void_p, C.c_char_p, _u32p, _u32p, C.c_size_t]
        lib.orc_last_error.restype = C.c_char_p
        lib.orc_last_stats.argtypes = [C.c_void_p, np.ctypeslib.ndpointer(dtype=np.uint64)]
        lib.orc_dim.restype = C.c_uint32
        lib.orc_dim.argtypes = [C.c_void_p, C.c_int, C.c_int]
        lib.orc_table.argtypes = [C.c_void_p, C.c_int, C.c_int, _f32p]
        lib.orc_dirty.restype = C.c_uint64
        lib.orc_dirty.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64]
        lib.orc_num_edges.restype = C.c_uint64
        lib.orc_num_edges.argtypes = [C.c_void_p]
        P = C.POINTER(C.c_uint32)
        lib.orc_verify.argtypes = [C.c_void_p, P, P, P, P]
        lib.orc_classify.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_int]
        lib.orc_matvec_affine.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]
        _orc = lib
    return _orc


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def format_stats_line(counters: np.ndarray, k: int, round_index: int) -> str:
    """RoundStats::to_line (proj/src/core/stats.cpp:20-48) from oracle counters."""
    per = counters[: k * len(COUNTERS)].reshape(k, len(COUNTERS))
    tail = counters[k * len(COUNTERS):]
    tot = per.sum(axis=0)
    s = (f"round={round_index} updates={tail[0]} layers={k} events={tot[0]} targets={tot[1]} "
         f"user_targets={tot[2]} no_deletion={tot[3]} deletion_no_effect={tot[4]} covered_reset={tot[5]} "
         f"exposed_reset={tot[6]} recomputes={tot[7]} dirty={tot[8]} ckpt_fetches={tail[1]} "
         f"feat_fetches={tail[2]}")
    if tail[3]:
        s += f" affected_fetches={tail[4]} full_fetches={tail[5]} area_nodes={tail[6]}"
    for i in range(k):
        p = f"l{i + 1}."
        s += "".join(f" {p}{name}={per[i][j]}" for j, name in enumerate(COUNTERS))
    return s


class Oracle:
    """CPU restatement engine (oracle/sgnn_oracle.c)."""

    def __init__(self, num_nodes, src, dst, features, model: model_io.ParsedModel):
        lib = orc_lib()
        self.lib = lib
        src = np.ascontiguousarray(src, dtype=np.uint32)
        dst = np.ascontiguousarray(dst, dtype=np.uint32)
        feats = np.ascontiguousarray(features, dtype=np.float32)
        ops = model.oracle_ops()
        self._keep = []
        arr = (_OrcOp * max(1, len(ops)))()
        for i, (kind, w, b, eps) in enumerate(ops):
            arr[i].kind = kind
            arr[i].eps = float(eps)
            if w is not None:
                w = np.ascontiguousarray(w, dtype=np.float32)
                self._keep.append(w)
                arr[i].w = w.ctypes.data
                arr[i].rows, arr[i].cols = w.shape
            if b is not None:
                b = np.ascontiguousarray(b, dtype=np.float32)
                self._keep.append(b)
                arr[i].bias = b.ctypes.data
        self._ops = arr
        st = C.c_int(0)
        self.h = lib.orc_create(num_nodes, src, dst, len(src), feats, feats.shape[1], C.cast(arr, C.c_void_p),
                                len(ops), int(model.is_max), C.byref(st))
        if not self.h:
            raise RuntimeError(f"oracle create failed ({st.value}): {lib.orc_last_error().decode()}")
        self.k = lib.orc_num_layers(self.h)
        self.rounds = 0

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_destroy(self.h)
            self.h = None

    def set_option(self, name: str, value: int) -> int:
        return self.lib.orc_set_option(self.h, name.encode(), value)

    def apply(self, ops: bytes, src, dst) -> int:
        src = np.ascontiguousarray(src, dtype=np.uint32)
        dst = np.ascontiguousarray(dst, dtype=np.uint32)
        st = self.lib.orc_apply(self.h, ops, src, dst, len(src))
        if st == 0:
            self.rounds += 1
        return st

    def last_error(self) -> str:
        return self.lib.orc_last_error().decode()

    def counters(self) -> np.ndarray:
        out = np.zeros(self.k * len(COUNTERS) + 7, dtype=np.uint64)
        self.lib.orc_last_stats(self.h, out)
        return out

    def stats_line(self) -> str:
        return format_stats_line(self.counters(), self.k, self.rounds - 1)

    def table(self, layer: int, stage: int) -> np.ndarray:
        d = self.lib.orc_dim(self.h, layer, stage)
        n = self.num_nodes
        out = np.empty((n, d), dtype=np.float32)
        self.lib.orc_table(self.h, layer, stage, out)
        return out

    @property
    def num_nodes(self) -> int:
        return self._n

    @num_nodes.setter
    def num_nodes(self, v):
        self._n = v

    def dirty(self, layer: int) -> np.ndarray:
        n = self.lib.orc_dirty(self.h, layer, None, 0)
        out = np.empty(n, dtype=np.uint32)
        self.lib.orc_dirty(self.h, layer, _ptr(out), n)
        return out

    def num_edges(self) -> int:
        return self.lib.orc_num_edges(self.h)

    def verify(self):
        vals = [C.c_uint32(0) for _ in range(4)]
        rc = self.lib.orc_verify(self.h, *[C.byref(v) for v in vals])
        return rc, tuple(v.value for v in vals)


def make_oracle(num_nodes, src, dst, features, model) -> Oracle:
    o = Oracle(num_nodes, src, dst, features, model)
    o.num_nodes = num_nodes
    return o


def classify(alpha_prev, dele, add, is_max: bool) -> int:
    lib = orc_lib()
    a = np.ascontiguousarray(alpha_prev, dtype=np.float32)
    d = None if dele is None else np.ascontiguousarray(dele, dtype=np.float32)
    p = None if add is None else np.ascontiguousarray(add, dtype=np.float32)
    return lib.orc_classify(_ptr(a), _ptr(d), _ptr(p), len(a), int(is_max))


def matvec_affine(w, x, bias=None) -> np.ndarray:
    lib = orc_lib()
    w = np.ascontiguousarray(w, dtype=np.float32)
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    out = np.empty(w.shape[0], dtype=np.float32)
    lib.orc_matvec_affine(_ptr(w), w.shape[0], w.shape[1], _ptr(x), _ptr(b), _ptr(out))
    return out


# ---------------------------------------------------------------------------
# The unmodified reference (oracle/_ref), when built.

_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        lib = _load(REF_SO)
        lib.ref_engine_create.restype = C.c_void_p
        lib.ref_engine_create.argtypes = [C.c_uint32, _u32p, _u32p, C.c_uint64, _f32p, C.c_uint32, C.c_uint32,
                                          C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_int)]
        lib.ref_engine_destroy.argtypes = [C.c_void_p]
        lib.ref_engine_set_option.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        lib.ref_engine_apply.argtypes = [C.c_void_p, C.c_char_p, _u32p, _u32p, C.c_size_t, C.c_char_p, C.c_size_t]
        lib.ref_engine_apply_timed.restype = C.c_double
        lib.ref_engine_apply_timed.argtypes = [C.c_void_p, C.c_char_p, _u32p, _u32p, C.c_size_t,
                                               C.POINTER(C.c_int)]
        lib.ref_engine_stats_line.restype = C.c_uint64
        lib.ref_engine_stats_line.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64]
        lib.ref_engine_dirty.restype = C.c_uint64
        lib.ref_engine_dirty.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64]
        lib.ref_engine_dim.restype = C.c_uint32
        lib.ref_engine_dim.argtypes = [C.c_void_p, C.c_int, C.c_int]
        lib.ref_engine_table.argtypes = [C.c_void_p, C.c_int, C.c_int, _f32p]
        lib.ref_engine_verify.argtypes = [C.c_void_p]
        lib.ref_engine_save_checkpoints.argtypes = [C.c_void_p, C.c_char_p]
        lib.ref_affected_inference_ms.restype = C.c_double
        lib.ref_affected_inference_ms.argtypes = [C.c_void_p, C.c_char_p, _u32p, _u32p, C.c_size_t]
        lib.ref_last_error.restype = C.c_char_p
        lib.sgnn_gen_model.restype = C.c_int
        lib.sgnn_gen_model.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_double,
                                       C.c_char_p]
        lib.ref_classify.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_int]
        lib.ref_matvec_affine.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]
        _ref = lib
    return _ref


def ref_gen_model(kind, feature_len, hidden, layers, seed, epsilon, out_dir):
    """The reference's own sgnn_gen_model (proj/src/capi/capi.cpp, synth.cpp:113-152)."""
    st = ref_lib().sgnn_gen_model(kind.encode(), feature_len, hidden, layers, seed, epsilon, out_dir.encode())
    if st:
        raise RuntimeError(f"sgnn_gen_model failed ({st})")


def ref_generator():
    """The benchmark-input generator compiled into oracle/_ref (tools/rmat_gen.hpp)."""
    from tools.datagen import Generator
    return Generator(ref_lib(), "ref")


class RefEngine:
    """The reference Engine (proj/src/core/engine.hpp:69-118) via oracle/ref_harness.cpp."""

    def __init__(self, num_nodes, src, dst, features, desc_path, manifest_path, ckpt_dir=None):
        lib = ref_lib()
        self.lib = lib
        feats = np.ascontiguousarray(features, dtype=np.float32)
        st = C.c_int(0)
        self.h = lib.ref_engine_create(num_nodes, np.ascontiguousarray(src, dtype=np.uint32),
                                       np.ascontiguousarray(dst, dtype=np.uint32), len(src), feats,
                                       feats.shape[0], feats.shape[1], desc_path.encode(), manifest_path.encode(),
                                       ckpt_dir.encode() if ckpt_dir else None, C.byref(st))
        if not self.h:
            raise RuntimeError(f"reference create failed ({st.value}): {lib.ref_last_error().decode()}")
        self.num_nodes = feats.shape[0]
        self.status = st.value

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_engine_destroy(self.h)
            self.h = None

    def set_option(self, name, value):
        return self.lib.ref_engine_set_option(self.h, name.encode(), value)

    def apply(self, ops: bytes, src, dst):
        buf = C.create_string_buffer(1 << 16)
        st = self.lib.ref_engine_apply(self.h, ops, np.ascontiguousarray(src, dtype=np.uint32),
                                       np.ascontiguousarray(dst, dtype=np.uint32), len(src), buf, len(buf))
        self.line = buf.value.decode() if st == 0 else None
        return st

    def apply_timed(self, ops: bytes, src, dst) -> float:
        st = C.c_int(0)
        ms = self.lib.ref_engine_apply_timed(self.h, ops, np.ascontiguousarray(src, dtype=np.uint32),
                                             np.ascontiguousarray(dst, dtype=np.uint32), len(src), C.byref(st))
        if st.value:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return ms

    def affected_inference_ms(self, ops: bytes, src, dst) -> float:
        return self.lib.ref_affected_inference_ms(self.h, ops, np.ascontiguousarray(src, dtype=np.uint32),
                                                  np.ascontiguousarray(dst, dtype=np.uint32), len(src))

    def last_error(self):
        return self.lib.ref_last_error().decode()

    def dirty(self, layer):
        n = self.lib.ref_engine_dirty(self.h, layer, None, 0)
        out = np.empty(n, dtype=np.uint32)
        self.lib.ref_engine_dirty(self.h, layer, _ptr(out), n)
        return out

    def stats_line(self):
        buf = C.create_string_buffer(1 << 16)
        self.lib.ref_engine_stats_line(self.h, buf, len(buf))
        return buf.value.decode()

    def table(self, layer, stage):
        d = self.lib.ref_engine_dim(self.h, layer, stage)
        out = np.empty((self.num_nodes, d), dtype=np.float32)
        self.lib.ref_engine_table(self.h, layer, stage, out)
        return out

    def verify(self) -> int:
        return self.lib.ref_engine_verify(self.h)

    def save_checkpoints(self, path):
        return self.lib.ref_engine_save_checkpoints(self.h, path.encode())
