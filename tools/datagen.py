"""BENCHMARK / TEST HARNESS — synthetic inputs for the BASELINE.json configs.

ctypes over tools/libsgnn_datagen.so (tools/rmat_gen.hpp). The same header is
compiled into oracle/_ref/libstreamgnn_ref.so (ref_gen_* entry points), which
is what bench.py's reference arm uses, so neither arm needs the other's library
to build byte-identical inputs. Not product code.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libsgnn_datagen.so")
_lib = None


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def bind(lib, prefix):
    """Declares the three generator entry points of `lib` (prefix 'dg' or 'ref')."""
    vp = C.c_void_p
    f = getattr(lib, f"{prefix}_gen_rmat")
    f.restype, f.argtypes = C.c_int, [C.c_uint32, C.c_uint64, C.c_uint64, vp, vp]
    f = getattr(lib, f"{prefix}_gen_rmat_stream")
    f.restype, f.argtypes = C.c_int, [C.c_uint32, vp, vp, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, vp, vp, vp]
    f = getattr(lib, f"{prefix}_gen_features")
    f.restype, f.argtypes = C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, vp]
    return lib


class Generator:
    """R-MAT graph / stream / features through one harness library."""

    def __init__(self, lib=None, prefix="dg"):
        global _lib
        if lib is None:
            if _lib is None:
                if not os.path.exists(SO):
                    raise FileNotFoundError(f"{SO} not built (make -C tools)")
                _lib = bind(C.CDLL(SO), "dg")
            lib = _lib
        else:
            bind(lib, prefix)
        self.lib, self.prefix = lib, prefix

    def _call(self, name, *args):
        if getattr(self.lib, f"{self.prefix}_{name}")(*args) != 0:
            err = getattr(self.lib, f"{self.prefix}_last_error")
            err.restype = C.c_char_p
            raise RuntimeError(f"{name}: {err().decode()}")

    def rmat(self, num_nodes: int, num_edges: int, seed: int):
        src = np.empty(num_edges, dtype=np.uint32)
        dst = np.empty(num_edges, dtype=np.uint32)
        self._call("gen_rmat", num_nodes, num_edges, seed, _p(src), _p(dst))
        return src, dst

    def rmat_stream(self, num_nodes: int, src, dst, stream_len: int, insert_fraction: float, seed: int):
        src = np.ascontiguousarray(src, dtype=np.uint32)
        dst = np.ascontiguousarray(dst, dtype=np.uint32)
        ops = np.empty(stream_len, dtype=np.uint8)
        s = np.empty(stream_len, dtype=np.uint32)
        d = np.empty(stream_len, dtype=np.uint32)
        self._call("gen_rmat_stream", num_nodes, _p(src), _p(dst), len(src), stream_len, insert_fraction, seed,
                   _p(ops), _p(s), _p(d))
        return ops.tobytes(), s, d

    def features(self, rows: int, cols: int, seed: int) -> np.ndarray:
        out = np.empty((rows, cols), dtype=np.float32)
        self._call("gen_features", rows, cols, seed, _p(out))
        return out
