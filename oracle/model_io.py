"""TEST INFRASTRUCTURE — file-format readers for the oracle harness.

Re-expresses the reference's file formats so the C restatement
(oracle/sgnn_oracle.c) can be fed parsed inputs:
  * TNSR tensors: proj/src/core/tensor_io.cpp:17-66 (magic, u32 rank, u32 dims,
    f32 payload; NaN rejected, -0 flushed on load)
  * model description grammar: proj/src/core/model.cpp:29-99
  * weight manifest: proj/src/core/model.cpp:130-166
  * edge lists / update streams: proj/src/core/graph.cpp:149-214
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import os
import struct

import numpy as np

AGGREGATE, LINEAR, RELU, SAGE_SELF, GIN_SELF = 0, 1, 2, 3, 4


def read_tnsr(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:4] != b"TNSR":
        raise ValueError(f"not a tensor file: {path}")
    (rank,) = struct.unpack_from("<I", raw, 4)
    dims = struct.unpack_from("<%dI" % rank, raw, 8)
    data = np.frombuffer(raw, dtype="<f4", offset=8 + 4 * rank).copy()
    if np.isnan(data).any():
        raise ValueError("NaN in tensor file")
    data[data == 0] = 0.0  # flush -0 (tensor_io.cpp:64)
    return data.reshape(dims)


def write_tnsr(path: str, arr: np.ndarray) -> None:
    arr = np.ascontiguousarray(arr, dtype="<f4")
    with open(path, "wb") as f:
        f.write(b"TNSR")
        f.write(struct.pack("<I", arr.ndim))
        f.write(struct.pack("<%dI" % arr.ndim, *arr.shape))
        f.write(arr.tobytes())


class ParsedModel:
    """Ops of a model description bound to its weights (model.cpp:29-99, 130-166)."""

    def __init__(self, ops, is_max, weights, epsilon):
        self.ops = ops  # list of (kind, weight name, bias name, hook)
        self.is_max = is_max
        self.weights = weights
        self.epsilon = epsilon

    @property
    def num_layers(self) -> int:
        return sum(1 for o in self.ops if o[0] == AGGREGATE)

    def partition_of(self, op_index: int) -> int:
        p = -1
        for i, o in enumerate(self.ops):
            if o[0] == AGGREGATE:
                p += 1
            if i == op_index:
                return max(p, 0)
        return p

    def oracle_ops(self):
        """[(kind, w, bias, eps)] with hooks resolved to their weights (hooks.cpp:11-22)."""
        out = []
        for i, (kind, w, b, hook) in enumerate(self.ops):
            p = self.partition_of(i)
            if kind == LINEAR:
                out.append((LINEAR, self.weights[w], self.weights[b] if b else None, 0.0))
            elif kind == SAGE_SELF:
                out.append((SAGE_SELF, self.weights[f"W2_{p}"], None, 0.0))
            elif kind == GIN_SELF:
                out.append((GIN_SELF, None, None, self.epsilon[p]))
            else:
                out.append((kind, None, None, 0.0))
        return out


def parse_description(text: str):
    ops = []
    agg = None
    for line in text.splitlines():
        toks = line.split()
        if not toks or toks[0].startswith("#"):
            continue
        kw = toks[0]
        if kw in ("min", "max"):
            agg = kw
            ops.append((AGGREGATE, None, None, None))
        elif kw == "relu":
            ops.append((RELU, None, None, None))
        elif kw == "lin":
            ops.append((LINEAR, toks[1], toks[3] if len(toks) >= 4 else None, None))
        elif kw == "user_apply":
            ops.append((SAGE_SELF if toks[1] == "sage_self" else GIN_SELF, None, None, toks[1]))
        else:
            raise ValueError(f"unknown keyword {kw}")
    return ops, agg == "max"


def load_model(desc_path: str, manifest_path: str) -> ParsedModel:
    with open(desc_path) as f:
        ops, is_max = parse_description(f.read())
    weights, eps = {}, {}
    base = os.path.dirname(manifest_path)
    with open(manifest_path) as f:
        for line in f:
            toks = line.split()
            if not toks or toks[0].startswith("#"):
                continue
            if toks[0] == "epsilon":
                eps[int(toks[1])] = np.float32(float(toks[2]))
                continue
            weights[toks[0]] = read_tnsr(os.path.join(base, toks[1]))
    return ParsedModel(ops, is_max, weights, eps)


def read_edge_list(path: str):
    src, dst = [], []
    with open(path) as f:
        for line in f:
            toks = line.split()
            if not toks or toks[0].startswith("#"):
                continue
            src.append(int(toks[0]))
            dst.append(int(toks[1]))
    return np.array(src, dtype=np.uint32), np.array(dst, dtype=np.uint32)


def read_stream(path: str):
    ops, src, dst = [], [], []
    with open(path) as f:
        for line in f:
            toks = line.split()
            if not toks or toks[0].startswith("#"):
                continue
            ops.append(toks[0])
            src.append(int(toks[1]))
            dst.append(int(toks[2]))
    return "".join(ops).encode(), np.array(src, dtype=np.uint32), np.array(dst, dtype=np.uint32)
