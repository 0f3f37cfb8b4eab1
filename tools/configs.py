"""BENCHMARK / TEST HARNESS — BASELINE.json's configurations and their inputs.

One place that turns a config name into (graph, features, model files, update
stream), used by bench.py (both arms), the config-scale golden script
(tests/golden/make_config_golden.py) and the config-scale GPU parity tests.

`gen` is a tools.datagen.Generator over either harness library (the B200 arm's
tools/libsgnn_datagen.so or the copy inside oracle/_ref); `gen_model` is either
the product's or the reference's own `sgnn_gen_model` (byte-identical output,
tests/test_host_abi.py). Shapes: SURVEY.md §8 (hidden dims from the paper's
Table 2 where BASELINE.json is silent); weights from the reference's make_model
with seed 7 and the aggregation lines rewritten min -> max.
"""
from __future__ import annotations

import hashlib
import os
import tempfile
import time

import numpy as np

CONFIGS = {
    "c1": dict(workload="C1: 2-layer GraphSAGE-max, synthetic 10K-node R-MAT graph (100K edges, 64-d)",
               nodes=10_000, edges=100_000, feat=64, hidden=64, layers=2, kind="sage", batch=100),
    "c2": dict(workload="C2: 2-layer GCN-max, synthetic Reddit-shape R-MAT graph (233K nodes, 114M edges, 602-d)",
               nodes=233_000, edges=114_000_000, feat=602, hidden=256, layers=2, kind="gcn", batch=1000),
    "c3": dict(workload="C3: 2-layer GIN-max, synthetic ogbn-products-shape R-MAT graph (2.4M nodes, 62M edges, "
                        "100-d)",
               nodes=2_400_000, edges=62_000_000, feat=100, hidden=64, layers=2, kind="gin", batch=1000),
    # configs[3] (C4, 111M nodes / 1.6B edges, 8 GPUs) at one GPU's share: the
    # same 3-layer SAGE-max 128-d model, 1/8 of the nodes and edges, so the
    # engine holds the per-GPU table bytes of an 8-way vertex-sharded C4
    # (7 tables x 13.9M x 512 B = 49.7 GB). The reference CPU path is not run
    # at this size (its init alone is hours of single-threaded work).
    "c4s": dict(workload="C4/8: 3-layer GraphSAGE-max, one GPU's share of the papers100M-shape R-MAT graph "
                         "(13.9M nodes, 200M edges, 128-d)",
                nodes=13_875_000, edges=200_000_000, feat=128, hidden=128, layers=3, kind="sage", batch=1000,
                cpu=False),
}
GRAPH_SEED, MODEL_SEED, STREAM_SEED, EPSILON = 2024, 7, 2025, 0.1
DATA = ("synthetic: seeded R-MAT (0.57,0.19,0.19,0.05) graph, uniform [0,1) features, reference make_model "
        "weights (seed 7, min->max), 50/50 insert/delete R-MAT stream")
CACHE = os.path.join(tempfile.gettempdir(), "sgnn_bench_cache")


def dims(cfg):
    return [cfg["feat"]] + [cfg["hidden"]] * cfg["layers"]


def graph(name, gen, log=None):
    """R-MAT base graph (cached under /tmp only to skip regeneration; the bytes
    are the generator's either way)."""
    cfg = CONFIGS[name]
    os.makedirs(CACHE, exist_ok=True)
    path = os.path.join(CACHE, f"{name}_graph_v2.npz")
    if os.path.exists(path):
        z = np.load(path)
        return z["src"], z["dst"]
    t = time.time()
    src, dst = gen.rmat(cfg["nodes"], cfg["edges"], GRAPH_SEED)
    tmp = f"{path}.{os.getpid()}.tmp.npz"  # ranks of one box may generate concurrently
    np.savez(tmp, src=src, dst=dst)
    os.replace(tmp, path)
    if log:
        log(f"[inputs] generated the {name} R-MAT graph in {time.time() - t:.1f}s")
    return src, dst


def features(name, gen):
    cfg = CONFIGS[name]
    return gen.features(cfg["nodes"], cfg["feat"], GRAPH_SEED)


def model_files(name, gen_model, out_dir):
    """Writes description.txt + weights.txt through `gen_model`; returns their paths."""
    cfg = CONFIGS[name]
    gen_model(cfg["kind"], cfg["feat"], cfg["hidden"], cfg["layers"], MODEL_SEED, EPSILON, out_dir)
    desc = os.path.join(out_dir, "description.txt")
    text = open(desc).read().replace("min\n", "max\n")  # GCN/SAGE-max
    open(desc, "w").write(text)
    return desc, os.path.join(out_dir, "weights.txt")


def batches(name, gen, src, dst, n_batches, seed=STREAM_SEED, batch=None):
    cfg = CONFIGS[name]
    b = batch or cfg["batch"]
    ops, ss, dd = gen.rmat_stream(cfg["nodes"], src, dst, n_batches * b, 0.5, seed)
    return [(ops[i * b:(i + 1) * b], ss[i * b:(i + 1) * b], dd[i * b:(i + 1) * b]) for i in range(n_batches)]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def table_digests(read_table, k):
    """{"m1": …, "a1": …, …, "m{k+1}": …}: sha256 prefix of every message /
    aggregate table (row-major fp32, unpadded)."""
    out = {}
    for layer in range(1, k + 2):
        out[f"m{layer}"] = sha(read_table(layer, 0))
        if layer <= k:
            out[f"a{layer}"] = sha(read_table(layer, 1))
    return out


def dirty_digest(dirty_nodes, k):
    """Per layer: (count, sha256 prefix of the ascending dirty id list)."""
    out = []
    for layer in range(1, k + 1):
        d = np.ascontiguousarray(dirty_nodes(layer), dtype=np.uint32)
        out.append([int(len(d)), sha(d)])
    return out
