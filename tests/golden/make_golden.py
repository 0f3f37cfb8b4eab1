"""Generates the golden fixtures under tests/golden/ from the UNMODIFIED reference.

Runs only where /root/reference exists (oracle/_ref built by `make`): datasets and
models are written by the reference's own C ABI (sgnn_gen_synthetic,
sgnn_gen_model; proj/src/capi/capi.cpp:347-399), every stream is processed by the
reference Engine (proj/src/core/engine.cpp:171-319, via oracle/ref_harness.cpp),
and the expected per-round stats lines, per-layer dirty sets and table digests
are stored in tests/golden/expected.json.gz. Error cases record the reference's
status codes and messages through its C ABI.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import gzip
import hashlib
import json
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import model_io, oracle  # noqa: E402

DATA = os.path.join(HERE, "data")


class GenCfg(C.Structure):
    _fields_ = [("num_nodes", C.c_uint32), ("avg_degree", C.c_double), ("feature_len", C.c_uint32),
                ("stream_len", C.c_uint32), ("seed", C.c_uint64), ("insert_fraction", C.c_double)]


def ref_capi():
    lib = oracle.ref_lib()
    lib.sgnn_last_error.restype = C.c_char_p
    lib.sgnn_gen_synthetic.argtypes = [C.POINTER(GenCfg), C.c_char_p]
    lib.sgnn_gen_model.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_double,
                                   C.c_char_p]
    return lib


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


DATASETS = {
    # the acceptance dataset (proj/tests/acceptance_tests.cpp:27-64)
    "accept": dict(nodes=1000, deg=8.0, feat=16, stream=200, seed=2024, ins=0.6),
    "maxagg": dict(nodes=300, deg=6.0, feat=24, stream=140, seed=77, ins=0.55),
    "wide": dict(nodes=150, deg=10.0, feat=602, stream=60, seed=5, ins=0.5),
    "small": dict(nodes=90, deg=4.0, feat=5, stream=60, seed=61, ins=0.6),
}

# (case name, dataset, model dir, batch, options, rounds limit)
CASES = [
    ("accept_gcn_b1", "accept", "gcn", 1, {"baseline_counters": 1}, None),
    ("accept_sage_b1", "accept", "sage", 1, {"baseline_counters": 1}, None),
    ("accept_gin5_b1", "accept", "gin5", 1, {"baseline_counters": 1}, None),
    ("accept_gcn_b10", "accept", "gcn", 10, {}, 10),
    ("accept_gcn_b100", "accept", "gcn", 100, {}, 1),
    ("accept_gcn_dup", "accept", "gcn", 1, {"duplicate_seed_events": 1}, 20),
    ("maxagg_gcn_b7", "maxagg", "gcn_max", 7, {"baseline_counters": 1}, None),
    ("maxagg_sage_b7", "maxagg", "sage_max", 7, {}, None),
    ("maxagg_gin_b7", "maxagg", "gin_max", 7, {}, None),
    ("wide_gcn_b5", "wide", "gcn_max", 5, {}, None),
    ("small_prefix_b1", "small", "prefix", 1, {"baseline_counters": 1}, None),
]


def make_models(lib, name, cfg):
    d = os.path.join(DATA, name)
    F = cfg["feat"]
    models = {}
    if name == "accept":
        for kind, hidden, layers in [("gcn", 16, 2), ("sage", 16, 2)]:
            lib.sgnn_gen_model(kind.encode(), F, hidden, layers, 7, 0.1, os.path.join(d, kind).encode())
            models[kind] = kind
        lib.sgnn_gen_model(b"gin", F, 8, 5, 7, 0.1, os.path.join(d, "gin5").encode())
    elif name in ("maxagg", "wide"):
        for kind, hidden in [("gcn", 32), ("sage", 32), ("gin", 16)]:
            if name == "wide" and kind != "gcn":
                continue
            md = os.path.join(d, f"{kind}_max")
            lib.sgnn_gen_model(kind.encode(), F, hidden if name == "maxagg" else 64, 2, 7, 0.1, md.encode())
            desc = os.path.join(md, "description.txt")
            text = open(desc).read().replace("min\n", "max\n")
            open(desc, "w").write(text)
    elif name == "small":
        # combination-before-aggregation model (proj/tests/test_engine.cpp:399-446 shape)
        md = os.path.join(d, "prefix")
        os.makedirs(md, exist_ok=True)
        rng = np.random.default_rng(60)
        w = {"W0": rng.uniform(-0.3, 0.5, (6, F)), "W1": rng.uniform(-0.3, 0.5, (6, 6)),
             "b1": np.array([0.1, 0.2, 0.0, 0.1, 0.2, 0.0]), "W2": rng.uniform(-0.3, 0.5, (4, 6)),
             "b2": np.array([0.1, 0.0, 0.2, 0.1])}
        lines = []
        for k, v in w.items():
            model_io.write_tnsr(os.path.join(md, k + ".tnsr"), np.asarray(v, dtype=np.float32))
            lines.append(f"{k} {k}.tnsr")
        open(os.path.join(md, "weights.txt"), "w").write("\n".join(lines) + "\n")
        open(os.path.join(md, "description.txt"), "w").write(
            "lin W0\nmin\nlin W1 bias b1\nrelu\nmin\nlin W2 bias b2\nrelu\n")


def run_case(case, dset, model, batch, options, limit):
    d = os.path.join(DATA, dset)
    src, dst = model_io.read_edge_list(os.path.join(d, "edges.txt"))
    feats = model_io.read_tnsr(os.path.join(d, "features.tnsr"))
    ops, ss, dd = model_io.read_stream(os.path.join(d, "stream.txt"))
    desc = os.path.join(d, model, "description.txt")
    man = os.path.join(d, model, "weights.txt")
    ref = oracle.RefEngine(feats.shape[0], src, dst, feats, desc, man)
    for k, v in options.items():
        assert ref.set_option(k, v) == 0
    k = model_io.load_model(desc, man).num_layers
    rounds = []

    def tables():
        out = {}
        for layer in range(1, k + 2):
            for stage in (0, 1):
                if stage == 1 and layer > k:
                    continue
                out[f"{layer}.{stage}"] = digest(ref.table(layer, stage))
        return out

    init = tables()
    r = 0
    for i in range(0, len(ss), batch):
        if limit is not None and r >= limit:
            break
        st = ref.apply(ops[i:i + batch], ss[i:i + batch], dd[i:i + batch])
        assert st == 0, ref.last_error()
        entry = {"line": ref.line, "dirty": [ref.dirty(layer).tolist() for layer in range(1, k + 1)]}
        if (r + 1) % 25 == 0:
            entry["tables"] = tables()
        rounds.append(entry)
        r += 1
    assert ref.verify() == 0
    return {"dataset": dset, "model": model, "batch": batch, "options": options, "limit": limit, "layers": k,
            "init_tables": init, "rounds": rounds, "final_tables": tables()}


def error_cases(lib):
    """Status codes and messages of the reference C ABI for invalid inputs."""
    out = {}
    g = C.c_void_p()
    lib.sgnn_graph_create.argtypes = [C.c_uint32, C.POINTER(C.c_void_p)]
    lib.sgnn_graph_add_edge.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32]
    lib.sgnn_graph_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
    lib.sgnn_model_load.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]
    lib.sgnn_graph_destroy.argtypes = [C.c_void_p]
    lib.sgnn_model_destroy.argtypes = [C.c_void_p]

    def rec(name, st):
        out[name] = [int(st), lib.sgnn_last_error().decode()]

    rec("graph_create_zero", lib.sgnn_graph_create(0, C.byref(g)))
    lib.sgnn_graph_create(4, C.byref(g))
    lib.sgnn_graph_add_edge(g, 0, 1)
    rec("add_edge_dup", lib.sgnn_graph_add_edge(g, 0, 1))
    rec("add_edge_range", lib.sgnn_graph_add_edge(g, 0, 99))
    rec("add_edge_range_src", lib.sgnn_graph_add_edge(g, 77, 1))
    lib.sgnn_graph_destroy(g)
    tmp = os.path.join(DATA, "_err")
    os.makedirs(tmp, exist_ok=True)
    texts = {"bad_line": "0 1\n1 x\n", "extra_tok": "0 1 2\n", "neg": "-1 2\n", "dup": "0 1\n1 2\n0 1\n",
             "comment_ok": "# c\n\n0 1\n 2 3 \n", "big": "4294967296 1\n"}
    for key, text in texts.items():
        p = os.path.join(tmp, key + ".txt")
        open(p, "w").write(text)
        gg = C.c_void_p()
        rec(f"graph_load_{key}", lib.sgnn_graph_load(p.encode(), 0, C.byref(gg)))
        if gg:
            lib.sgnn_graph_destroy(gg)
    rec("graph_load_missing", lib.sgnn_graph_load(b"/nonexistent/edges.txt", 0, C.byref(g)))
    descs = {"unsupported": "min\nsoftmax\n", "mixed": "min\nmax\n", "noagg": "relu\n",
             "user_first": "user_apply sage_self\nmin\n", "bad_lin": "min\nlin W x\n", "unknown": "min\nfoo\n",
             "trailing": "min extra\n", "empty": ""}
    man = os.path.join(tmp, "weights.txt")
    open(man, "w").write("")
    for key, text in descs.items():
        p = os.path.join(tmp, f"desc_{key}.txt")
        open(p, "w").write(text)
        m = C.c_void_p()
        rec(f"model_{key}", lib.sgnn_model_load(p.encode(), man.encode(), C.byref(m)))
        if m:
            lib.sgnn_model_destroy(m)
    return out


def main():
    if not oracle.ref_available():
        raise SystemExit("oracle/_ref not built; run make in a container that has /root/reference")
    lib = ref_capi()
    shutil.rmtree(DATA, ignore_errors=True)
    os.makedirs(DATA)
    for name, c in DATASETS.items():
        cfg = GenCfg(c["nodes"], c["deg"], c["feat"], c["stream"], c["seed"], c["ins"])
        assert lib.sgnn_gen_synthetic(C.byref(cfg), os.path.join(DATA, name).encode()) == 0
        make_models(lib, name, c)
    expected = {"cases": {}, "errors": error_cases(lib)}
    for case, dset, model, batch, options, limit in CASES:
        expected["cases"][case] = run_case(case, dset, model, batch, options, limit)
        print(case, "rounds", len(expected["cases"][case]["rounds"]))
    with gzip.open(os.path.join(HERE, "expected.json.gz"), "wt") as f:
        json.dump(expected, f)


if __name__ == "__main__":
    main()
