"""CPU: the product library's boundary and host-side logic (no GPU needed).

- libstreamgnn.so loads and exports exactly what include/*.h declares;
- host-side entry points (generators, file formats, graph handle, model
  loading, stream reader) behave like the reference: byte-identical generated
  datasets, identical status codes and messages (tests/golden/ error cases);
- engine creation fails loudly when no CUDA device is present (no CPU fallback).
"""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2309_11071_b200 as sg
from paper_2309_11071_b200 import _lib
from oracle import oracle
from tests import golden_util

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in ("streamgnn.h", "streamgnn_b200.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        names |= set(re.findall(r"\b(sgnn_\w+)\s*\(", text))
    return names


def test_exports_match_headers():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    declared = declared_symbols()
    assert declared == exported, (declared ^ exported)
    assert set(_lib.REFERENCE_SYMBOLS) <= exported and len(_lib.REFERENCE_SYMBOLS) == 31
    lib = _lib.lib()
    for name in declared:
        assert getattr(lib, name) is not None


def test_status_names_are_stable():
    assert sg.status_name(0) == "ok"
    assert sg.status_name(11) == "verification mismatch"
    assert sg.status_name(12) == "unknown error"


@pytest.mark.parametrize("name", sorted(golden_util.expected()["errors"]))
def test_error_codes_and_messages_match_reference(name, tmp_path):
    status, message = golden_util.expected()["errors"][name]
    lib = _lib.lib()
    import ctypes as C
    g = C.c_void_p()
    err = os.path.join(golden_util.DATA, "_err")
    if name == "graph_create_zero":
        st = lib.sgnn_graph_create(0, C.byref(g))
    elif name.startswith("add_edge"):
        lib.sgnn_graph_create(4, C.byref(g))
        lib.sgnn_graph_add_edge(g, 0, 1)
        args = {"add_edge_dup": (0, 1), "add_edge_range": (0, 99), "add_edge_range_src": (77, 1)}[name]
        st = lib.sgnn_graph_add_edge(g, *args)
        lib.sgnn_graph_destroy(g)
    elif name == "graph_load_missing":
        st = lib.sgnn_graph_load(b"/nonexistent/edges.txt", 0, C.byref(g))
    elif name.startswith("graph_load_"):
        st = lib.sgnn_graph_load(os.path.join(err, name[len("graph_load_"):] + ".txt").encode(), 0, C.byref(g))
    elif name.startswith("model_"):
        m = C.c_void_p()
        st = lib.sgnn_model_load(os.path.join(err, f"desc_{name[6:]}.txt").encode(),
                                 os.path.join(err, "weights.txt").encode(), C.byref(m))
    else:
        pytest.fail(name)
    got = lib.sgnn_last_error().decode()
    assert st == status
    assert got.replace(err, "<dir>") == message.replace(err, "<dir>")


def test_generators_byte_identical_to_reference(tmp_path):
    """sgnn_gen_synthetic / sgnn_gen_model reproduce the reference's files (synth.cpp)."""
    for name, c in (("accept", (1000, 8.0, 16, 200, 2024, 0.6)), ("small", (90, 4.0, 5, 60, 61, 0.6))):
        d = str(tmp_path / name)
        sg.gen_synthetic(d, *c)
        for f in ("edges.txt", "features.tnsr", "stream.txt", "gen.txt"):
            assert open(os.path.join(d, f), "rb").read() == open(os.path.join(golden_util.DATA, name, f), "rb").read()
    d = str(tmp_path / "accept")
    sg.gen_model("gcn", 16, 16, 2, 7, 0.1, os.path.join(d, "gcn"))
    sg.gen_model("gin", 16, 8, 5, 7, 0.1, os.path.join(d, "gin5"))
    for model in ("gcn", "gin5"):
        ref_dir = os.path.join(golden_util.DATA, "accept", model)
        for f in os.listdir(ref_dir):
            assert open(os.path.join(d, model, f), "rb").read() == open(os.path.join(ref_dir, f), "rb").read(), f


def test_graph_handle_roundtrip(tmp_path):
    g = sg.Graph.load(os.path.join(golden_util.DATA, "accept", "edges.txt"))
    assert g.num_nodes == 1000 and g.num_edges == 8000
    out0 = g.out_neighbors(0)
    assert list(out0) == sorted(out0)
    for v in out0:
        assert 0 in g.in_neighbors(int(v))
    p = str(tmp_path / "e.txt")
    g.save(p)
    assert open(p).read() == open(os.path.join(golden_util.DATA, "accept", "edges.txt")).read()
    with pytest.raises(sg.StreamGNNError) as e:
        g.out_neighbors(5000)
    assert e.value.status == 7
    # bulk construction applies add_edge semantics, first failure in input order
    with pytest.raises(sg.StreamGNNError) as e:
        sg.Graph.from_edges(5, [0, 1, 0, 2], [1, 2, 1, 9])
    assert e.value.status == 4 and "0->1" in e.value.message
    with pytest.raises(sg.StreamGNNError) as e:
        sg.Graph.from_edges(5, [0, 1, 3], [1, 7, 1])
    assert e.value.status == 7 and "7" in e.value.message
    h = sg.Graph.from_edges(4, [0, 1, 2], [1, 0, 2], symmetrize=True)
    assert h.num_edges == 3  # 0<->1 deduplicated, self loop once


def test_symmetrized_load_matches_reference(tmp_path):
    p = str(tmp_path / "e.txt")
    open(p, "w").write("0 1\n1 0\n2 2\n3 1\n")
    g = sg.Graph.load(p, symmetrize=True)
    assert g.num_edges == 5 and list(g.out_neighbors(1)) == [0, 3]  # 0->1 1->0 2->2 3->1 1->3


def test_stream_reader():
    r = sg.StreamReader(os.path.join(golden_util.DATA, "accept", "stream.txt"))
    events = list(r)
    assert len(events) == 200 and all(op in "+-" for op, _, _ in events)


def test_model_introspection():
    d = os.path.join(golden_util.DATA, "accept", "gcn")
    m = sg.Model.load(os.path.join(d, "description.txt"), os.path.join(d, "weights.txt"))
    assert m.num_layers == 2 and m.aggregator == 0
    d = os.path.join(golden_util.DATA, "maxagg", "gin_max")
    m = sg.Model.load(os.path.join(d, "description.txt"), os.path.join(d, "weights.txt"))
    assert m.aggregator == 1


def test_engine_input_errors_before_touching_the_device(tmp_path):
    """File/format/dimension errors of engine creation come from host code and
    match the reference's order (capi.cpp:210-229)."""
    d = os.path.join(golden_util.DATA, "accept")
    g = sg.Graph.load(os.path.join(d, "edges.txt"))
    m = sg.Model.load(os.path.join(d, "gcn", "description.txt"), os.path.join(d, "gcn", "weights.txt"))
    with pytest.raises(sg.StreamGNNError) as e:
        sg.Engine.create(g, m, str(tmp_path / "missing.tnsr"))
    assert e.value.status == 1
    bad = np.zeros((1000, 3), np.float32)  # wrong feature length for W_0 (16 columns)
    with pytest.raises(sg.StreamGNNError) as e:
        sg.Engine.create_from_array(g, m, bad)
    assert e.value.status == 3
    nan = np.full((1000, 16), np.nan, np.float32)
    with pytest.raises(sg.StreamGNNError) as e:
        sg.Engine.create_from_array(g, m, nan)
    assert e.value.status == 10
    few = np.zeros((10, 16), np.float32)  # graph has more nodes than feature rows
    with pytest.raises(sg.StreamGNNError) as e:
        sg.Engine.create_from_array(g, m, few)
    assert e.value.status == 3 and "feature rows" in e.value.message


def test_no_cpu_fallback(has_gpu):
    if has_gpu:
        pytest.skip("a CUDA device is present")
    d = os.path.join(golden_util.DATA, "accept")
    g = sg.Graph.load(os.path.join(d, "edges.txt"))
    m = sg.Model.load(os.path.join(d, "gcn", "description.txt"), os.path.join(d, "gcn", "weights.txt"))
    with pytest.raises(sg.StreamGNNError) as e:
        sg.Engine.create(g, m, os.path.join(d, "features.tnsr"))
    assert e.value.status == 12 and "CUDA" in e.value.message


def test_rmat_generator_deterministic_and_simple():
    """Harness generator (tools/rmat_gen.hpp): the B200 arm's library and the
    copy compiled into oracle/_ref give byte-identical inputs."""
    from tools.datagen import Generator
    gen = Generator()
    s1, d1 = gen.rmat(5000, 40000, 3)
    s2, d2 = gen.rmat(5000, 40000, 3)
    assert np.array_equal(s1, s2) and np.array_equal(d1, d2)
    keys = (s1.astype(np.uint64) << 32) | d1
    assert len(np.unique(keys)) == 40000 and np.all(np.diff(keys.astype(np.int64)) > 0)
    assert not np.any(s1 == d1) and s1.max() < 5000 and d1.max() < 5000
    indeg = np.bincount(d1, minlength=5000)
    assert indeg.max() > 20 * np.median(indeg)  # power-law hubs
    ops, ss, dd = gen.rmat_stream(5000, s1, d1, 2000, 0.5, 9)
    feats = gen.features(5000, 8, 3)
    if oracle.ref_available():
        ref = Generator(oracle.ref_lib(), "ref")
        r1, r2 = ref.rmat(5000, 40000, 3)
        assert np.array_equal(r1, s1) and np.array_equal(r2, d2)
        assert ref.rmat_stream(5000, s1, d1, 2000, 0.5, 9)[0] == ops
        assert np.array_equal(ref.features(5000, 8, 3), feats)
    live = set(keys.tolist())
    for op, a, b in zip(ops, ss, dd):
        k = (int(a) << 32) | int(b)
        if op == ord("+"):
            assert k not in live and a != b
            live.add(k)
        else:
            assert k in live
            live.remove(k)
