"""CPU: binary edge-list ingest.

sgnn_b200_graph_load_binary must build exactly the graph the reference's text
loader builds from the same pairs in the same order (graph.cpp:149-183): the
graph the product loads from a binary file, saved as text, is byte-identical
to what the unmodified reference (oracle/_ref, through its own C ABI) saves
after loading the text file; failures (duplicate edge, bad header, short file)
keep the reference's status codes and messages.
"""
import ctypes as C
import os
import struct

import numpy as np
import pytest

import paper_2309_11071_b200 as sg
from oracle import model_io, oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "data")


def write_binary(path, src, dst, num_nodes=0):
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    with open(path, "wb") as f:
        f.write(b"SGNNEDG1" + struct.pack("<IIQ", num_nodes, 0, len(src)))
        f.write(src.tobytes())
        f.write(dst.tobytes())


def ref_load_save(text_path, out_path, symmetrize=False):
    """The reference's own sgnn_graph_load + sgnn_graph_save (capi.cpp)."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    L = C.CDLL(oracle.REF_SO)
    L.sgnn_graph_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
    L.sgnn_graph_save.argtypes = [C.c_void_p, C.c_char_p]
    L.sgnn_graph_destroy.argtypes = [C.c_void_p]
    L.sgnn_last_error.restype = C.c_char_p
    h = C.c_void_p()
    st = L.sgnn_graph_load(text_path.encode(), symmetrize, C.byref(h))
    if st:
        return st, L.sgnn_last_error().decode()
    assert L.sgnn_graph_save(h, out_path.encode()) == 0
    L.sgnn_graph_destroy(h)
    return 0, ""


@pytest.mark.parametrize("dataset,symmetrize", [("accept", False), ("maxagg", False), ("small", True)])
def test_binary_matches_reference_text_load(tmp_path, dataset, symmetrize):
    text = os.path.join(GOLDEN, dataset, "edges.txt")
    src, dst = model_io.read_edge_list(text)
    b = str(tmp_path / "g.bin")
    write_binary(b, src, dst)
    g = sg.Graph.load_binary(b, symmetrize)
    mine = str(tmp_path / "mine.txt")
    g.save(mine)
    ref = str(tmp_path / "ref.txt")
    assert ref_load_save(text, ref, symmetrize)[0] == 0
    assert open(mine, "rb").read() == open(ref, "rb").read()
    # save_binary -> load_binary round trip keeps nodes, edges and lists
    b2 = str(tmp_path / "g2.bin")
    g.save_binary(b2)
    g2 = sg.Graph.load_binary(b2)
    assert (g2.num_nodes, g2.num_edges) == (g.num_nodes, g.num_edges)
    for v in range(0, g.num_nodes, max(1, g.num_nodes // 50)):
        assert np.array_equal(g2.out_neighbors(v), g.out_neighbors(v))
        assert np.array_equal(g2.in_neighbors(v), g.in_neighbors(v))


def test_binary_header_node_count_and_errors(tmp_path):
    b = str(tmp_path / "g.bin")
    write_binary(b, [0, 1], [1, 2], num_nodes=10)  # isolated trailing nodes survive
    g = sg.Graph.load_binary(b)
    assert (g.num_nodes, g.num_edges) == (10, 2)
    # a duplicate edge fails like the text loader on the same pairs (reference status + message)
    write_binary(b, [0, 1, 0], [1, 2, 1])
    t = str(tmp_path / "dup.txt")
    open(t, "w").write("0 1\n1 2\n0 1\n")
    ref_st, ref_msg = ref_load_save(t, str(tmp_path / "unused.txt"))
    with pytest.raises(sg.StreamGNNError) as ei:
        sg.Graph.load_binary(b)
    assert (ei.value.status, ei.value.message) == (ref_st, ref_msg)
    open(b, "wb").write(b"NOTMAGIC" + bytes(16))
    with pytest.raises(sg.StreamGNNError) as ei:
        sg.Graph.load_binary(b)
    assert ei.value.status == 2 and "header" in ei.value.message
    write_binary(b, [0, 1, 2], [1, 2, 3])
    open(b, "r+b").truncate(os.path.getsize(b) - 4)
    with pytest.raises(sg.StreamGNNError) as ei:
        sg.Graph.load_binary(b)
    assert ei.value.status == 2 and "truncated" in ei.value.message
    with pytest.raises(sg.StreamGNNError) as ei:
        sg.Graph.load_binary(str(tmp_path / "missing.bin"))
    assert ei.value.status == 1
