"""Full-size parity through size-independent properties.

At BASELINE.json's products shape (C3: 2.4M nodes, 62M R-MAT edges, 100-d,
2-layer GIN-max) the oracle is too slow to replay, so the checks are
properties that must hold bit for bit at any size:
  * incremental tables == a from-scratch full inference on the final graph
    (verify, baseline.cpp:234-256) after a stream of 1K-edge batches;
  * the k-hop comparator (affected_inference, baseline.cpp:177-207) leaves the
    same tables as the incremental path on the same stream;
  * every round's counters are internally consistent (targets split exactly
    into the four conditions, engine.cpp:45-78).
"""
import numpy as np
import pytest

import paper_2309_11071_b200 as sg
from tools.datagen import Generator

pytestmark = pytest.mark.gpu


def _kv(line):
    return {k: int(v) for k, v in (t.split("=", 1) for t in line.split())}


def test_products_shape_incremental_equals_full_and_khop(tmp_path):
    n, e, f, hidden = 2_400_000, 62_000_000, 100, 64
    gen = Generator()
    src, dst = gen.rmat(n, e, 2024)
    feats = gen.features(n, f, 2024)
    sg.gen_model("gin", f, hidden, 2, 7, 0.1, str(tmp_path))
    desc = str(tmp_path / "description.txt")
    text = open(desc).read().replace("min\n", "max\n")
    open(desc, "w").write(text)
    m = sg.Model.load(desc, str(tmp_path / "weights.txt"))
    inc = sg.Engine.create_from_array(sg.Graph.from_edges(n, src, dst), m, feats)
    ops, ss, dd = gen.rmat_stream(n, src, dst, 12_000, 0.5, 2025)
    kh = sg.Engine.create_from_array(sg.Graph.from_edges(n, src, dst), m, feats)
    kh.set_option("khop_recompute", 1)
    for i in range(0, len(ss), 1000):
        inc.apply_update(ops[i:i + 1000], ss[i:i + 1000], dd[i:i + 1000])
        kh.apply_update(ops[i:i + 1000], ss[i:i + 1000], dd[i:i + 1000])
        s = _kv(inc.stats_line())
        for layer in (1, 2):
            p = f"l{layer}."
            assert s[p + "targets"] == (s[p + "no_deletion"] + s[p + "deletion_no_effect"] + s[p + "covered_reset"]
                                        + s[p + "exposed_reset"]), s
            assert s[p + "recomputes"] == s[p + "exposed_reset"]
    assert inc.num_edges == kh.num_edges
    st, where = inc.verify()
    assert st == 0, where
    for layer, stage in ((1, 1), (2, 0), (2, 1), (3, 0)):
        assert inc.read_table(layer, stage).tobytes() == kh.read_table(layer, stage).tobytes(), (layer, stage)
