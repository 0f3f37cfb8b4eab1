"""Parity at BASELINE.json's own configurations (C1, C2, C3; tools/configs.py).

tests/golden/configs.json.gz holds what the UNMODIFIED reference (oracle/_ref)
produced on exactly these inputs from its own initial full inference
(tests/golden/make_config_golden.py): table digests after init, every round's
stats line and per-layer dirty set, and table digests after the last round.
The product replays the same inputs through the C ABI and must match all of it
bit for bit — on the power-law hubs, bound-code grids, slab relocations and
edge-hash sizes of the benchmark graphs, not only on toy graphs.

C1 (10K nodes) is additionally replayed through the C restatement round by
round with full table comparisons.
"""
import gzip
import json
import os

import numpy as np
import pytest

import paper_2309_11071_b200 as sg
from oracle import model_io, oracle
from tests.util import tables_equal
from tools import configs as CF
from tools.datagen import Generator

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "configs.json.gz")


def _golden():
    return json.load(gzip.open(GOLDEN, "rt"))


def _inputs(name, tmp_path):
    gen = Generator()
    src, dst = CF.graph(name, gen)
    feats = CF.features(name, gen)
    desc, man = CF.model_files(name, sg.gen_model, str(tmp_path))
    return gen, src, dst, feats, desc, man


def _replay(name, eng, gen, src, dst, G, shards_note=""):
    k = CF.CONFIGS[name]["layers"]
    assert CF.table_digests(eng.read_table, k) == G["init"], f"{name}{shards_note}: init tables differ"
    for i, (ops, ss, dd) in enumerate(CF.batches(name, gen, src, dst, G["rounds"])):
        eng.apply_update(ops, ss, dd)
        assert eng.stats_line() == G["lines"][i], f"{name}{shards_note} round {i}\n gpu {eng.stats_line()}\n " \
                                                  f"ref {G['lines'][i]}"
        assert CF.dirty_digest(eng.dirty_nodes, k) == G["dirty"][i], f"{name}{shards_note} round {i}: dirty sets"
    assert CF.table_digests(eng.read_table, k) == G["final"], f"{name}{shards_note}: final tables differ"


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_config_matches_reference(name, tmp_path):
    G = _golden()[name]
    gen, src, dst, feats, desc, man = _inputs(name, tmp_path)
    n = CF.CONFIGS[name]["nodes"]
    eng = sg.Engine.create_from_array(sg.Graph.from_edges(n, src, dst), sg.Model.load(desc, man), feats)
    _replay(name, eng, gen, src, dst, G)
    st, where = eng.verify()
    assert st == 0, where


@pytest.mark.parametrize("name,shards", [("c1", 3), ("c3", 2)])
def test_config_sharded_matches_reference(name, shards, tmp_path):
    G = _golden()[name]
    gen, src, dst, feats, desc, man = _inputs(name, tmp_path)
    n = CF.CONFIGS[name]["nodes"]
    grp = sg.ShardGroup(sg.Graph.from_edges(n, src, dst), sg.Model.load(desc, man), feats, shards)
    _replay(name, grp, gen, src, dst, G, shards_note=f" x{shards} shards")


def test_c1_full_stream_against_oracle(tmp_path):
    """The whole C1 golden stream (300 rounds of 100 updates) through the C
    restatement too, with every table compared every 25 rounds."""
    name = "c1"
    gen, src, dst, feats, desc, man = _inputs(name, tmp_path)
    n, k = CF.CONFIGS[name]["nodes"], CF.CONFIGS[name]["layers"]
    eng = sg.Engine.create_from_array(sg.Graph.from_edges(n, src, dst), sg.Model.load(desc, man), feats)
    orc = oracle.make_oracle(n, src, dst, feats, model_io.load_model(desc, man))
    for i, (ops, ss, dd) in enumerate(CF.batches(name, gen, src, dst, _golden()[name]["rounds"])):
        eng.apply_update(ops, ss, dd)
        assert orc.apply(ops, ss, dd) == 0, orc.last_error()
        assert eng.stats_line() == orc.stats_line(), i
        for layer in range(1, k + 1):
            assert np.array_equal(eng.dirty_nodes(layer), orc.dirty(layer)), (i, layer)
        if (i + 1) % 25 == 0:
            err = tables_equal(eng, orc, k)
            assert err is None, f"round {i}: {err}"
