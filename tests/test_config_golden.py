"""CPU checks of the config-scale golden file (tests/golden/configs.json.gz):
the C restatement reproduces the reference's C1 record (init, every stats line,
every dirty set, final tables), so the oracle is pinned at a BASELINE config
too, and the file's own structure is sane for C2/C3."""
import gzip
import json
import os
import tempfile

import numpy as np

from oracle import model_io, oracle
from tools import configs as CF
from tools.datagen import Generator

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "configs.json.gz")


def test_golden_file_shape():
    G = json.load(gzip.open(GOLDEN, "rt"))
    for name in ("c1", "c2", "c3"):
        rec = G[name]
        k = CF.CONFIGS[name]["layers"]
        assert len(rec["lines"]) == len(rec["dirty"]) == rec["rounds"]
        assert set(rec["init"]) == set(rec["final"]) == {f"m{i}" for i in range(1, k + 2)} | {
            f"a{i}" for i in range(1, k + 1)}
        for line in rec["lines"]:
            kv = dict(t.split("=", 1) for t in line.split())
            assert int(kv["updates"]) == CF.CONFIGS[name]["batch"]
        assert rec["init"]["m1"] != rec["final"]["m2"]


def test_oracle_reproduces_c1_reference_record():
    G = json.load(gzip.open(GOLDEN, "rt"))["c1"]
    name, gen = "c1", Generator()
    n, k = CF.CONFIGS[name]["nodes"], CF.CONFIGS[name]["layers"]
    src, dst = CF.graph(name, gen)
    feats = CF.features(name, gen)
    with tempfile.TemporaryDirectory() as d:
        import paper_2309_11071_b200 as sg  # gen_model only (host code, byte-identical to the reference's)
        desc, man = CF.model_files(name, sg.gen_model, d)
        orc = oracle.make_oracle(n, src, dst, feats, model_io.load_model(desc, man))
    assert CF.table_digests(orc.table, k) == G["init"]
    for i, (ops, ss, dd) in enumerate(CF.batches(name, gen, src, dst, G["rounds"])):
        assert orc.apply(ops, ss, dd) == 0
        assert orc.stats_line() == G["lines"][i], i
        assert CF.dirty_digest(orc.dirty, k) == G["dirty"][i], i
    assert CF.table_digests(orc.table, k) == G["final"]
    assert np.all(np.isfinite(orc.table(k + 1, 0)))
