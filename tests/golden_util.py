"""Access to the reference-generated golden fixtures (tests/golden/)."""
from __future__ import annotations

import functools
import gzip
import hashlib
import json
import os

import numpy as np

from oracle import model_io

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
DATA = os.path.join(GOLDEN, "data")


@functools.lru_cache(maxsize=1)
def expected():
    with gzip.open(os.path.join(GOLDEN, "expected.json.gz"), "rt") as f:
        return json.load(f)


def case_names():
    return sorted(expected()["cases"])


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def load_case(name):
    c = expected()["cases"][name]
    d = os.path.join(DATA, c["dataset"])
    src, dst = model_io.read_edge_list(os.path.join(d, "edges.txt"))
    feats = model_io.read_tnsr(os.path.join(d, "features.tnsr"))
    ops, ss, dd = model_io.read_stream(os.path.join(d, "stream.txt"))
    desc = os.path.join(d, c["model"], "description.txt")
    man = os.path.join(d, c["model"], "weights.txt")
    return c, (src, dst), feats, (ops, ss, dd), desc, man


def replay(c, stream, apply, stats_line, dirty, table):
    """Drives one engine through a golden case and checks every recorded value."""
    ops, ss, dd = stream
    k, batch = c["layers"], c["batch"]

    def tables():
        out = {}
        for layer in range(1, k + 2):
            for stage in (0, 1):
                if stage == 1 and layer > k:
                    continue
                out[f"{layer}.{stage}"] = digest(table(layer, stage))
        return out

    assert tables() == c["init_tables"], "initial full inference differs from the reference"
    for r, exp in enumerate(c["rounds"]):
        i = r * batch
        apply(ops[i:i + batch], ss[i:i + batch], dd[i:i + batch])
        assert stats_line() == exp["line"], f"round {r}\n got {stats_line()}\n ref {exp['line']}"
        for layer in range(1, k + 1):
            got = list(map(int, dirty(layer)))
            assert got == exp["dirty"][layer - 1], f"round {r} layer {layer} dirty set"
        if "tables" in exp:
            assert tables() == exp["tables"], f"round {r} tables differ"
    assert tables() == c["final_tables"], "final tables differ"
