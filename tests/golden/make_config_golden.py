"""Generates tests/golden/configs.json.gz: the UNMODIFIED reference (oracle/_ref,
compiled from /root/reference by oracle/ref.mk) run at BASELINE.json's own
configurations C1, C2 and C3 (tools/configs.py), from its OWN initial full
inference (CheckpointStore::init_full_inference, checkpoint.cpp:105-145).

Recorded per config:
  init   — sha256 prefixes of every table after the reference's init;
  lines  — the stats line of every round (RoundStats::to_line, stats.cpp:20-48);
  dirty  — per round, per layer: (count, sha256 of the ascending dirty ids)
           (Engine::last_dirty_nodes, engine.hpp:99-100);
  final  — table digests after the last round.
Inputs come from the harness generator compiled into oracle/_ref and the
reference's own sgnn_gen_model, so nothing here loads the product library.

Run in the build container (needs /root/reference built into oracle/_ref and a
few GB of RAM; C2's single-threaded init takes ~1-2 min):
    python tests/golden/make_config_golden.py [c1 c2 c3]
The GPU tests (tests/test_gpu_configs.py) and bench.py's parity block replay
the same inputs through the product and compare against this file.
"""
from __future__ import annotations

import gzip
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from tools import configs as CF  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "configs.json.gz")
ROUNDS = {"c1": 300, "c2": 25, "c3": 60}


def run(name):
    cfg = CF.CONFIGS[name]
    gen = O.ref_generator()
    t0 = time.time()
    src, dst = CF.graph(name, gen, log=print)
    feats = CF.features(name, gen)
    mdir = tempfile.mkdtemp(prefix=f"golden_{name}_")
    desc, man = CF.model_files(name, O.ref_gen_model, mdir)
    stream = CF.batches(name, gen, src, dst, ROUNDS[name])
    print(f"[{name}] inputs {time.time() - t0:.1f}s", flush=True)
    t0 = time.time()
    ref = O.RefEngine(cfg["nodes"], src, dst, feats, desc, man)
    print(f"[{name}] reference init {time.time() - t0:.1f}s", flush=True)
    k = cfg["layers"]
    rec = {"workload": cfg["workload"], "rounds": ROUNDS[name], "batch": cfg["batch"],
           "stream_seed": CF.STREAM_SEED, "init": CF.table_digests(ref.table, k), "lines": [], "dirty": [],
           "ms": []}
    for ops, ss, dd in stream:
        rec["ms"].append(round(ref.apply_timed(ops, ss, dd), 3))
        rec["lines"].append(ref.stats_line())
        rec["dirty"].append(CF.dirty_digest(ref.dirty, k))
    rec["final"] = CF.table_digests(ref.table, k)
    print(f"[{name}] {ROUNDS[name]} rounds, median {sorted(rec['ms'])[len(rec['ms']) // 2]} ms", flush=True)
    return rec


def main():
    names = sys.argv[1:] or ["c1", "c2", "c3"]
    data = {}
    if os.path.exists(OUT):
        data = json.load(gzip.open(OUT, "rt"))
    for n in names:
        data[n] = run(n)
        with gzip.open(OUT, "wt") as f:
            json.dump(data, f)


if __name__ == "__main__":
    main()
