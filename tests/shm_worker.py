"""One rank of tests/test_gpu_sharded.py::test_shm_two_processes_one_gpu.

    python tests/shm_worker.py NAME RANK WORLD DATA_DIR DESC MANIFEST OUT_JSON

Creates shard RANK of WORLD over the shared-memory transport NAME (CUDA IPC
for the peers' tables and pack buffers), replays DATA_DIR/stream.txt in
batches of 10 beside the C restatement (oracle, test infrastructure), and
writes what it saw: every round's stats line, and any mismatch of the stats
line, of this shard's dirty nodes or of its table rows against the oracle.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2309_11071_b200 as sg  # noqa: E402
from oracle import model_io, oracle  # noqa: E402


def main():
    name, rank, world, data, desc, man, out = sys.argv[1:8]
    rank, world = int(rank), int(world)
    src, dst = model_io.read_edge_list(os.path.join(data, "edges.txt"))
    feats = model_io.read_tnsr(os.path.join(data, "features.tnsr"))
    ops, ss, dd = model_io.read_stream(os.path.join(data, "stream.txt"))
    n = feats.shape[0]
    m = sg.Model.load(desc, man)
    k = m.num_layers
    e = sg.Engine.create_shm(name, rank, world, sg.Graph.from_edges(n, src, dst), m, feats)
    lo, hi = e.shard_range()
    orc = oracle.make_oracle(n, src, dst, feats, model_io.load_model(desc, man))
    lines, errors = [], []

    def check_tables(tag):
        for layer in range(1, k + 2):
            for stage in (0, 1):
                if stage == 1 and layer > k:
                    continue
                got = e.read_rows(layer, stage, lo, hi)
                want = orc.table(layer, stage)[lo:hi]
                if got.tobytes() != want.tobytes():
                    errors.append(f"{tag}: table ({layer}, {stage}) rows [{lo}, {hi}) differ")

    check_tables("init")
    rounds = 0
    for i in range(0, len(ss), 10):
        e.apply_update(ops[i:i + 10], ss[i:i + 10], dd[i:i + 10])
        if orc.apply(ops[i:i + 10], ss[i:i + 10], dd[i:i + 10]) != 0:
            errors.append(f"round {rounds}: oracle rejected the batch")
            break
        line = e.stats_line()
        lines.append(line)
        if line != orc.stats_line():
            errors.append(f"round {rounds}: stats\n gpu {line}\n orc {orc.stats_line()}")
        for layer in range(1, k + 1):
            mine = e.dirty_nodes(layer)
            mine = mine[(mine >= lo) & (mine < hi)]
            want = orc.dirty(layer)
            want = want[(want >= lo) & (want < hi)]
            if not np.array_equal(mine, want):
                errors.append(f"round {rounds}: layer {layer} owned dirty nodes differ")
        rounds += 1
        if errors:
            break
    check_tables("final")
    st, where = e.verify()  # collective: every rank calls it
    if st != 0:
        errors.append(f"verify: {where}")
    json.dump({"rank": rank, "range": [lo, hi], "rounds": rounds, "lines": lines, "errors": errors,
               "memory": e.memory()}, open(out, "w"))


if __name__ == "__main__":
    main()
