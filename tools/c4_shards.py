"""BENCHMARK HARNESS — C4's model and partitioning at reduced scale on one GPU.

configs[3] (C4) is a 3-layer GraphSAGE-max, 128-d, papers100M-shape graph
vertex-sharded over 8 B200s. This harness builds the same model on a scaled
R-MAT graph (default 1/64: 1.73M nodes, 25M edges), partitions it over 8
in-process shards (sgnn_b200_group_create: every shard holds only its own rows
of every table, reads the others' through peer memory, and exchanges dirty
lists and pre-images per layer through the device-side mailboxes), runs the
same update stream through the 8-shard group and through one unsharded engine,
and checks per round that the global stats lines and the union of the owners'
dirty sets are identical, then verify() (collective full inference) on the
group. It reports each shard's table / graph bytes next to the unsharded
engine's. The 8 shards time-share one GPU here, so round times are not a
multi-GPU measurement.

    python tools/c4_shards.py [--scale 64] [--rounds 20] [--shards 8]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=64)
    ap.add_argument("--rounds", type=int, default=20)
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--batch", type=int, default=1000)
    args = ap.parse_args()
    import tempfile
    import paper_2309_11071_b200 as sg
    from tools import configs as CF
    from tools.datagen import Generator
    n, e = 111_000_000 // args.scale, 1_600_000_000 // args.scale
    gen = Generator()
    t0 = time.time()
    src, dst = gen.rmat(n, e, CF.GRAPH_SEED)
    feats = gen.features(n, 128, CF.GRAPH_SEED)
    mdir = tempfile.mkdtemp(prefix="sgnn_c4x_")
    sg.gen_model("sage", 128, 128, 3, CF.MODEL_SEED, CF.EPSILON, mdir)
    desc = os.path.join(mdir, "description.txt")
    text = open(desc).read().replace("min\n", "max\n")  # SAGE-max
    open(desc, "w").write(text)
    model = sg.Model.load(desc, os.path.join(mdir, "weights.txt"))
    out = {"workload": f"C4 model (3-layer GraphSAGE-max, 128-d) on a 1/{args.scale}-scale papers100M-shape R-MAT "
                       f"graph ({n} nodes, {e} edges), {args.shards} partitioned shards on one GPU vs one engine",
           "inputs_s": round(time.time() - t0, 1)}
    t0 = time.time()
    grp = sg.ShardGroup(sg.Graph.from_edges(n, src, dst), model, feats, args.shards)
    out["group_create_s"] = round(time.time() - t0, 1)
    t0 = time.time()
    one = sg.Engine.create_from_array(sg.Graph.from_edges(n, src, dst), model, feats)
    out["single_create_s"] = round(time.time() - t0, 1)
    out["shard_ranges"] = grp.ranges
    out["shard_memory"] = grp.memory()
    out["single_memory"] = one.memory()
    ops, ss, dd = gen.rmat_stream(n, src, dst, args.rounds * args.batch, 0.5, CF.STREAM_SEED)
    equal_lines = equal_dirty = 0
    tg, t1 = [], []
    for r in range(args.rounds):
        sl = slice(r * args.batch, (r + 1) * args.batch)
        t = time.perf_counter()
        grp.apply_update(ops[sl], ss[sl], dd[sl])
        tg.append((time.perf_counter() - t) * 1e3)
        t = time.perf_counter()
        one.apply_update(ops[sl], ss[sl], dd[sl])
        t1.append((time.perf_counter() - t) * 1e3)
        equal_lines += grp.stats_line() == one.stats_line()
        equal_dirty += all(np.array_equal(grp.dirty_nodes(l), one.dirty_nodes(l)) for l in range(1, 4))
    st, where = grp.verify()
    out.update({"rounds": args.rounds, "stats_lines_equal": equal_lines, "dirty_sets_equal": equal_dirty,
                "group_verify": "ok" if st == 0 else str(where), "last_stats": one.stats_line(),
                "group_round_ms_p50": float(np.median(tg)), "single_round_ms_p50": float(np.median(t1)),
                "table_bytes_ratio_max_shard_over_single":
                    max(m["tables"] for m in out["shard_memory"]) / out["single_memory"]["tables"]})
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
