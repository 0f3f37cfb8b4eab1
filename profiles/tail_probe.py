"""Where do the slow rounds go? (VERDICT r01 "cut the hub tail")

    python profiles/tail_probe.py [--config c2] [--rounds 100] [--out FILE]

Replays the bench stream (same seeds, same warm-up) through one engine with the
per-kernel-class CUDA events on, L2 flushed before every round, and writes per
round: the class times, the recompute bytes, and the stats-line counters that
explain them (exposed resets and fetched rows per layer). Run under gpurun;
measurement tooling only (not part of the product or the bench line).
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from tools import configs as CF  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--rounds", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--ncu-round", type=int, default=-1,
                    help="bracket this round (stream index) with cudaProfilerStart/Stop for "
                         "`ncu --profile-from-start off` (timings of that run are not measurements)")
    args = ap.parse_args()
    import torch
    import paper_2309_11071_b200 as sg
    cfg = CF.CONFIGS[args.config]
    gen, src, dst, feats, desc, man = bench.product_inputs(args.config)
    stream = CF.batches(args.config, gen, src, dst, args.warmup + args.rounds, seed=CF.STREAM_SEED, batch=cfg["batch"])
    eng = sg.Engine.create_from_array(sg.Graph.from_edges(cfg["nodes"], src, dst), sg.Model.load(desc, man), feats)
    dev = [(torch.frombuffer(bytearray(o), dtype=torch.uint8).cuda(), torch.from_numpy(s.astype(np.int32)).cuda(),
            torch.from_numpy(d.astype(np.int32)).cuda()) for o, s, d in stream]
    B = cfg["batch"]
    for o, s, d in dev[:args.warmup]:
        eng.apply_update_device(o.data_ptr(), s.data_ptr(), d.data_ptr(), B)
    eng.set_option("profile_kernels", 1)
    rows = []
    for i, (o, s, d) in enumerate(dev[args.warmup:]):
        eng.flush_l2()
        mark = args.warmup + i == args.ncu_round
        if mark:
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStart()
        eng.apply_update_device(o.data_ptr(), s.data_ptr(), d.data_ptr(), B)
        if mark:
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStop()
        kt = eng.kernel_times()
        st = dict(kv.split("=") for kv in eng.stats_line().split() if "=" in kv)
        rows.append({"round": args.warmup + i, **{k: round(v, 4) for k, v in kt.items()},
                     **{k: int(v) for k, v in st.items() if k.startswith(("l1.", "l2.", "l3."))
                        and k.split(".")[1] in ("exposed_reset", "recomputes", "fetch_rows", "dirty", "targets")}})
    tot = [r["total"] for r in rows]
    med = statistics.median(tot)
    summary = {"config": args.config, "rounds": len(rows), "p50_ms": med, "mean_ms": statistics.mean(tot),
               "p90_ms": float(np.percentile(tot, 90)), "max_ms": max(tot),
               "slow_rounds": [r for r in rows if r["total"] > 1.5 * med]}
    classes = ("graph_update", "events", "sort_group", "classify", "recompute", "compact", "combine", "finalize",
               "commit")
    summary["mean_by_class_ms"] = {c: statistics.mean(r[c] for r in rows) for c in classes}
    summary["median_by_class_ms"] = {c: statistics.median(r[c] for r in rows) for c in classes}
    summary["excess_over_median_by_class_ms"] = {
        c: sum(r[c] - summary["median_by_class_ms"][c] for r in summary["slow_rounds"]) / len(rows) for c in classes}
    out = json.dumps({"summary": summary, "rounds": rows}, indent=1)
    if args.out:
        open(args.out, "w").write(out)
    print(json.dumps({k: v for k, v in summary.items() if k != "slow_rounds"}, indent=1))
    for r in summary["slow_rounds"]:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
