"""Whole-graph inference at C2 shape in the three combination modes (exact,
3xTF32, TF32), timed with CUDA events around sgnn_engine_set_option
("combination_mode", m) — which recomputes every table — and the per-value
error of each tensor-core mode against the exact tables. Run under ncu with
-k regex:k_gemm to read the tensor-pipe utilisation of k_gemm_tc.

    python profiles/tc_gemm_probe.py [c2|c3]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (benchmark inputs only)


def main():
    import torch
    import paper_2309_11071_b200 as sg
    key = sys.argv[1] if len(sys.argv) > 1 else "c2"
    cfg = bench.CONFIGS[key]
    _, src, dst, feats, desc, man = bench.product_inputs(key)
    m = sg.Model.load(desc, man)
    t0 = time.time()
    eng = sg.Engine.create_from_array(sg.Graph.from_edges(cfg["nodes"], src, dst), m, feats)
    exact = {(layer, stage): eng.read_table(layer, stage) for layer in range(2, cfg["layers"] + 2)
             for stage in (0, 1) if not (stage == 1 and layer > cfg["layers"])}
    out = {"config": cfg["workload"], "create_s": time.time() - t0, "modes": {},
           "tma": os.environ.get("SGNN_B200_TMA", "1") != "0"}
    est = torch.cuda.ExternalStream(eng.stream)
    for mode in (2, 1, 0):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(est)
        eng.set_option("combination_mode", mode)
        b.record(est)
        torch.cuda.synchronize()
        worst_abs = worst_rel = 0.0
        for (layer, stage), ref in exact.items():
            got = eng.read_table(layer, stage)
            err = np.abs(ref.astype(np.float64) - got)
            worst_abs = max(worst_abs, float(err.max()))
            worst_rel = max(worst_rel, float((err / np.maximum(1.0, np.abs(ref))).max()))
        out["modes"][{0: "exact", 1: "3xtf32", 2: "tf32"}[mode]] = {
            "set_option_wall_ms_incl_host_feature_upload": a.elapsed_time(b), "max_abs_err": worst_abs, "max_rel_err": worst_rel}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
