"""BENCHMARK HARNESS — C4-scale ingest.

Generates the papers100M-shape R-MAT graph of configs[3] (111M nodes, 1.6B
edges, seed 2024, the harness generator of tools/rmat_gen.hpp), writes it as a
binary edge list (sgnn_b200_graph_save_binary's format), and times the
product's sgnn_b200_graph_load_binary: read + the text loader's validation
(first failing edge decides) + adjacency build. Prints one JSON line.

    python tools/c4_ingest.py [--nodes N] [--edges E] [--path /tmp/c4.bin]
"""
import argparse
import json
import os
import resource
import struct
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, default=111_000_000)
    ap.add_argument("--edges", type=int, default=1_600_000_000)
    ap.add_argument("--path", default="/tmp/sgnn_c4_edges.bin")
    args = ap.parse_args()
    import paper_2309_11071_b200 as sg
    from tools.datagen import Generator
    out = {"nodes": args.nodes, "edges": args.edges, "threads": os.cpu_count()}
    t = time.time()
    if not (os.path.exists(args.path) and os.path.getsize(args.path) == 24 + 8 * args.edges):
        src, dst = Generator().rmat(args.nodes, args.edges, 2024)
        out["generate_s"] = round(time.time() - t, 1)
        t = time.time()
        with open(args.path, "wb") as f:
            f.write(b"SGNNEDG1" + struct.pack("<IIQ", args.nodes, 0, len(src)))
            f.write(src.tobytes())
            f.write(dst.tobytes())
        del src, dst
        out["write_s"] = round(time.time() - t, 1)
    out["file_gb"] = round(os.path.getsize(args.path) / 1e9, 2)
    t = time.time()
    g = sg.Graph.load_binary(args.path)
    out["load_binary_s"] = round(time.time() - t, 1)
    out["loaded_nodes"], out["loaded_edges"] = g.num_nodes, g.num_edges
    out["peak_rss_gb"] = round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
