"""Shared helpers: datasets, model files and product-vs-oracle stream runs."""
from __future__ import annotations

import os

import numpy as np

import paper_2309_11071_b200 as sg
from oracle import model_io, oracle


def make_dataset(d, nodes=300, deg=6.0, feat=16, stream=120, seed=2024, insert_fraction=0.6):
    sg.gen_synthetic(d, num_nodes=nodes, avg_degree=deg, feature_len=feat, stream_len=stream, seed=seed,
                     insert_fraction=insert_fraction)
    return d


def make_model(d, kind, feat, hidden, layers, seed=7, eps=0.1, agg=None, name=None):
    """Reference-generated model; agg='max'/'min' rewrites the aggregation lines."""
    md = os.path.join(d, name or f"{kind}_{agg or 'def'}_{layers}_{hidden}")
    sg.gen_model(kind, feat, hidden, layers, seed, eps, md)
    desc = os.path.join(md, "description.txt")
    if agg:
        text = open(desc).read().replace("min\n", f"{agg}\n").replace("max\n", f"{agg}\n")
        open(desc, "w").write(text)
    return desc, os.path.join(md, "weights.txt")


def write_custom_model(d, name, text, weights: dict, epsilon: dict | None = None):
    md = os.path.join(d, name)
    os.makedirs(md, exist_ok=True)
    lines = []
    for k, v in weights.items():
        model_io.write_tnsr(os.path.join(md, k + ".tnsr"), np.asarray(v, dtype=np.float32))
        lines.append(f"{k} {k}.tnsr")
    for layer, e in (epsilon or {}).items():
        lines.append(f"epsilon {layer} {e}")
    open(os.path.join(md, "weights.txt"), "w").write("\n".join(lines) + "\n")
    open(os.path.join(md, "description.txt"), "w").write(text)
    return os.path.join(md, "description.txt"), os.path.join(md, "weights.txt")


def tables_equal(engine, orc, k):
    for layer in range(1, k + 2):
        for stage in (0, 1):
            if stage == 1 and layer > k:
                continue
            a = engine.read_table(layer, stage)
            b = orc.table(layer, stage)
            if a.tobytes() != b.tobytes():
                bad = np.argwhere(a.view(np.uint32) != b.view(np.uint32))
                return f"layer {layer} stage {stage}: {len(bad)} differing values, first at {bad[0].tolist()}"
    return None


def run_parity(d, desc, man, batch, edges=None, features=None, stream=None, options=(), check_every=1,
               rounds=None, shards=None):
    """Runs the same stream through the product (GPU) and the oracle; asserts
    bitwise equality of stats lines, dirty sets and tables."""
    if edges is None:
        src, dst = model_io.read_edge_list(os.path.join(d, "edges.txt"))
        feats = model_io.read_tnsr(os.path.join(d, "features.tnsr"))
        ops, ss, dd = model_io.read_stream(os.path.join(d, "stream.txt"))
        n = feats.shape[0]
    else:
        src, dst = edges
        feats = features
        ops, ss, dd = stream
        n = feats.shape[0]
    m = sg.Model.load(desc, man)
    if shards:  # owner-computes shard group in this process (one thread per shard)
        e = sg.ShardGroup(sg.Graph.from_edges(n, src, dst), m, feats, shards)
    else:
        e = sg.Engine.create_from_array(sg.Graph.from_edges(n, src, dst), m, feats)
    orc = oracle.make_oracle(n, src, dst, feats, model_io.load_model(desc, man))
    for name, value in options:
        e.set_option(name, value)
        assert orc.set_option(name, value) == 0
    k = m.num_layers
    err = tables_equal(e, orc, k)
    assert err is None, "after init: " + err
    r = 0
    for i in range(0, len(ss), batch):
        if rounds is not None and r >= rounds:
            break
        e.apply_update(ops[i:i + batch], ss[i:i + batch], dd[i:i + batch])
        assert orc.apply(ops[i:i + batch], ss[i:i + batch], dd[i:i + batch]) == 0, orc.last_error()
        assert e.stats_line() == orc.stats_line(), f"round {r}\n gpu {e.stats_line()}\n orc {orc.stats_line()}"
        for layer in range(1, k + 1):
            a, b = e.dirty_nodes(layer), orc.dirty(layer)
            assert np.array_equal(a, b), f"round {r} layer {layer} dirty sets differ ({len(a)} vs {len(b)})"
        if (r + 1) % check_every == 0:
            err = tables_equal(e, orc, k)
            assert err is None, f"round {r}: {err}"
        r += 1
    err = tables_equal(e, orc, k)
    assert err is None, "final: " + err
    st, where = e.verify()
    assert st == 0, where
    return e, orc
