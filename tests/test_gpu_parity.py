"""GPU parity: the product C ABI (sm_100a kernels) against the C restatement.

Each case runs one update stream through both and requires, after every round,
identical stats lines (reference stats.cpp:20-48 format), identical per-layer
dirty sets (engine.hpp:99-100) and bitwise-identical tables (checkpoint
semantics of proj/src/core/checkpoint.cpp), then a full-inference verify on the
device (baseline.cpp:234-256). Tolerance: none — the combination runs in exact
mode (serial-k, separately rounded fp32), so embeddings are bit-exact too.
"""
import numpy as np
import pytest

from tests import util

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def data(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("parity"))
    return util.make_dataset(d, nodes=300, deg=6.0, feat=16, stream=120)


@pytest.mark.parametrize("kind,layers", [("gcn", 2), ("sage", 2), ("gin", 3)])
@pytest.mark.parametrize("agg", [None, "max"])
@pytest.mark.parametrize("batch", [1, 7, 40])
def test_stream_parity_small(data, kind, layers, agg, batch):
    desc, man = util.make_model(data, kind, 16, 16 if kind != "gin" else 8, layers, agg=agg)
    util.run_parity(data, desc, man, batch)


@pytest.mark.parametrize("feat,hidden", [(100, 64), (200, 130), (602, 256), (1100, 40)])
def test_stream_parity_wide_rows(tmp_path, feat, hidden):
    """Row widths covering every per-lane vector count of the classify/aggregate kernels."""
    d = util.make_dataset(str(tmp_path), nodes=250, deg=8.0, feat=feat, stream=60, seed=11)
    desc, man = util.make_model(d, "gcn", feat, hidden, 2, agg="max")
    util.run_parity(d, desc, man, 10, check_every=3)


@pytest.mark.parametrize("summary", ["1", "0"])
@pytest.mark.parametrize("agg", ["min", "max"])
@pytest.mark.parametrize("hidden,nodes,deg", [(130, 600, 300.0), (300, 250, 8.0), (700, 250, 8.0)])
def test_filter_bound_codes_signed_rows(tmp_path, monkeypatch, summary, agg, hidden, nodes, deg):
    """Layer-2 rows of > 128 floats through the filter's pre-tests: the float
    per-target summary (default) and, with SGNN_B200_SUMMARY=0, the 16-bit
    alpha bound codes (CPL 2 / 4 / 8); no ReLU, so messages and aggregates are
    signed, for both aggregation directions (min is oriented as negated max)."""
    monkeypatch.setenv("SGNN_B200_SUMMARY", summary)
    d = util.make_dataset(str(tmp_path), nodes=nodes, deg=deg, feat=40, stream=60, seed=19)
    rng = np.random.default_rng(hidden)
    w = {"W1": rng.uniform(-0.5, 0.5, (hidden, 40)), "W2": rng.uniform(-0.5, 0.5, (8, hidden))}
    text = f"{agg}\nlin W1\n{agg}\nlin W2\n"
    desc, man = util.write_custom_model(d, f"signed_{agg}_{hidden}", text, w)
    util.run_parity(d, desc, man, 6, check_every=2)


def test_options_duplicate_and_baseline(data):
    desc, man = util.make_model(data, "gcn", 16, 16, 2)
    util.run_parity(data, desc, man, 5, options=[("duplicate_seed_events", 1), ("baseline_counters", 1)])


@pytest.mark.parametrize("kind,layers,agg", [("gcn", 2, "max"), ("sage", 2, None), ("gin", 3, "max")])
def test_emit_changed_only(data, kind, layers, agg):
    """North-star item 5: next-layer events only from changed messages; the
    oracle runs the same option, so counters are pinned too (and tables / dirty
    sets equal the reference's, tests/test_oracle.py)."""
    desc, man = util.make_model(data, kind, 16, 16 if kind != "gin" else 8, layers, agg=agg)
    util.run_parity(data, desc, man, 6, options=[("emit_changed_only", 1)])


def test_emit_changed_only_saturated_messages(data):
    """A layer whose ReLU output is 0 for every node: every dirty node's next
    message is unchanged, so the gated mode emits no expansion events at all."""
    rng = np.random.default_rng(5)
    w = {"W0": -rng.uniform(0.1, 0.5, (8, 16)), "b0": np.zeros(8), "W1": rng.uniform(-0.3, 0.5, (6, 8)),
         "b1": np.full(6, 0.1)}
    text = "max\nlin W0 bias b0\nrelu\nmax\nlin W1 bias b1\nrelu\n"
    desc, man = util.write_custom_model(data, "sat", text, w)
    e, _ = util.run_parity(data, desc, man, 6, options=[("emit_changed_only", 1)])
    kv = dict(t.split("=") for t in e.stats_line().split())
    assert int(kv["l2.events"]) == int(kv["l1.events"])  # seeds only


def test_prefix_model(data):
    rng = np.random.default_rng(60)
    w = {"W0": rng.uniform(-0.3, 0.5, (6, 16)), "W1": rng.uniform(-0.3, 0.5, (6, 6)),
         "b1": np.array([0.1, 0.2, 0.0, 0.1, 0.2, 0.0]), "W2": rng.uniform(-0.3, 0.5, (4, 6)),
         "b2": np.array([0.1, 0.0, 0.2, 0.1])}
    text = "lin W0\nmin\nlin W1 bias b1\nrelu\nmin\nlin W2 bias b2\nrelu\n"
    desc, man = util.write_custom_model(data, "prefix", text, w)
    util.run_parity(data, desc, man, 3, options=[("baseline_counters", 1)])


def test_identity_model(data):
    desc, man = util.write_custom_model(data, "ident", "max\nmax\n", {})
    util.run_parity(data, desc, man, 4)


@pytest.mark.parametrize("summary", ["1", "0"])
@pytest.mark.parametrize("agg", ["min", "max"])
def test_filter_bound_codes_constant_columns(tmp_path, monkeypatch, summary, agg):
    """Alpha columns that are constant (zero step: the grid collapses to its
    base; the summary's normalisation falls back to inv 1), all-zero, or
    two-valued, next to random ones, 200 wide (summary and bound codes)."""
    import os
    monkeypatch.setenv("SGNN_B200_SUMMARY", summary)
    from oracle import model_io
    d = util.make_dataset(str(tmp_path), nodes=400, deg=40.0, feat=200, stream=80, seed=23)
    f = model_io.read_tnsr(os.path.join(d, "features.tnsr"))
    f[:, :50] = 0.5
    f[:, 50:100] = 0.0
    f[:, 100:120] = np.where(np.arange(f.shape[0])[:, None] % 2 == 0, 0.25, 0.75)
    # near-ties: values 0-2 ulps below 1 (PAIRs within float rounding of alpha,
    # where the summary's directed rounding must keep the PAIR open)
    rng = np.random.default_rng(29)
    one = np.float32(1.0)
    ulps = np.array([one, np.nextafter(one, np.float32(0)), np.nextafter(np.nextafter(one, np.float32(0)), np.float32(0))],
                    dtype=np.float32)
    f[:, 120:140] = ulps[rng.integers(0, 3, size=(f.shape[0], 20))]
    # extreme magnitudes: column ranges that overflow (step inf) or sit near the
    # denormal range
    f[:, 140:145] = rng.choice(np.array([-3e38, 3e38, 1e30], dtype=np.float32), size=(f.shape[0], 5))
    f[:, 145:150] = (rng.random((f.shape[0], 5)) * 1e-37).astype(np.float32)
    model_io.write_tnsr(os.path.join(d, "features.tnsr"), f)
    desc, man = util.write_custom_model(d, f"ident_{agg}", f"{agg}\n{agg}\n", {})
    util.run_parity(d, desc, man, 8, check_every=2)


def test_hub_multichunk_recompute(tmp_path):
    """Hubs with > 512 in-neighbours exercise the multi-chunk atomic reduction."""
    rng = np.random.default_rng(5)
    n = 3000
    src = list(range(1, n))           # every node -> hub 0
    dst = [0] * (n - 1)
    extra = rng.integers(1, n, size=(6000, 2))
    seen = set(zip(src, dst))
    for a, b in extra:
        if a != b and (a, b) not in seen:
            seen.add((int(a), int(b)))
            src.append(int(a))
            dst.append(int(b))
    feats = rng.random((n, 24), dtype=np.float32)
    # stream: delete and re-insert edges into the hub (exposed resets on a 3000-in-degree target)
    ops, ss, dd = [], [], []
    for u in rng.choice(np.arange(1, n), size=60, replace=False):
        ops.append("-"); ss.append(int(u)); dd.append(0)
    for u in rng.choice(np.arange(1, n), size=30, replace=False):
        if ("-", int(u)) in zip(ops, ss):
            ops.append("+"); ss.append(int(u)); dd.append(0)
    d = str(tmp_path)
    desc, man = util.make_model(d, "gcn", 24, 16, 2, agg="max")
    stream = ("".join(ops).encode(), np.array(ss, dtype=np.uint32), np.array(dd, dtype=np.uint32))
    util.run_parity(d, desc, man, 9, edges=(np.array(src, np.uint32), np.array(dst, np.uint32)), features=feats,
                    stream=stream)


def test_slab_relocation(tmp_path):
    """Many inserts into one vertex per round overflow its slab and relocate it."""
    rng = np.random.default_rng(9)
    n = 2000
    src = rng.integers(0, n, 4000)
    dst = rng.integers(0, n, 4000)
    pairs = sorted({(int(a), int(b)) for a, b in zip(src, dst) if a != b})
    src = np.array([p[0] for p in pairs], np.uint32)
    dst = np.array([p[1] for p in pairs], np.uint32)
    present = set(pairs)
    feats = rng.random((n, 16), dtype=np.float32)
    ops, ss, dd = [], [], []
    for v in range(1, 1200):
        for e in ((7, v), (v, 11)):
            if e[0] != e[1] and e not in present:
                present.add(e)
                ops.append("+"); ss.append(e[0]); dd.append(e[1])
    stream = ("".join(ops).encode(), np.array(ss, np.uint32), np.array(dd, np.uint32))
    desc, man = util.make_model(str(tmp_path), "sage", 16, 16, 2, agg="max")
    util.run_parity(str(tmp_path), desc, man, 300, edges=(src, dst), features=feats, stream=stream)


def _hub_case(tmp_path, feat=24, n=3000, seed=5):
    rng = np.random.default_rng(seed)
    src = list(range(1, n))
    dst = [0] * (n - 1)
    seen = set(zip(src, dst))
    for a, b in rng.integers(1, n, size=(8000, 2)):
        if a != b and (int(a), int(b)) not in seen:
            seen.add((int(a), int(b)))
            src.append(int(a))
            dst.append(int(b))
    feats = rng.random((n, feat), dtype=np.float32)
    edges = list(zip(src, dst))
    pick = rng.choice(len(edges), size=400, replace=False)
    ops = "".join("-" for _ in pick).encode()
    ss = np.array([edges[i][0] for i in pick], np.uint32)
    dd = np.array([edges[i][1] for i in pick], np.uint32)
    return (np.array(src, np.uint32), np.array(dst, np.uint32)), feats, (ops, ss, dd)


@pytest.mark.parametrize("sparse", ["1", "0"])
def test_sparse_and_dense_recompute(tmp_path, monkeypatch, capfd, sparse):
    """Exposed resets with few uncovered positions take the sparse recompute
    (per-position gathers); with SGNN_B200_SPARSE=0 every one takes the dense
    row path. Both must stay bit-exact; the trace proves which path ran."""
    monkeypatch.setenv("SGNN_B200_SPARSE", sparse)
    monkeypatch.setenv("SGNN_B200_TRACE", "1")
    edges, feats, stream = _hub_case(tmp_path)
    d = str(tmp_path)
    desc, man = util.make_model(d, "gcn", 24, 16, 2, agg="max")
    util.run_parity(d, desc, man, 25, edges=edges, features=feats, stream=stream)
    err = capfd.readouterr().err
    sparse_slots = sum(int(t.split("=")[1]) for t in err.split() if t.startswith("sparse="))
    dense_items = sum(int(t.split("=")[1]) for t in err.split() if t.startswith("work="))
    if sparse == "1":
        assert sparse_slots > 0 and dense_items > 0, (sparse_slots, dense_items)
    else:
        assert sparse_slots == 0 and dense_items > 0


def _kv(line):
    return {k: int(v) for k, v in (t.split("=", 1) for t in line.split())}


@pytest.mark.parametrize("kind,layers,agg", [("gcn", 2, "max"), ("sage", 2, None), ("gin", 3, "max")])
@pytest.mark.parametrize("batch", [1, 12])
def test_khop_recompute_matches_incremental(data, kind, layers, agg, batch):
    """The k-hop comparator (baseline::affected_inference, baseline.cpp:177-207)
    and the incremental path must leave bit-identical tables after every round;
    the comparator's counted row reads equal the reference's
    affected_fetch_count (baseline.cpp:209-222) for the same delta."""
    from oracle import model_io
    import os
    import paper_2309_11071_b200 as sg
    desc, man = util.make_model(data, kind, 16, 16 if kind != "gin" else 8, layers, agg=agg)
    src, dst = model_io.read_edge_list(os.path.join(data, "edges.txt"))
    feats = model_io.read_tnsr(os.path.join(data, "features.tnsr"))
    ops, ss, dd = model_io.read_stream(os.path.join(data, "stream.txt"))
    n = feats.shape[0]
    m = sg.Model.load(desc, man)
    inc = sg.Engine.create_from_array(sg.Graph.from_edges(n, src, dst), m, feats)
    kh = sg.Engine.create_from_array(sg.Graph.from_edges(n, src, dst), m, feats)
    inc.set_option("baseline_counters", 1)
    kh.set_option("khop_recompute", 1)
    k = m.num_layers
    for r, i in enumerate(range(0, len(ss), batch)):
        inc.apply_update(ops[i:i + batch], ss[i:i + batch], dd[i:i + batch])
        kh.apply_update(ops[i:i + batch], ss[i:i + batch], dd[i:i + batch])
        a, b = _kv(inc.stats_line()), _kv(kh.stats_line())
        assert b["ckpt_fetches"] + b["feat_fetches"] == a["affected_fetches"], (r, a, b)
        assert b[f"l{k}.recomputes"] == a["area_nodes"], (r, a, b)
        if r % 3 == 0 or i + batch >= len(ss):
            for layer in range(1, k + 2):
                for stage in (0, 1):
                    if stage == 1 and layer > k:
                        continue
                    x, y = inc.read_table(layer, stage), kh.read_table(layer, stage)
                    assert x.tobytes() == y.tobytes(), f"round {r} layer {layer} stage {stage}"
    st, where = kh.verify()
    assert st == 0, where


def test_khop_recompute_wide_and_hub(tmp_path):
    """Comparator on 602-wide rows (bulk-copy aggregation) and a > 512 in-degree hub."""
    import paper_2309_11071_b200 as sg
    edges, feats, stream = _hub_case(tmp_path, feat=602, n=1500, seed=8)
    d = str(tmp_path)
    desc, man = util.make_model(d, "gcn", 602, 64, 2, agg="max")
    m = sg.Model.load(desc, man)
    n = feats.shape[0]
    inc = sg.Engine.create_from_array(sg.Graph.from_edges(n, *edges), m, feats)
    kh = sg.Engine.create_from_array(sg.Graph.from_edges(n, *edges), m, feats)
    kh.set_option("khop_recompute", 1)
    ops, ss, dd = stream
    for i in range(0, 200, 25):
        inc.apply_update(ops[i:i + 25], ss[i:i + 25], dd[i:i + 25])
        kh.apply_update(ops[i:i + 25], ss[i:i + 25], dd[i:i + 25])
    for layer, stage in ((1, 1), (2, 0), (2, 1), (3, 0)):
        assert inc.read_table(layer, stage).tobytes() == kh.read_table(layer, stage).tobytes(), (layer, stage)


@pytest.mark.parametrize("batch,k1", [(1500, "cluster"), (2048, "cluster"), (2000, "pre"), (2000, "one"),
                                      (4096, "one"), (4097, "sort"), (6000, "sort")])
def test_batch_paths_grouping_and_sort(tmp_path, monkeypatch, batch, k1):
    """Batches up to 2048 updates are grouped by an 8-CTA cluster
    (k_batch_cluster; SGNN_B200_K1CLUSTER=0: one CTA with prefetched state,
    k_batch_group_pre; SGNN_B200_K1PRE=0 too: k_batch_group), up to 4096 by one
    CTA (k_batch_group, hash table in shared memory); larger ones take the
    radix-sort path. All must give the reference's net delta and first-failure
    semantics — including repeated keys inside one batch (insert, delete,
    re-insert of one edge)."""
    if k1 in ("pre", "one"):
        monkeypatch.setenv("SGNN_B200_K1CLUSTER", "0")
    if k1 == "one":
        monkeypatch.setenv("SGNN_B200_K1PRE", "0")
    rng = np.random.default_rng(batch)
    n = 3000
    pairs = {(int(a), int(b)) for a, b in rng.integers(0, n, size=(12000, 2)) if a != b}
    base = sorted(pairs)[:9000]
    src = np.array([p[0] for p in base], np.uint32)
    dst = np.array([p[1] for p in base], np.uint32)
    present = set(base)
    ops, ss, dd = [], [], []
    while len(ss) < batch:
        if rng.random() < 0.5 and present:
            e = base[int(rng.integers(0, len(base)))]
            if e in present:
                present.discard(e); ops.append("-"); ss.append(e[0]); dd.append(e[1])
                if rng.random() < 0.3:  # re-insert within the same batch
                    present.add(e); ops.append("+"); ss.append(e[0]); dd.append(e[1])
        else:
            a, b = (int(x) for x in rng.integers(0, n, 2))
            if a != b and (a, b) not in present:
                present.add((a, b)); ops.append("+"); ss.append(a); dd.append(b)
    ops, ss, dd = ops[:batch], ss[:batch], dd[:batch]
    feats = rng.random((n, 16), dtype=np.float32)
    stream = ("".join(ops).encode(), np.array(ss, np.uint32), np.array(dd, np.uint32))
    desc, man = util.make_model(str(tmp_path), "gcn", 16, 16, 2, agg="max")
    util.run_parity(str(tmp_path), desc, man, batch, edges=(src, dst), features=feats, stream=stream)


@pytest.mark.parametrize("batch", [1500, 3000, 5000])
def test_large_batch_first_failure(tmp_path, batch):
    """The first failing op in batch order decides the status on both batch
    paths, and the rejected batch leaves the engine untouched."""
    import paper_2309_11071_b200 as sg
    rng = np.random.default_rng(4)
    n = 4000
    base = sorted({(int(a), int(b)) for a, b in rng.integers(0, n, size=(9000, 2)) if a != b})
    src = np.array([p[0] for p in base], np.uint32)
    dst = np.array([p[1] for p in base], np.uint32)
    feats = rng.random((n, 8), dtype=np.float32)
    desc, man = util.make_model(str(tmp_path), "gcn", 8, 8, 2, agg="max")
    e = sg.Engine.create_from_array(sg.Graph.from_edges(n, src, dst), sg.Model.load(desc, man), feats)
    present = set(base)
    ops, ss, dd = [], [], []
    while len(ss) < batch:
        a, b = (int(x) for x in rng.integers(0, n, 2))
        if a != b and (a, b) not in present:
            present.add((a, b)); ops.append("+"); ss.append(a); dd.append(b)
    bad_at = batch - 700
    ops[bad_at], ss[bad_at], dd[bad_at] = "+", base[5][0], base[5][1]      # duplicate insert
    ops[bad_at + 300], ss[bad_at + 300], dd[bad_at + 300] = "-", 1, 1      # later: missing delete
    before = e.read_table(3, 0).tobytes()
    with pytest.raises(sg.StreamGNNError) as ex:
        e.apply_update("".join(ops), ss, dd)
    assert ex.value.status == 4 and f"{base[5][0]}->{base[5][1]}" in ex.value.message
    assert e.read_table(3, 0).tobytes() == before and e.num_edges == len(base)
    ops[bad_at] = "-"  # now a valid delete; the missing delete is the first failure
    with pytest.raises(sg.StreamGNNError) as ex:
        e.apply_update("".join(ops), ss, dd)
    assert ex.value.status == 5 and "1->1" in ex.value.message
    assert e.verify()[0] == 0
