"""GPU parity of the owner-computes partitioned round.

A ShardGroup partitions the graph over 2-4 engines of this process (one host
thread each, LocalTransport): every shard holds only its own rows of every
table and reads the others' through peer memory — the same round code the
multi-process path (shared-memory transport + CUDA IPC, tested below with two
processes on one GPU) runs, with only the transport swapped. The all-reduced
stats line, the union of the owners' dirty sets and the owner-assembled
tables must equal the oracle's bit for bit after every round (reference
semantics: proj/src/core/engine.cpp:171-319).
"""
import os

import numpy as np
import pytest

from tests import util
from tests.test_gpu_parity import _hub_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def data(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("sharded"))
    return util.make_dataset(d, nodes=300, deg=6.0, feat=16, stream=120)


@pytest.mark.parametrize("shards", [2, 3])
@pytest.mark.parametrize("kind,layers,agg", [("gcn", 2, "max"), ("sage", 2, None), ("gin", 3, "max")])
@pytest.mark.parametrize("batch", [1, 10])
def test_sharded_stream_parity(data, shards, kind, layers, agg, batch):
    desc, man = util.make_model(data, kind, 16, 16 if kind != "gin" else 8, layers, agg=agg)
    util.run_parity(data, desc, man, batch, shards=shards)


def test_sharded_options(data):
    desc, man = util.make_model(data, "gcn", 16, 16, 2)
    util.run_parity(data, desc, man, 5, shards=2, options=[("duplicate_seed_events", 1), ("baseline_counters", 1)])


def test_sharded_wide_rows(tmp_path):
    d = util.make_dataset(str(tmp_path), nodes=250, deg=8.0, feat=602, stream=60, seed=11)
    desc, man = util.make_model(d, "gcn", 602, 256, 2, agg="max")
    util.run_parity(d, desc, man, 10, check_every=3, shards=4)


def test_sharded_hub(tmp_path):
    edges, feats, stream = _hub_case(tmp_path)
    d = str(tmp_path)
    desc, man = util.make_model(d, "sage", 24, 16, 2, agg="max")
    util.run_parity(d, desc, man, 25, edges=edges, features=feats, stream=stream, shards=3)


def test_sharded_invalid_batch_is_atomic(data):
    """A rejected batch fails on every shard with the reference's status and
    leaves all of them untouched."""
    import os
    import paper_2309_11071_b200 as sg
    from oracle import model_io
    desc, man = util.make_model(data, "gcn", 16, 16, 2)
    src, dst = model_io.read_edge_list(os.path.join(data, "edges.txt"))
    feats = model_io.read_tnsr(os.path.join(data, "features.tnsr"))
    n = feats.shape[0]
    grp = sg.ShardGroup(sg.Graph.from_edges(n, src, dst), sg.Model.load(desc, man), feats, 2)
    before = grp.read_table(3, 0)
    with pytest.raises(sg.StreamGNNError) as ei:
        grp.apply_update("+", [int(src[0])], [int(dst[0])])  # duplicate insert
    assert ei.value.status == 4
    assert grp.read_table(3, 0).tobytes() == before.tobytes()
    st, _ = grp.verify()
    assert st == 0


def test_sharding_partitions_the_work(data):
    """Each shard's last-layer dirty list (never exchanged) lies inside its own
    range, the ranges tile the graph, and together they cover every dirty
    node of the unsharded engine."""
    import os
    import paper_2309_11071_b200 as sg
    from oracle import model_io
    desc, man = util.make_model(data, "gcn", 16, 16, 2, agg="max")
    src, dst = model_io.read_edge_list(os.path.join(data, "edges.txt"))
    feats = model_io.read_tnsr(os.path.join(data, "features.tnsr"))
    ops, ss, dd = model_io.read_stream(os.path.join(data, "stream.txt"))
    n = feats.shape[0]
    m = sg.Model.load(desc, man)
    grp = sg.ShardGroup(sg.Graph.from_edges(n, src, dst), m, feats, 3)
    one = sg.Engine.create_from_array(sg.Graph.from_edges(n, src, dst), m, feats)
    assert grp.ranges[0][0] == 0 and grp.ranges[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(grp.ranges, grp.ranges[1:]))
    assert sum(hi > lo for lo, hi in grp.ranges) >= 2
    owned_total = 0
    for i in range(0, 60, 20):
        grp.apply_update(ops[i:i + 20], ss[i:i + 20], dd[i:i + 20])
        one.apply_update(ops[i:i + 20], ss[i:i + 20], dd[i:i + 20])
        for e, (lo, hi) in zip(grp.engines, grp.ranges):
            d2 = e.dirty_nodes(2)
            assert ((d2 >= lo) & (d2 < hi)).all()
            owned_total += len(d2)
        assert np.array_equal(grp.dirty_nodes(2), one.dirty_nodes(2))
    assert owned_total > 0
    # every shard reports its kernel launches per round (bench.py gpu_launches)
    assert all(e.launches_per_round() > 10 for e in grp.engines)


def _shm_name(tag):
    import os
    return f"sgnn_test_{tag}_{os.getpid()}"


def test_shm_transport_single_rank(data):
    """The multi-process path in one process: a 1-rank shared-memory group
    (host collectives through POSIX shm, the exchange through the rank's own
    pack buffers) stays bit-identical to the oracle."""
    import os
    import paper_2309_11071_b200 as sg
    from oracle import model_io, oracle
    desc, man = util.make_model(data, "sage", 16, 16, 2, agg="max")
    src, dst = model_io.read_edge_list(os.path.join(data, "edges.txt"))
    feats = model_io.read_tnsr(os.path.join(data, "features.tnsr"))
    ops, ss, dd = model_io.read_stream(os.path.join(data, "stream.txt"))
    n = feats.shape[0]
    e = sg.Engine.create_shm(_shm_name("one"), 0, 1, sg.Graph.from_edges(n, src, dst), sg.Model.load(desc, man),
                             feats)
    assert e.shard_range() == (0, n)
    orc = oracle.make_oracle(n, src, dst, feats, model_io.load_model(desc, man))
    for i in range(0, len(ss), 12):
        e.apply_update(ops[i:i + 12], ss[i:i + 12], dd[i:i + 12])
        assert orc.apply(ops[i:i + 12], ss[i:i + 12], dd[i:i + 12]) == 0
        assert e.stats_line() == orc.stats_line()
    err = util.tables_equal(e, orc, 2)
    assert err is None, err


def test_shm_two_processes_one_gpu(data, tmp_path):
    """Two processes, one shard each, on the same GPU: shared-memory barriers
    and collectives, CUDA IPC mappings of each other's tables and pack buffers.
    Every round's global stats line, each rank's owned dirty nodes and owned
    table rows equal the oracle's (tests/shm_worker.py)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    desc, man = util.make_model(data, "gin", 16, 8, 3, agg="max")
    name = _shm_name("two")
    procs = [subprocess.Popen([sys.executable, os.path.join(root, "tests", "shm_worker.py"), name, str(r), "2", data,
                               desc, man, str(tmp_path / f"rank{r}.json")], cwd=root)
             for r in range(2)]
    for p in procs:
        assert p.wait(timeout=600) == 0
    outs = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(2)]
    for o in outs:
        assert o["errors"] == [], o["errors"]
        assert o["rounds"] > 0
    assert outs[0]["lines"] == outs[1]["lines"]
    r0, r1 = outs[0]["range"], outs[1]["range"]
    assert r0[0] == 0 and r0[1] == r1[0] and r1[1] > r1[0]


def test_sharded_and_khop_rounds_with_kernel_profiling(data):
    """Per-kernel-class timing (bench.py's profiled pass) also works on the
    uncaptured round paths: sharded (exchange needs host-known counts) and the
    k-hop comparator."""
    import os
    import paper_2309_11071_b200 as sg
    from oracle import model_io
    desc, man = util.make_model(data, "gcn", 16, 16, 2, agg="max")
    src, dst = model_io.read_edge_list(os.path.join(data, "edges.txt"))
    feats = model_io.read_tnsr(os.path.join(data, "features.tnsr"))
    ops, ss, dd = model_io.read_stream(os.path.join(data, "stream.txt"))
    n = feats.shape[0]
    m = sg.Model.load(desc, man)
    a = sg.Engine.create_shm(_shm_name("prof"), 0, 1, sg.Graph.from_edges(n, src, dst), m, feats)
    b = sg.Engine.create_from_array(sg.Graph.from_edges(n, src, dst), m, feats)
    b.set_option("khop_recompute", 1)
    for e in (a, b):
        e.set_option("profile_kernels", 1)
        e.apply_update(ops[:20], ss[:20], dd[:20])
        t = e.kernel_times()
        assert t["total"] > 0 and t["graph_update"] > 0, t


def test_sharded_owner_only_readout_and_options(data):
    """A shard holds its own rows of every table: other rows cannot be read,
    save_checkpoints on one shard fails, and the k-hop comparator is refused
    on sharded engines — each with SGNN_ERR_INVALID_ARGUMENT (7)."""
    import os
    import paper_2309_11071_b200 as sg
    from oracle import model_io
    desc, man = util.make_model(data, "gcn", 16, 16, 2)
    src, dst = model_io.read_edge_list(os.path.join(data, "edges.txt"))
    feats = model_io.read_tnsr(os.path.join(data, "features.tnsr"))
    n = feats.shape[0]
    grp = sg.ShardGroup(sg.Graph.from_edges(n, src, dst), sg.Model.load(desc, man), feats, 2)
    e0 = grp.engines[0]
    lo, hi = grp.ranges[0]
    assert e0.read_rows(1, 1, lo, hi).shape == (hi - lo, 16)
    assert e0.read_rows(2, 0, lo, hi).shape == (hi - lo, 16)
    for layer, stage in ((1, 0), (1, 1), (2, 0), (2, 1), (3, 0)):
        with pytest.raises(sg.StreamGNNError) as err:
            e0.read_rows(layer, stage, hi, n)
        assert err.value.status == 7 and "not owned" in err.value.message
        with pytest.raises(sg.StreamGNNError):
            e0.read_table(layer, stage)
    with pytest.raises(sg.StreamGNNError) as err:
        e0.save_checkpoints(os.path.join(data, "ck_shard"))
    assert err.value.status == 7
    with pytest.raises(sg.StreamGNNError) as err:
        e0.set_option("khop_recompute", 1)
    assert err.value.status == 7


def test_partitioned_table_memory(tmp_path):
    """Per-shard table bytes scale as the owned share of the vertices: the
    shards' tables sum to the unsharded engine's (allocation granularity
    aside), and no shard holds more than its range needs."""
    import paper_2309_11071_b200 as sg
    from oracle import model_io
    d = util.make_dataset(str(tmp_path), nodes=4000, deg=5.0, feat=64, stream=10, seed=5)
    desc, man = util.make_model(d, "sage", 64, 64, 2, agg="max")
    src, dst = model_io.read_edge_list(os.path.join(d, "edges.txt"))
    feats = model_io.read_tnsr(os.path.join(d, "features.tnsr"))
    n = feats.shape[0]
    m = sg.Model.load(desc, man)
    one = sg.Engine.create_from_array(sg.Graph.from_edges(n, src, dst), m, feats)
    full = one.memory()["tables"]
    grp = sg.ShardGroup(sg.Graph.from_edges(n, src, dst), m, feats, 4)
    parts = [mem["tables"] for mem in grp.memory()]
    assert abs(sum(parts) - full) <= 4 * 16 * 256
    for (lo, hi), b in zip(grp.ranges, parts):
        assert b <= full * (hi - lo) / n + 16 * 256
    st, _ = grp.verify()
    assert st == 0


def test_apply_update_device_waits_for_producer_stream(data):
    """sgnn_b200_engine_apply_update_device_async orders the batch staging after
    the producer stream: the batch is written by a kernel on a side torch
    stream right before the call, without any host synchronization."""
    import os
    import torch
    import paper_2309_11071_b200 as sg
    from oracle import model_io, oracle
    desc, man = util.make_model(data, "sage", 16, 16, 2)
    src, dst = model_io.read_edge_list(os.path.join(data, "edges.txt"))
    feats = model_io.read_tnsr(os.path.join(data, "features.tnsr"))
    ops, ss, dd = model_io.read_stream(os.path.join(data, "stream.txt"))
    n = feats.shape[0]
    e = sg.Engine.create_from_array(sg.Graph.from_edges(n, src, dst), sg.Model.load(desc, man), feats)
    orc = oracle.make_oracle(n, src, dst, feats, model_io.load_model(desc, man))
    side = torch.cuda.Stream()
    big = torch.zeros(1 << 24, device="cuda")
    for i in range(0, len(ss), 20):
        o, s_, d_ = ops[i:i + 20], ss[i:i + 20], dd[i:i + 20]
        host = [torch.frombuffer(bytearray(o), dtype=torch.uint8).pin_memory(),
                torch.from_numpy(s_.astype(np.int32)).pin_memory(), torch.from_numpy(d_.astype(np.int32)).pin_memory()]
        with torch.cuda.stream(side):
            for _ in range(20):  # keep the side stream busy before the batch lands
                big.mul_(1.0001)
            devt = [t.to("cuda", non_blocking=True) for t in host]
        e.apply_update_device(devt[0].data_ptr(), devt[1].data_ptr(), devt[2].data_ptr(), len(s_),
                              producer_stream=side.cuda_stream)
        assert orc.apply(o, s_, d_) == 0
        assert e.stats_line() == orc.stats_line()
    assert util.tables_equal(e, orc, 2) is None


def test_sharded_host_collective_path(data, monkeypatch):
    """The host-collective exchange (per-layer count all-gather and counter
    all-reduce through the transport, graph segments between them) — what
    baseline_counters and profiled rounds use — stays bit-exact too
    (SGNN_B200_DEVICE_EXCHANGE=0 makes every round take it)."""
    monkeypatch.setenv("SGNN_B200_DEVICE_EXCHANGE", "0")
    desc, man = util.make_model(data, "gin", 16, 8, 3, agg="max")
    util.run_parity(data, desc, man, 7, shards=3)
