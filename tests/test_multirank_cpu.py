"""World-size 2-3 host protocol of the partitioned round on CPU (no GPU).

A multi-process shard group (sgnn_b200_engine_create_shm) runs every
host-side step of a round through the shared-memory transport: per layer
boundary one all-gather of the shards' dirty counts (which gives every shard
the global dirty offsets of the peers' records), per round one all-reduce of
the u64 counters, barriers around device-memory sharing. Those collectives
are exercised here exactly as the engine calls them (sgnn_b200_shm_*), in
separate processes rendezvoused over torch.distributed (gloo), and checked
against gloo's own collectives: 60 rounds of a 3-layer sequence, values that
differ per rank and per round. The device side (the peers' rows over CUDA
IPC) is covered by tests/test_gpu_sharded.py::test_shm_two_processes_one_gpu.
The ranks also derive the same owner ranges from their copies of the graph.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import paper_2309_11071_b200 as sg
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        box = [f"sgnn_cpu_test_{os.getpid()}" if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        ch = sg.ShmChannel(box[0], rank, world, timeout_s=60.0)
        rng = np.random.default_rng(100 + rank)
        mismatches = 0
        layers, n_ctr = 3, 4 * 20
        for rnd in range(60):
            for _ in range(layers - 1):  # one count exchange per layer boundary
                mine = int(rng.integers(0, 1 << 40))
                got = ch.all_gather(mine)
                ref = [None] * world
                dist.all_gather_object(ref, mine)
                mismatches += got != ref
            ctr = rng.integers(0, 1 << 50, size=n_ctr, dtype=np.uint64)
            summed = ch.allreduce(ctr)
            t = torch.from_numpy(ctr.astype(np.int64))
            dist.all_reduce(t)
            mismatches += not np.array_equal(summed.astype(np.int64), t.numpy())
            if rnd % 7 == 0:
                ch.barrier()
        # owner ranges from each rank's copy of the graph
        deg = (np.random.default_rng(3).pareto(1.5, 5000) * 4).astype(np.uint32)
        b = sg.shard_bounds(deg, world)
        got = [None] * world
        dist.all_gather_object(got, b.tolist())
        ch.close()
        q.put((rank, mismatches, got, deg.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shm_protocol_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mismatches, got, deg in out:
        assert mismatches == 0, f"rank {rank}: {mismatches} collectives disagree with gloo"
        bounds = {tuple(g) for g in got}
        assert len(bounds) == 1, "ranks disagree on the owner ranges"
        b = list(next(iter(bounds)))
        assert b[0] == 0 and b[-1] == len(deg) and b == sorted(b)
        w = np.asarray(deg, dtype=np.float64) + 1
        parts = [w[b[r]:b[r + 1]].sum() for r in range(world)]
        assert max(parts) <= w.sum() / world + w.max() + 1


def test_shm_errors():
    import paper_2309_11071_b200 as sg
    with pytest.raises(sg.StreamGNNError) as ei:
        sg.ShmChannel("bad/name", 0, 1)
    assert ei.value.status == 7
    with pytest.raises(sg.StreamGNNError) as ei:
        sg.ShmChannel(f"sgnn_cpu_err_{os.getpid()}", 2, 2)
    assert ei.value.status == 7
    # a rank whose peers never arrive times out instead of hanging
    with pytest.raises(sg.StreamGNNError) as ei:
        sg.ShmChannel(f"sgnn_cpu_alone_{os.getpid()}", 1, 2, timeout_s=0.5)
    assert "timed out" in ei.value.message
    ch = sg.ShmChannel(f"sgnn_cpu_one_{os.getpid()}", 0, 1)
    assert ch.all_gather(7) == [7]
    assert ch.allreduce([1, 2, 3]).tolist() == [1, 2, 3]
    with pytest.raises(sg.StreamGNNError):
        ch.allreduce(np.zeros(2000, np.uint64))
    ch.close()


def test_shard_bounds_edge_cases():
    import paper_2309_11071_b200 as sg
    assert sg.shard_bounds(np.zeros(0, np.uint32), 2).tolist() == [0, 0, 0]
    assert sg.shard_bounds(np.ones(10, np.uint32), 1).tolist() == [0, 10]
    b = sg.shard_bounds(np.array([0, 0, 100, 0, 0], np.uint32), 4)
    assert b[0] == 0 and b[-1] == 5 and list(b) == sorted(b)
    with pytest.raises(sg.StreamGNNError):
        sg.shard_bounds(np.ones(3, np.uint32), 0)
