"""World-size-2 host logic of the sharded round on CPU (gloo).

What a multi-GPU launch does before its first round, per rank: rank 0 makes the
NCCL unique id (sgnn_b200_nccl_unique_id), the launcher broadcasts it over
torch.distributed, and every rank derives the same owner ranges from its
replica of the graph (sgnn_b200_shard_bounds). Checked here with gloo: the id
arrives intact, ranges agree across ranks, tile [0, N) and balance in-degree.
The device-side exchange itself is covered by tests/test_gpu_sharded.py.
"""
import os
import socket

import numpy as np
import pytest
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
        box = [sg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        uid = box[0]
        rng = np.random.default_rng(3)  # every rank holds the same graph
        deg = (rng.pareto(1.5, 5000) * 4).astype(np.uint32)
        b = sg.shard_bounds(deg, world)
        got = [None] * world
        dist.all_gather_object(got, (uid, b.tolist()))
        q.put((rank, got, deg.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_rank_setup_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, deg in out:
        uids = {g[0] for g in got}
        assert len(uids) == 1 and len(next(iter(uids))) == 128
        bounds = {tuple(g[1]) for g in got}
        assert len(bounds) == 1, "ranks disagree on the owner ranges"
        b = list(next(iter(bounds)))
        assert b[0] == 0 and b[-1] == len(deg) and b == sorted(b)
        w = np.asarray(deg, dtype=np.float64) + 1
        parts = [w[b[r]:b[r + 1]].sum() for r in range(world)]
        assert max(parts) <= w.sum() / world + w.max() + 1


def test_shard_bounds_edge_cases():
    import paper_2309_11071_b200 as sg
    assert sg.shard_bounds(np.zeros(0, np.uint32), 2).tolist() == [0, 0, 0]
    assert sg.shard_bounds(np.ones(10, np.uint32), 1).tolist() == [0, 10]
    b = sg.shard_bounds(np.array([0, 0, 100, 0, 0], np.uint32), 4)
    assert b[0] == 0 and b[-1] == 5 and list(b) == sorted(b)
    with pytest.raises(sg.StreamGNNError):
        sg.shard_bounds(np.ones(3, np.uint32), 0)
