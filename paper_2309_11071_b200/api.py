"""Python mirror of the streamgnn C ABI (include/streamgnn.h).

Same names, argument meaning and error behaviour as the reference interface
(/root/reference/proj/include/streamgnn/streamgnn.h): every non-OK status raises
``StreamGNNError`` carrying the status code and sgnn_last_error(). Numpy arrays
travel as plain pointers; the engine work happens in libstreamgnn.so on the GPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

SGNN_STAGE_MESSAGE = 0
SGNN_STAGE_AGGREGATED = 1


class StreamGNNError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{_lib.STATUS.get(status, status)}: {message}")
        self.status = status
        self.message = message


def _check(status: int) -> None:
    if status != 0:
        raise StreamGNNError(status, _lib.lib().sgnn_last_error().decode())


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def status_name(status: int) -> str:
    return _lib.lib().sgnn_status_name(status).decode()


def last_error() -> str:
    return _lib.lib().sgnn_last_error().decode()


def device_available() -> tuple[bool, str]:
    buf = C.create_string_buffer(256)
    ok = _lib.lib().sgnn_b200_device_available(buf, len(buf))
    return bool(ok), buf.value.decode()


class Graph:
    """sgnn_graph: host-side graph handle (streamgnn.h:46-59)."""

    def __init__(self, handle):
        self.h = handle

    @classmethod
    def create(cls, num_nodes: int) -> "Graph":
        h = C.c_void_p()
        _check(_lib.lib().sgnn_graph_create(num_nodes, C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path: str, symmetrize: bool = False) -> "Graph":
        h = C.c_void_p()
        _check(_lib.lib().sgnn_graph_load(path.encode(), int(symmetrize), C.byref(h)))
        return cls(h)

    @classmethod
    def from_edges(cls, num_nodes: int, src, dst, symmetrize: bool = False) -> "Graph":
        src = np.ascontiguousarray(src, dtype=np.uint32)
        dst = np.ascontiguousarray(dst, dtype=np.uint32)
        h = C.c_void_p()
        _check(_lib.lib().sgnn_b200_graph_from_edges(num_nodes, _p(src), _p(dst), len(src), int(symmetrize),
                                                     C.byref(h)))
        return cls(h)

    def __del__(self):
        if getattr(self, "h", None):
            _lib.lib().sgnn_graph_destroy(self.h)
            self.h = None

    @property
    def num_nodes(self) -> int:
        return _lib.lib().sgnn_graph_num_nodes(self.h)

    @property
    def num_edges(self) -> int:
        return _lib.lib().sgnn_graph_num_edges(self.h)

    def add_edge(self, src: int, dst: int) -> None:
        _check(_lib.lib().sgnn_graph_add_edge(self.h, src, dst))

    def _neighbors(self, fn, node):
        count = C.c_size_t(0)
        _check(fn(self.h, node, None, 0, C.byref(count)))
        out = np.empty(count.value, dtype=np.uint32)
        _check(fn(self.h, node, _p(out), len(out), C.byref(count)))
        return out

    def out_neighbors(self, node: int) -> np.ndarray:
        return self._neighbors(_lib.lib().sgnn_graph_out_neighbors, node)

    def in_neighbors(self, node: int) -> np.ndarray:
        return self._neighbors(_lib.lib().sgnn_graph_in_neighbors, node)

    @classmethod
    def load_binary(cls, path: str, symmetrize: bool = False) -> "Graph":
        """Binary edge list (sgnn_b200_graph_load_binary)."""
        h = C.c_void_p()
        _check(_lib.lib().sgnn_b200_graph_load_binary(path.encode(), int(symmetrize), C.byref(h)))
        return cls(h)

    def save_binary(self, path: str) -> None:
        _check(_lib.lib().sgnn_b200_graph_save_binary(self.h, path.encode()))

    def save(self, path: str) -> None:
        _check(_lib.lib().sgnn_graph_save(self.h, path.encode()))


class Model:
    """sgnn_model: parsed description + weights (streamgnn.h:63-68)."""

    def __init__(self, handle):
        self.h = handle

    @classmethod
    def load(cls, description_path: str, weights_manifest_path: str) -> "Model":
        h = C.c_void_p()
        _check(_lib.lib().sgnn_model_load(description_path.encode(), weights_manifest_path.encode(), C.byref(h)))
        return cls(h)

    def __del__(self):
        if getattr(self, "h", None):
            _lib.lib().sgnn_model_destroy(self.h)
            self.h = None

    @property
    def num_layers(self) -> int:
        return _lib.lib().sgnn_model_num_layers(self.h)

    @property
    def aggregator(self) -> int:
        return _lib.lib().sgnn_model_aggregator(self.h)


class Engine:
    """sgnn_engine: the device-resident incremental engine (streamgnn.h:72-111)."""

    def __init__(self, handle, graph: Graph, model: Model):
        self.h = handle
        self._graph, self._model = graph, model  # keep handles alive like the caller would
        self.num_layers = model.num_layers

    @classmethod
    def create(cls, graph: Graph, model: Model, features_path: str) -> "Engine":
        h = C.c_void_p()
        _check(_lib.lib().sgnn_engine_create(graph.h, model.h, features_path.encode(), C.byref(h)))
        return cls(h, graph, model)

    @classmethod
    def create_from_array(cls, graph: Graph, model: Model, features: np.ndarray) -> "Engine":
        f = np.ascontiguousarray(features, dtype=np.float32)
        h = C.c_void_p()
        _check(_lib.lib().sgnn_b200_engine_create_mem(graph.h, model.h, _p(f), f.shape[0], f.shape[1], C.byref(h)))
        return cls(h, graph, model)

    @classmethod
    def open(cls, graph: Graph, model: Model, features_path: str, checkpoint_dir: str) -> "Engine":
        h = C.c_void_p()
        _check(_lib.lib().sgnn_engine_open(graph.h, model.h, features_path.encode(), checkpoint_dir.encode(),
                                           C.byref(h)))
        return cls(h, graph, model)

    def __del__(self):
        if getattr(self, "h", None):
            _lib.lib().sgnn_engine_destroy(self.h)
            self.h = None

    def apply_update(self, ops, src, dst) -> None:
        """One round (sgnn_engine_apply_update): ops is bytes/str of '+'/'-'."""
        if isinstance(ops, str):
            ops = ops.encode()
        if isinstance(ops, np.ndarray):
            ops = ops.tobytes()
        src = np.ascontiguousarray(src, dtype=np.uint32)
        dst = np.ascontiguousarray(dst, dtype=np.uint32)
        n = len(src)
        obuf = C.create_string_buffer(ops, max(1, len(ops)))
        _check(_lib.lib().sgnn_engine_apply_update(self.h, obuf if n else None, _p(src) if n else None,
                                                   _p(dst) if n else None, n))

    def apply_update_device(self, d_ops: int, d_src: int, d_dst: int, count: int, producer_stream: int = 0) -> None:
        """Batch already in device memory (raw device pointers). `producer_stream`
        (a cudaStream_t, e.g. torch.cuda.current_stream().cuda_stream): the engine
        waits for it before staging the batch; without it the producer's work must
        already be complete."""
        if producer_stream:
            _check(_lib.lib().sgnn_b200_engine_apply_update_device_async(
                self.h, C.c_void_p(d_ops), C.c_void_p(d_src), C.c_void_p(d_dst), count, C.c_void_p(producer_stream)))
        else:
            _check(_lib.lib().sgnn_b200_engine_apply_update_device(self.h, C.c_void_p(d_ops), C.c_void_p(d_src),
                                                                   C.c_void_p(d_dst), count))

    def set_option(self, name: str, value: int) -> None:
        _check(_lib.lib().sgnn_engine_set_option(self.h, name.encode(), int(value)))

    def stats_line(self) -> str:
        n = C.c_size_t(0)
        _check(_lib.lib().sgnn_engine_stats_line(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(_lib.lib().sgnn_engine_stats_line(self.h, buf, len(buf), C.byref(n)))
        return buf.value.decode()

    def embedding_dim(self, layer: int, stage: int) -> int:
        d = C.c_uint32(0)
        _check(_lib.lib().sgnn_engine_embedding_dim(self.h, layer, stage, C.byref(d)))
        return d.value

    def read_embedding(self, layer: int, stage: int, node: int) -> np.ndarray:
        out = np.empty(self.embedding_dim(layer, stage), dtype=np.float32)
        _check(_lib.lib().sgnn_engine_read_embedding(self.h, layer, stage, node, _p(out), len(out)))
        return out

    def read_rows(self, layer: int, stage: int, lo: int, hi: int) -> np.ndarray:
        d = self.embedding_dim(layer, stage)
        out = np.empty((hi - lo, d), dtype=np.float32)
        _check(_lib.lib().sgnn_b200_engine_read_rows(self.h, layer, stage, lo, hi, _p(out) if hi > lo else None,
                                                     out.size))
        return out

    def read_table(self, layer: int, stage: int) -> np.ndarray:
        d = self.embedding_dim(layer, stage)
        out = np.empty((self.num_nodes, d), dtype=np.float32)
        _check(_lib.lib().sgnn_b200_engine_read_table(self.h, layer, stage, _p(out), out.size))
        return out

    def dirty_nodes(self, layer: int) -> np.ndarray:
        n = C.c_size_t(0)
        _check(_lib.lib().sgnn_b200_engine_dirty_nodes(self.h, layer, None, 0, C.byref(n)))
        out = np.empty(n.value, dtype=np.uint32)
        _check(_lib.lib().sgnn_b200_engine_dirty_nodes(self.h, layer, _p(out), len(out), C.byref(n)))
        return out

    def verify(self):
        """(status, (layer, stage, node, index)); status 0 when identical."""
        v = [C.c_uint32(0) for _ in range(4)]
        st = _lib.lib().sgnn_engine_verify(self.h, *[C.byref(x) for x in v])
        return st, tuple(x.value for x in v)

    def save_checkpoints(self, path: str) -> None:
        _check(_lib.lib().sgnn_engine_save_checkpoints(self.h, path.encode()))

    def save_graph(self, path: str) -> None:
        _check(_lib.lib().sgnn_engine_save_graph(self.h, path.encode()))

    @property
    def num_nodes(self) -> int:
        return _lib.lib().sgnn_b200_engine_num_nodes(self.h)

    @property
    def num_edges(self) -> int:
        return _lib.lib().sgnn_b200_engine_num_edges(self.h)

    def kernel_times(self) -> dict:
        keys = ["graph_update", "events", "sort_group", "classify", "recompute", "compact", "combine", "finalize",
                "commit", "total", "recompute_bytes", "classify_bytes", "events_bytes", "filter_entries",
                "filter_code_pairs", "filter_rows"]
        out = np.zeros(len(keys), dtype=np.float64)
        n = _lib.lib().sgnn_b200_engine_kernel_times(self.h, _p(out), len(out))
        return dict(zip(keys[:n], out[:n].tolist()))

    def launches_per_round(self) -> int:
        return _lib.lib().sgnn_b200_engine_launches_per_round(self.h)

    def flush_l2(self) -> None:
        _check(_lib.lib().sgnn_b200_engine_flush_l2(self.h))

    @property
    def stream(self) -> int:
        return _lib.lib().sgnn_b200_engine_stream(self.h) or 0

    # ---- owner-computes sharding (include/streamgnn_b200.h)
    @classmethod
    def create_shm(cls, name: str, rank: int, world: int, graph: Graph, model: Model,
                   features: np.ndarray) -> "Engine":
        """Shard `rank` of `world` processes of one host (sgnn_b200_engine_create_shm):
        collective over a shared-memory segment `name`, peers' rows through CUDA IPC."""
        f = np.ascontiguousarray(features, dtype=np.float32)
        h = C.c_void_p()
        _check(_lib.lib().sgnn_b200_engine_create_shm(name.encode(), rank, world, graph.h, model.h, _p(f),
                                                      f.shape[0], f.shape[1], C.byref(h)))
        return cls(h, graph, model)

    def memory(self) -> dict:
        """Table bytes held, graph bytes, device memory in use (sgnn_b200_engine_memory)."""
        out = (C.c_uint64 * 3)()
        _check(_lib.lib().sgnn_b200_engine_memory(self.h, out))
        return {"tables": out[0], "graph": out[1], "device_used": out[2]}

    def shard_range(self) -> tuple[int, int]:
        lo, hi = C.c_uint32(0), C.c_uint32(0)
        _check(_lib.lib().sgnn_b200_engine_shard_range(self.h, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value


def shard_bounds(in_degree, world: int) -> np.ndarray:
    """Vertex range boundaries of `world` shards (world + 1 values)."""
    deg = np.ascontiguousarray(in_degree, dtype=np.uint32)
    out = np.zeros(world + 1, dtype=np.uint32)
    _check(_lib.lib().sgnn_b200_shard_bounds(_p(deg) if len(deg) else None, len(deg), world, _p(out)))
    return out


class ShmChannel:
    """The shared-memory transport's host protocol on its own (sgnn_b200_shm_*):
    barrier, all-gather and all-reduce between the processes of one host."""

    def __init__(self, name: str, rank: int, world: int, timeout_s: float = 120.0):
        h = C.c_void_p()
        _check(_lib.lib().sgnn_b200_shm_open(name.encode(), rank, world, timeout_s, C.byref(h)))
        self.h, self.world = h, world

    def barrier(self) -> None:
        _check(_lib.lib().sgnn_b200_shm_barrier(self.h))

    def all_gather(self, value: int) -> list:
        out = (C.c_uint64 * self.world)()
        _check(_lib.lib().sgnn_b200_shm_all_gather(self.h, value, out))
        return list(out)

    def allreduce(self, values) -> np.ndarray:
        v = np.ascontiguousarray(values, dtype=np.uint64).copy()
        _check(_lib.lib().sgnn_b200_shm_allreduce(self.h, _p(v), len(v)))
        return v

    def close(self) -> None:
        if getattr(self, "h", None):
            _lib.lib().sgnn_b200_shm_close(self.h)
            self.h = None

    __del__ = close


class ShardGroup:
    """`shards` engines of one process partitioning one graph
    (sgnn_b200_group_create): each owns a vertex range and that range's rows of
    every table; a round runs on all of them at once (one host thread per shard)
    and they exchange dirty lists and pre-images per layer. Readout assembles
    each table from the owners' rows. verify() and set_option() of a collective
    option run on every shard concurrently."""

    COLLECTIVE_OPTIONS = ("combination_mode",)

    def __init__(self, graph: "Graph", model: "Model", features: np.ndarray, shards: int):
        f = np.ascontiguousarray(features, dtype=np.float32)
        arr = (C.c_void_p * shards)()
        _check(_lib.lib().sgnn_b200_group_create(graph.h, model.h, _p(f), f.shape[0], f.shape[1], shards, arr))
        self.engines = [Engine(C.c_void_p(arr[i]), graph, model) for i in range(shards)]
        self._arr = arr
        self.ranges = [e.shard_range() for e in self.engines]
        self.num_layers = model.num_layers

    def _each(self, fn):
        """fn(engine) on every shard concurrently (collective calls)."""
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(len(self.engines)) as ex:
            return list(ex.map(fn, self.engines))

    def apply_update(self, ops, src, dst) -> None:
        if isinstance(ops, str):
            ops = ops.encode()
        if isinstance(ops, np.ndarray):
            ops = ops.tobytes()
        src = np.ascontiguousarray(src, dtype=np.uint32)
        dst = np.ascontiguousarray(dst, dtype=np.uint32)
        n = len(src)
        obuf = C.create_string_buffer(ops, max(1, len(ops)))
        _check(_lib.lib().sgnn_b200_group_apply_update(self._arr, len(self.engines), obuf if n else None,
                                                       _p(src) if n else None, _p(dst) if n else None, n))

    def stats_line(self) -> str:
        return self.engines[0].stats_line()

    def read_table(self, layer: int, stage: int) -> np.ndarray:
        """Each shard's owned rows (the owner-only tables are valid there only)."""
        return np.concatenate([e.read_rows(layer, stage, lo, hi) for e, (lo, hi) in zip(self.engines, self.ranges)])

    def dirty_nodes(self, layer: int) -> np.ndarray:
        parts = []
        for e, (lo, hi) in zip(self.engines, self.ranges):
            d = e.dirty_nodes(layer)
            parts.append(d[(d >= lo) & (d < hi)])
        return np.sort(np.concatenate(parts)) if parts else np.zeros(0, np.uint32)

    def set_option(self, name: str, value: int) -> None:
        if name in self.COLLECTIVE_OPTIONS:
            self._each(lambda e: e.set_option(name, value))
        else:
            for e in self.engines:
                e.set_option(name, value)

    def verify(self):
        for st, where in self._each(lambda e: e.verify()):
            if st:
                return st, where
        return 0, (0, 0, 0, 0)

    def memory(self) -> list:
        return [e.memory() for e in self.engines]


class StreamReader:
    """sgnn_stream_reader (streamgnn.h:115-118)."""

    def __init__(self, path: str):
        h = C.c_void_p()
        _check(_lib.lib().sgnn_stream_open(path.encode(), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            _lib.lib().sgnn_stream_destroy(self.h)
            self.h = None

    def __iter__(self):
        op = C.create_string_buffer(1)
        s, d = C.c_uint32(0), C.c_uint32(0)
        while _lib.lib().sgnn_stream_next(self.h, op, C.byref(s), C.byref(d)):
            yield op.raw.decode(), s.value, d.value


def gen_synthetic(out_dir: str, num_nodes=1000, avg_degree=8.0, feature_len=16, stream_len=200, seed=1,
                  insert_fraction=0.6) -> None:
    cfg = _lib.GenConfig(num_nodes, avg_degree, feature_len, stream_len, seed, insert_fraction)
    _check(_lib.lib().sgnn_gen_synthetic(C.byref(cfg), out_dir.encode()))


def gen_model(kind: str, feature_len: int, hidden: int, layers: int, seed: int, epsilon: float, out_dir: str) -> None:
    _check(_lib.lib().sgnn_gen_model(kind.encode(), feature_len, hidden, layers, seed, epsilon, out_dir.encode()))


def _text_call(fn, *args) -> str:
    n = C.c_size_t(0)
    _check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(fn(*args, buf, len(buf), C.byref(n)))
    return buf.value.decode()


def stats_report(*paths: str) -> str:
    """The reference CLI's `report` text for stats files (streamgnn_cli.cpp:93-172)."""
    arr = (C.c_char_p * max(1, len(paths)))(*[p.encode() for p in paths])
    return _text_call(_lib.lib().sgnn_b200_stats_report, arr, len(paths))


def stats_canonical(line: str) -> str:
    """RoundStats::from_line + to_line (stats.cpp:50-119, 20-48)."""
    return _text_call(_lib.lib().sgnn_b200_stats_canonical, line.encode())
