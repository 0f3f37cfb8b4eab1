"""B200-native InkStream engine: incremental min/max-GNN inference on streaming graphs.

The product is ``libstreamgnn.so`` in this directory — a drop-in for the
reference C ABI (include/streamgnn.h) whose update path runs as hand-written
sm_100a kernels. This package is a thin ctypes mirror of that ABI.
"""
from .api import (SGNN_STAGE_AGGREGATED, SGNN_STAGE_MESSAGE, Engine, Graph, Model, ShardGroup, StreamGNNError,
                  ShmChannel, StreamReader, shard_bounds, stats_canonical, stats_report,
                  device_available, gen_model, gen_synthetic, last_error,
                  status_name)

__all__ = ["Engine", "Graph", "Model", "ShardGroup", "ShmChannel", "StreamReader", "shard_bounds", "stats_report", "stats_canonical", "StreamGNNError", "SGNN_STAGE_MESSAGE",
           "SGNN_STAGE_AGGREGATED", "device_available", "gen_model",
           "gen_synthetic", "last_error", "status_name"]
