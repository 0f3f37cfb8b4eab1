/*
 * B200 extensions to the streamgnn C ABI. Nothing here replaces a reference
 * symbol; these entry points exist for bulk loading, device-resident batches,
 * parity readout and measurement. Plain pointers and sizes only.
 */
#ifndef STREAMGNN_B200_H
#define STREAMGNN_B200_H

#include "streamgnn.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- owner-computes sharding ------------------------
 * Every shard holds the same graph and model; shard r classifies, recomputes
 * and combines only targets in its [lo, hi) vertex range, and the dirty nodes
 * of each layer are exchanged with their old/new next-layer messages. Stats
 * lines are global (counters all-reduced); a_l and m_{k+1} rows are valid on
 * their owner only. */

/* A fresh NCCL unique id (128 bytes) for sgnn_b200_engine_join_nccl. */
sgnn_status sgnn_b200_nccl_unique_id(uint8_t* out128);

/* Makes `e` shard `rank` of `world` processes (one GPU each) over NCCL. */
sgnn_status sgnn_b200_engine_join_nccl(sgnn_engine* e, const uint8_t* id128, int rank, int world);

/* Makes `count` engines of this process (created alike) the shards of one
 * graph. Rounds must then be applied to all of them together:
 * sgnn_b200_group_apply_update runs one host thread per shard. */
sgnn_status sgnn_b200_engines_join_local(sgnn_engine* const* engines, int count);
sgnn_status sgnn_b200_group_apply_update(sgnn_engine* const* engines, int count, const char* ops,
                                         const uint32_t* src, const uint32_t* dst, size_t n);

/* The contiguous vertex ranges the shards own: bounds[r]..bounds[r+1] for
 * r < world (world + 1 values), balancing sum(in_degree + 1). Host only. */
sgnn_status sgnn_b200_shard_bounds(const uint32_t* in_degree, uint32_t n, int world, uint32_t* bounds);

/* The [lo, hi) target range the engine owns (the whole graph unsharded). */
sgnn_status sgnn_b200_engine_shard_range(const sgnn_engine* e, uint32_t* lo, uint32_t* hi);

/* 1 when a CUDA device is usable; otherwise 0 and the reason in `why`. */
int sgnn_b200_device_available(char* why, size_t cap);

/* Graph from edge arrays, checked as a sequence of sgnn_graph_add_edge calls
 * (the first failing edge in input order decides the status). */
sgnn_status sgnn_b200_graph_from_edges(uint32_t num_nodes, const uint32_t* src, const uint32_t* dst,
                                       uint64_t count, int symmetrize, sgnn_graph** out);

/* sgnn_engine_create with the features given in memory (rows x cols,
 * row-major). NaN is rejected and -0 flushed as for a tensor file. */
sgnn_status sgnn_b200_engine_create_mem(const sgnn_graph* g, const sgnn_model* m, const float* features,
                                        uint32_t rows, uint32_t cols, sgnn_engine** out);

/* sgnn_engine_apply_update with the batch already resident in device memory
 * (ops/src/dst are device pointers). Same semantics and status codes.
 * Precondition: the work that wrote the three buffers has completed (e.g. the
 * producing stream was synchronized); the engine copies them on its own
 * stream. Use the _async variant to order the copy after a producer stream. */
sgnn_status sgnn_b200_engine_apply_update_device(sgnn_engine* e, const char* d_ops, const uint32_t* d_src,
                                                 const uint32_t* d_dst, size_t count);

/* As sgnn_b200_engine_apply_update_device, but the engine's stream first waits
 * (cudaStreamWaitEvent) for everything enqueued so far on producer_stream (a
 * cudaStream_t, e.g. torch's current stream), so the caller need not
 * synchronize. The call still returns with the round complete. */
sgnn_status sgnn_b200_engine_apply_update_device_async(sgnn_engine* e, const char* d_ops, const uint32_t* d_src,
                                                       const uint32_t* d_dst, size_t count, void* producer_stream);

/* Rows [lo, hi) of a table (packed (hi-lo) x dim floats; cap in floats). On a
 * sharded engine the aggregated tables and the output messages m_{k+1} hold
 * valid rows for the shard's own range only: reading other rows of those
 * tables (here, through sgnn_engine_read_embedding or through
 * sgnn_b200_engine_read_table) is SGNN_ERR_INVALID_ARGUMENT, and so is
 * sgnn_engine_save_checkpoints on a shard of a multi-shard group. */
sgnn_status sgnn_b200_engine_read_rows(const sgnn_engine* e, int layer, int stage, uint32_t lo, uint32_t hi,
                                       float* buf, size_t cap);

/* Nodes written in the last round at `layer` (1..k), ascending
 * (Engine::last_dirty_nodes of the reference). *count = full size. */
sgnn_status sgnn_b200_engine_dirty_nodes(const sgnn_engine* e, int layer, uint32_t* buf, size_t cap,
                                         size_t* count);

/* Whole table (num_nodes x dim floats, row-major); cap in floats. */
sgnn_status sgnn_b200_engine_read_table(const sgnn_engine* e, int layer, int stage, float* buf, size_t cap);

uint32_t sgnn_b200_engine_num_nodes(const sgnn_engine* e);
uint64_t sgnn_b200_engine_num_edges(const sgnn_engine* e);

/* Device time (ms) of the last round per kernel class, when the option
 * "profile_kernels" is 1: [graph_update, events, sort_group, classify,
 * recompute, compact, combine, finalize, commit, total, recompute_bytes,
 * classify_bytes, events_bytes]. Returns the number of values written. */
size_t sgnn_b200_engine_kernel_times(const sgnn_engine* e, double* out, size_t cap);

/* Kernel launches (CUDA-graph kernel nodes) one round of the current batch
 * size executes; 0 before the first round. */
size_t sgnn_b200_engine_launches_per_round(const sgnn_engine* e);

/* Writes a 256 MiB scratch buffer on the engine's stream (L2 flush between
 * timed rounds). */
sgnn_status sgnn_b200_engine_flush_l2(sgnn_engine* e);

/* The cudaStream_t every kernel of this engine is launched on. */
void* sgnn_b200_engine_stream(const sgnn_engine* e);

/* ---- stats lines ---------------------------
 * The reference CLI's `report` aggregation (proj/tools/streamgnn_cli.cpp:93-172:
 * summarize + print_report) over stats files written one sgnn_engine_stats_line
 * per line; the text for every path is concatenated in order, byte-identical
 * to what `streamgnn report <paths...>` prints. Text out-parameters follow
 * sgnn_engine_stats_line: *len = full length, truncated + NUL and
 * SGNN_ERR_INVALID_ARGUMENT when cap < len + 1. Unreadable file: SGNN_ERR_IO
 * "cannot open stats file: <path>". */
sgnn_status sgnn_b200_stats_report(const char* const* paths, size_t n_paths, char* buf, size_t cap, size_t* len);

/* RoundStats::from_line then to_line (proj/src/core/stats.cpp:50-119, 20-48):
 * parses a stats line (SGNN_ERR_FORMAT "bad stats token: ..." / "bad layer
 * index in stats: ...") and writes it back in canonical form (totals
 * recomputed from the per-layer fields, unknown keys dropped). */
sgnn_status sgnn_b200_stats_canonical(const char* line, char* buf, size_t cap, size_t* len);

#ifdef __cplusplus
}
#endif

#endif /* STREAMGNN_B200_H */
