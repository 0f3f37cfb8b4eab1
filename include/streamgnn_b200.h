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
 * A graph is partitioned over up to 8 shards (one per GPU of a B200 box, or
 * several on one GPU): shard r owns a contiguous vertex range (balancing
 * sum(in_degree + 1)), holds only those rows of every message and aggregate
 * table, and classifies, recomputes and combines only its own targets. Rows of
 * other shards (in-neighbour messages, boundary sources) are read in place
 * through peer memory (NVLink P2P / CUDA IPC); per layer the shards exchange
 * only their dirty-node lists and pre-images. Creation and sgnn_engine_verify
 * / set_option("combination_mode") are collective: every shard calls them.
 * Stats lines are global; readouts cover the shard's own rows. */

typedef struct sgnn_shm sgnn_shm;

/* `count` engines of one process sharing one graph (one shard each, created
 * concurrently on the current device). Rounds must then be applied to all of
 * them together: sgnn_b200_group_apply_update runs one host thread per shard. */
sgnn_status sgnn_b200_group_create(const sgnn_graph* g, const sgnn_model* m, const float* features, uint32_t rows,
                                   uint32_t cols, int count, sgnn_engine** out);
sgnn_status sgnn_b200_group_apply_update(sgnn_engine* const* engines, int count, const char* ops,
                                         const uint32_t* src, const uint32_t* dst, size_t n);

/* Shard `rank` of `world` processes on one host (each on its current device):
 * host collectives through the POSIX shared-memory segment `name` (created by
 * rank 0; a plain name, unique per job), device memory through CUDA IPC. Every
 * rank calls this with the same graph, model and features. */
sgnn_status sgnn_b200_engine_create_shm(const char* name, int rank, int world, const sgnn_graph* g,
                                        const sgnn_model* m, const float* features, uint32_t rows, uint32_t cols,
                                        sgnn_engine** out);

/* out3 = {table bytes this engine holds, graph bytes, device memory in use}. */
sgnn_status sgnn_b200_engine_memory(const sgnn_engine* e, uint64_t* out3);

/* The host protocol of the shared-memory transport on its own (no device):
 * what the shards of a multi-process group run between their layers. */
sgnn_status sgnn_b200_shm_open(const char* name, int rank, int world, double timeout_s, sgnn_shm** out);
sgnn_status sgnn_b200_shm_barrier(sgnn_shm* s);
/* all[r] = rank r's value (world values). */
sgnn_status sgnn_b200_shm_all_gather(sgnn_shm* s, uint64_t mine, uint64_t* all);
/* In-place element-wise sum over the ranks (n <= 1024). */
sgnn_status sgnn_b200_shm_allreduce(sgnn_shm* s, uint64_t* values, size_t n);
void sgnn_b200_shm_close(sgnn_shm* s);

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

/* Binary edge list (ingest where text parsing would
 * dominate, e.g. C4's 1.6B edges): magic "SGNNEDG1", u32 num_nodes, u32 0,
 * u64 count, count u32 sources, count u32 destinations (little-endian).
 * Loading builds the same graph sgnn_graph_load builds from the same pairs in
 * the same order (first failing edge decides the status), with num_nodes =
 * max(header, max id + 1); SGNN_ERR_FORMAT on a bad header or short file. */
sgnn_status sgnn_b200_graph_load_binary(const char* path, int symmetrize, sgnn_graph** out);
sgnn_status sgnn_b200_graph_save_binary(const sgnn_graph* g, const char* path);

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

/* Rows [lo, hi) of a table (packed (hi-lo) x dim floats; cap in floats). A
 * sharded engine holds its own range of every table: reading other rows
 * (here, through sgnn_engine_read_embedding or sgnn_b200_engine_read_table) is
 * SGNN_ERR_INVALID_ARGUMENT, and so is sgnn_engine_save_checkpoints on a shard
 * of a multi-shard group. */
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
 * classify_bytes, events_bytes, filter_entries, filter_code_pairs,
 * filter_rows]. Returns the number of values written. */
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
