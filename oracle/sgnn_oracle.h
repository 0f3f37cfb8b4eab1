/*
 * TEST INFRASTRUCTURE — CPU restatement of the InkStream update path.
 *
 * Plain C11 restatement of the reference engine (proj/src/core/engine.cpp,
 * graph.cpp, checkpoint.cpp, tensor.cpp, hooks.cpp, model.cpp:238-284,
 * baseline.cpp), used ONLY by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the parity checker. It is never linked into, loaded by or
 * called from the product library (paper_2309_11071_b200/libstreamgnn.so).
 *
 * Parity of this restatement is pinned (tests/test_oracle.py) against
 *   - the reference's own known-answer vectors (proj/tests/test_engine.cpp,
 *     test_tensor.cpp, test_checkpoint.cpp) re-expressed as Python tests, and
 *   - golden fixtures produced by the unmodified reference compiled from
 *     /root/reference (oracle/ref.mk -> oracle/_ref, tests/golden/make_golden.py).
 *
 * Model description parsing / weight files are handled by the Python test
 * harness (oracle/model_io.py); this file receives the parsed op list.
 */
#ifndef SGNN_ORACLE_H
#define SGNN_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OP_AGGREGATE = 0, ORC_OP_LINEAR = 1, ORC_OP_RELU = 2, ORC_OP_SAGE_SELF = 3, ORC_OP_GIN_SELF = 4 };

/* One model op. LINEAR: w (rows x cols, row-major), bias (rows) or NULL.
 * SAGE_SELF: w = W2_<partition> (rows x cols). GIN_SELF: eps. */
typedef struct orc_op {
  int kind;
  const float* w;
  uint32_t rows, cols;
  const float* bias;
  float eps;
} orc_op;

typedef struct orc_engine orc_engine;

/* Per-layer counters, same order as LayerRoundStats (proj/src/core/stats.hpp:9-20). */
enum { ORC_EVENTS, ORC_TARGETS, ORC_USER_TARGETS, ORC_NO_DEL, ORC_DEL_NO_EFFECT, ORC_COVERED,
       ORC_EXPOSED, ORC_RECOMPUTES, ORC_DIRTY, ORC_FETCH_ROWS, ORC_NUM_COUNTERS };

/* Builds the graph with add_edge semantics (duplicates rejected), then runs
 * init_full_inference. Returns NULL and sets *status (reference Errc) on error. */
orc_engine* orc_create(uint32_t num_nodes, const uint32_t* src, const uint32_t* dst, uint64_t num_edges,
                       const float* features, uint32_t feature_len, const orc_op* ops, int num_ops,
                       int is_max, int* status);
void orc_destroy(orc_engine* e);
int orc_set_option(orc_engine* e, const char* name, int64_t value);
int orc_num_layers(const orc_engine* e);

/* One round (Engine::process_update_round). ops[i] in {'+','-'}. Returns 0 or
 * the Errc code; on error the graph and store are untouched. */
int orc_apply(orc_engine* e, const char* ops, const uint32_t* src, const uint32_t* dst, size_t count);
const char* orc_last_error(void);

/* Counters of the last round: layers x ORC_NUM_COUNTERS, then
 * [num_updates, ckpt_fetches, feat_fetches, has_baseline, affected_fetches,
 *  full_fetches, area_nodes]. */
void orc_last_stats(const orc_engine* e, uint64_t* out);

uint32_t orc_dim(const orc_engine* e, int layer, int stage);
void orc_table(const orc_engine* e, int layer, int stage, float* out);
uint64_t orc_dirty(const orc_engine* e, int layer, uint32_t* buf, uint64_t cap);
uint64_t orc_num_edges(const orc_engine* e);
/* Full inference + bitwise compare (baseline::verify_against_full). 0 = equal. */
int orc_verify(const orc_engine* e, uint32_t* layer, uint32_t* stage, uint32_t* node, uint32_t* index);

/* Scalar restatements exposed for known-answer tests. */
int orc_classify(const float* alpha_prev, const float* del, const float* add, uint32_t dim, int is_max);
void orc_matvec_affine(const float* w, uint32_t rows, uint32_t cols, const float* x, const float* bias,
                       float* out);

#ifdef __cplusplus
}
#endif

#endif
