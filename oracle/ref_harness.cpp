// TEST INFRASTRUCTURE ONLY (see oracle/ref.mk). Our own thin C-ABI harness over
// the UNMODIFIED reference C++ engine, compiled together with the reference
// sources into oracle/_ref/libstreamgnn_ref.so. It lets tests and bench.py:
//   * build a reference Engine straight from edge arrays (the reference C ABI
//     only loads edge-list text files, proj/src/core/graph.cpp:149-183),
//   * run Engine::process_update_round (proj/src/core/engine.cpp:171-319) and read
//     back stats lines, per-layer dirty sets (engine.hpp:99-100) and whole tables,
//   * time baseline::affected_inference, the k-hop recompute baseline
//     (proj/src/core/baseline.cpp:177-207),
//   * call the reference's scalar kernels (classify, matvec_affine) so the C
//     restatement in oracle/sgnn_oracle.c can be pinned on random inputs,
//   * build the benchmark's synthetic inputs (tools/rmat_gen.hpp, harness code
//     shared with tools/libsgnn_datagen.so) so bench.py's reference arm never
//     loads the product library.
// Nothing here is product code; the product is paper_2309_11071_b200/libstreamgnn.so.

#include <chrono>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>

#include "core/baseline.hpp"
#include "core/engine.hpp"
#include "core/tensor_io.hpp"
#include "rmat_gen.hpp"

using namespace streamgnn;

namespace {

struct RefEngine {
  std::unique_ptr<Engine> e;
  RoundStats last;
  uint64_t rounds = 0;
};

thread_local std::string g_err;

int code_of(const std::exception& ex) {
  if (auto* e = dynamic_cast<const Error*>(&ex)) return static_cast<int>(e->code());
  return 12;
}

std::string slurp(const char* path) {
  std::ifstream in(path);
  if (!in) fail(Errc::io, std::string("cannot open: ") + path);
  return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Graph from (src,dst) arrays via DynamicGraph::add_edge, model from the
// reference's own files, features from a row-major array. ckpt_dir != NULL
// resumes from checkpoint files (CheckpointStore::load) instead of running
// init_full_inference.
void* ref_engine_create(uint32_t num_nodes, const uint32_t* src, const uint32_t* dst, uint64_t num_edges,
                        const float* features, uint32_t rows, uint32_t cols, const char* desc_path,
                        const char* manifest_path, const char* ckpt_dir, int* status) {
  try {
    DynamicGraph g(num_nodes);
    for (uint64_t i = 0; i < num_edges; ++i) g.add_edge(src[i], dst[i]);
    std::vector<float> fv(features, features + static_cast<size_t>(rows) * cols);
    for (float& v : fv) v = flush_zero(v);
    Mat feat(rows, cols, std::move(fv));
    auto model = std::make_shared<const Model>(ModelSpec::parse(slurp(desc_path)),
                                               load_weights(manifest_path), cols);
    auto h = std::make_unique<RefEngine>();
    if (ckpt_dir) {
      CheckpointStore store = CheckpointStore::load(ckpt_dir, *model, g.num_nodes());
      h->e = std::make_unique<Engine>(std::move(g), model, std::move(feat), std::move(store));
    } else {
      h->e = std::make_unique<Engine>(std::move(g), model, std::move(feat));
    }
    *status = 0;
    return h.release();
  } catch (const std::exception& ex) {
    g_err = ex.what();
    *status = code_of(ex);
    return nullptr;
  }
}

void ref_engine_destroy(void* h) { delete static_cast<RefEngine*>(h); }

int ref_engine_set_option(void* h, const char* name, int64_t value) {
  auto* r = static_cast<RefEngine*>(h);
  std::string n(name);
  if (n == "baseline_counters") r->e->options().baseline_counters = value != 0;
  else if (n == "duplicate_seed_events") r->e->options().duplicate_seed_events = value != 0;
  else return 7;
  return 0;
}

// One round; returns 0 or the reference Errc code. The stats line is copied
// (NUL-terminated, truncated to cap) on success.
int ref_engine_apply(void* h, const char* ops, const uint32_t* src, const uint32_t* dst, size_t count,
                     char* line, size_t cap) {
  auto* r = static_cast<RefEngine*>(h);
  try {
    std::vector<EdgeDelta> delta;
    delta.reserve(count);
    for (size_t i = 0; i < count; ++i) {
      if (ops[i] != '+' && ops[i] != '-') fail(Errc::invalid_argument, "op must be '+' or '-'");
      delta.push_back({ops[i] == '+' ? EdgeOp::Insert : EdgeOp::Delete, src[i], dst[i]});
    }
    r->last = r->e->process_update_round(delta);
    r->last.round_index = r->rounds++;
    if (line && cap) {
      std::string s = r->last.to_line();
      size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
      std::memcpy(line, s.data(), n);
      line[n] = '\0';
    }
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return code_of(ex);
  }
}

// Wall time (ms) of process_update_round alone, for the CPU baseline.
double ref_engine_apply_timed(void* h, const char* ops, const uint32_t* src, const uint32_t* dst,
                              size_t count, int* status) {
  auto* r = static_cast<RefEngine*>(h);
  std::vector<EdgeDelta> delta;
  delta.reserve(count);
  for (size_t i = 0; i < count; ++i)
    delta.push_back({ops[i] == '+' ? EdgeOp::Insert : EdgeOp::Delete, src[i], dst[i]});
  try {
    auto t0 = std::chrono::steady_clock::now();
    r->last = r->e->process_update_round(delta);
    auto t1 = std::chrono::steady_clock::now();
    r->last.round_index = r->rounds++;
    *status = 0;
    return std::chrono::duration<double, std::milli>(t1 - t0).count();
  } catch (const std::exception& ex) {
    g_err = ex.what();
    *status = code_of(ex);
    return -1.0;
  }
}

// Stats line of the last successful round (RoundStats::to_line, stats.cpp:20-48).
uint64_t ref_engine_stats_line(void* h, char* line, uint64_t cap) {
  auto* r = static_cast<RefEngine*>(h);
  std::string s = r->last.to_line();
  if (line && cap) {
    size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(line, s.data(), n);
    line[n] = '\0';
  }
  return s.size();
}

uint64_t ref_engine_dirty(void* h, int layer, uint32_t* buf, uint64_t cap) {
  auto* r = static_cast<RefEngine*>(h);
  const auto& d = r->e->last_dirty_nodes();
  if (layer < 1 || layer > static_cast<int>(d.size())) return 0;
  const auto& v = d[layer - 1];
  if (buf) std::memcpy(buf, v.data(), std::min<uint64_t>(cap, v.size()) * sizeof(uint32_t));
  return v.size();
}

uint32_t ref_engine_dim(void* h, int layer, int stage) {
  auto* r = static_cast<RefEngine*>(h);
  return r->e->store().dim(layer, stage == 0 ? Stage::Message : Stage::Aggregated);
}

void ref_engine_table(void* h, int layer, int stage, float* out) {
  auto* r = static_cast<RefEngine*>(h);
  const Mat& m = r->e->store().table(layer, stage == 0 ? Stage::Message : Stage::Aggregated);
  std::memcpy(out, m.data().data(), m.data().size() * sizeof(float));
}

int ref_engine_verify(void* h) {
  auto* r = static_cast<RefEngine*>(h);
  auto mm = baseline::verify_against_full(r->e->store(), r->e->graph(), r->e->features(), r->e->model());
  return mm ? 11 : 0;
}

int ref_engine_save_checkpoints(void* h, const char* dir) {
  auto* r = static_cast<RefEngine*>(h);
  try {
    r->e->store().save(dir);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return code_of(ex);
  }
}

// CPU k-hop recompute baseline: applies the batch to a copy of the engine's
// graph and times baseline::affected_inference against the current tables.
double ref_affected_inference_ms(void* h, const char* ops, const uint32_t* src, const uint32_t* dst,
                                 size_t count) {
  auto* r = static_cast<RefEngine*>(h);
  const Engine& e = *r->e;
  const int k = e.model().num_layers();
  std::vector<EdgeDelta> delta;
  for (size_t i = 0; i < count; ++i)
    delta.push_back({ops[i] == '+' ? EdgeOp::Insert : EdgeOp::Delete, src[i], dst[i]});
  DynamicGraph post = e.graph();
  post.apply_delta(delta);
  post.commit();
  baseline::EmbeddingSet prev;
  for (int l = 1; l <= k + 1; ++l) prev.msg.push_back(e.store().table(l, Stage::Message));
  for (int l = 1; l <= k; ++l) prev.agg.push_back(e.store().table(l, Stage::Aggregated));
  auto t0 = std::chrono::steady_clock::now();
  auto out = baseline::affected_inference(post, delta, e.features(), e.model(), prev);
  auto t1 = std::chrono::steady_clock::now();
  (void)out;
  return std::chrono::duration<double, std::milli>(t1 - t0).count();
}

// ---- scalar kernels, for pinning the C restatement ----------------------

// kind: 0 NoDeletion, 1 DeletionNoEffect, 2 CoveredReset, 3 ExposedReset.
int ref_classify(const float* alpha_prev, const float* del, const float* add, uint32_t dim, int is_max) {
  GroupedEvents g;
  if (del) g.del_reduced = Vec(del, del + dim);
  if (add) g.add_reduced = Vec(add, add + dim);
  auto rep = classify(std::span<const float>(alpha_prev, dim), g, is_max ? Aggregator::Max : Aggregator::Min);
  return static_cast<int>(rep.kind);
}

void ref_matvec_affine(const float* w, uint32_t rows, uint32_t cols, const float* x, const float* bias,
                       float* out) {
  Mat m(rows, cols, std::vector<float>(w, w + static_cast<size_t>(rows) * cols));
  Vec b;
  if (bias) b.assign(bias, bias + rows);
  Vec r = matvec_affine(m, std::span<const float>(x, cols), bias ? &b : nullptr);
  std::memcpy(out, r.data(), rows * sizeof(float));
}

// ---- benchmark inputs (tools/rmat_gen.hpp) --------------------------------

int ref_gen_rmat(uint32_t num_nodes, uint64_t num_edges, uint64_t seed, uint32_t* src, uint32_t* dst) {
  try {
    sgnn_tools::gen_rmat_graph(num_nodes, num_edges, seed, src, dst);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return 1;
  }
}

int ref_gen_rmat_stream(uint32_t num_nodes, const uint32_t* base_src, const uint32_t* base_dst,
                        uint64_t num_edges, uint64_t stream_len, double insert_fraction, uint64_t seed, char* ops,
                        uint32_t* src, uint32_t* dst) {
  try {
    sgnn_tools::gen_rmat_stream(num_nodes, base_src, base_dst, num_edges, stream_len, insert_fraction, seed, ops,
                                src, dst);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return 1;
  }
}

int ref_gen_features(uint32_t rows, uint32_t cols, uint64_t seed, float* out) {
  sgnn_tools::gen_features(rows, cols, seed, out);
  return 0;
}

}  // extern "C"
