// BENCHMARK / TEST HARNESS — C entry points over tools/rmat_gen.hpp, built into
// tools/libsgnn_datagen.so (tools/Makefile). Returns 0, or 1 with a message in
// dg_last_error(). Not part of the product library.
#include <cstring>
#include <exception>
#include <string>

#include "rmat_gen.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}  // namespace

extern "C" {

const char* dg_last_error(void) { return g_err.c_str(); }

int dg_gen_rmat(uint32_t num_nodes, uint64_t num_edges, uint64_t seed, uint32_t* src, uint32_t* dst) {
  return guarded([&] { sgnn_tools::gen_rmat_graph(num_nodes, num_edges, seed, src, dst); });
}

int dg_gen_rmat_stream(uint32_t num_nodes, const uint32_t* base_src, const uint32_t* base_dst, uint64_t num_edges,
                       uint64_t stream_len, double insert_fraction, uint64_t seed, char* ops, uint32_t* src,
                       uint32_t* dst) {
  return guarded([&] {
    sgnn_tools::gen_rmat_stream(num_nodes, base_src, base_dst, num_edges, stream_len, insert_fraction, seed, ops,
                                src, dst);
  });
}

int dg_gen_features(uint32_t rows, uint32_t cols, uint64_t seed, float* out) {
  return guarded([&] { sgnn_tools::gen_features(rows, cols, seed, out); });
}

}  // extern "C"
