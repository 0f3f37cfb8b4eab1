// Host-side graph handle (the `sgnn_graph` of the C ABI) and the text formats
// of the load path. The engine never mutates this object: sgnn_engine_create
// copies it into the device-resident store (device/graph_store.cuh).
//
// Semantics follow the reference DynamicGraph for the operations the ABI
// exposes (proj/src/core/graph.hpp:27-56, graph.cpp:10-50, 81-85, 133-224):
// sorted, duplicate-free out/in adjacency; add_edge rejects duplicates and
// out-of-range ids; edge-list and update-stream text formats with the same
// tokenisation and error messages.
#pragma once

#include <string>
#include <vector>

#include "common.hpp"

namespace sgb {

class HostGraph {
 public:
  explicit HostGraph(uint32_t num_nodes);

  uint32_t num_nodes() const { return n_; }
  uint64_t num_edges() const { return m_; }
  bool has_edge(NodeId src, NodeId dst) const;
  void add_edge(NodeId src, NodeId dst);
  const std::vector<NodeId>& out(NodeId u) const;
  const std::vector<NodeId>& in(NodeId u) const;

  // Bulk construction. Edges are checked exactly as a sequence of add_edge
  // calls would be (first failing edge in input order wins).
  static HostGraph from_edges(uint32_t num_nodes, const NodeId* src, const NodeId* dst, size_t count,
                              bool symmetrize);

  // Copy with trailing isolated nodes (reference pad_nodes, capi.cpp:202-208).
  HostGraph padded(uint32_t num_nodes) const;

 private:
  void check_node(NodeId u) const;
  uint32_t n_;
  uint64_t m_ = 0;
  std::vector<std::vector<NodeId>> out_;
  std::vector<std::vector<NodeId>> in_;
};

// "src dst" per line; blank lines and '#' lines skipped (graph.cpp:149-183).
HostGraph load_edge_list(const std::string& path, bool symmetrize);
void save_edge_list(const HostGraph& g, const std::string& path);
// Same text, written from per-source sorted lists held elsewhere.
void save_edge_list_csr(uint32_t num_nodes, const uint64_t* offsets, const NodeId* targets,
                        const std::string& path);

// Binary edge list for graphs where text parsing dominates ingest (C4: 1.6B
// edges): magic "SGNNEDG1", u32 num_nodes, u32 0, u64
// count, count u32 sources, count u32 destinations (little-endian). Loading
// builds the graph exactly as the text loader would from the same pairs in
// the same order (graph.cpp:149-183), with num_nodes = max(header, max id + 1).
HostGraph load_edge_list_binary(const std::string& path, bool symmetrize);
void save_edge_list_binary(const HostGraph& g, const std::string& path);

// "<+|-> src dst" per line (graph.cpp:193-214).
std::vector<EdgeDelta> load_update_stream(const std::string& path);
void save_update_stream(const std::vector<EdgeDelta>& s, const std::string& path);

}  // namespace sgb
