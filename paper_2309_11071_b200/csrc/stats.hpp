// Per-round counters and their key=value record. Field meaning and line format
// are the reference's (proj/src/core/stats.hpp:9-41, stats.cpp:20-48) so
// sgnn_engine_stats_line is a drop-in; the counters are accumulated on the
// device (device/engine.cu) and copied back once per round.
#pragma once

#include <string>
#include <vector>

#include "common.hpp"

namespace sgb {

struct LayerStats {
  uint64_t events = 0, grouped_targets = 0, user_targets = 0, no_deletion = 0, deletion_no_effect = 0,
           covered_reset = 0, exposed_reset = 0, recomputes = 0, dirty_nodes = 0, fetch_rows = 0;
};

struct RoundStats {
  uint64_t round_index = 0;
  uint64_t num_updates = 0;
  std::vector<LayerStats> layers;
  uint64_t checkpoint_fetches = 0;
  uint64_t feature_fetches = 0;
  bool has_baseline = false;
  uint64_t affected_fetches = 0, full_fetches = 0, affected_area_nodes = 0;

  std::string to_line() const;
};

}  // namespace sgb

namespace sgb {

// RoundStats::from_line of the reference (stats.cpp:50-119): key=value tokens,
// per-layer keys l<i>.<field>; a token without '=' is Errc::format "bad stats
// token: <tok>", a layer index outside 1..layers is Errc::format "bad layer
// index in stats: <key>"; totals are recomputed from the layers, unknown keys
// ignored.
RoundStats stats_from_line(const std::string& line);

// The `report` aggregation of the reference CLI (tools/streamgnn_cli.cpp:93-172,
// summarize + print_report) for one stats file: condition distribution over
// visited targets, incremental fraction, engine fetches and, when the lines
// carry baseline counters, the fetch reduction and dirty/area ratio. Same text,
// byte for byte. Missing file: Errc::io "cannot open stats file: <path>".
std::string stats_report(const std::string& path);

}  // namespace sgb
