#include "stats.hpp"

#include <algorithm>
#include <cstdio>
#include <fstream>
#include <map>
#include <sstream>
#include <utility>

namespace sgb {

std::string RoundStats::to_line() const {
  LayerStats t;
  for (const LayerStats& l : layers) {
    t.events += l.events;
    t.grouped_targets += l.grouped_targets;
    t.user_targets += l.user_targets;
    t.no_deletion += l.no_deletion;
    t.deletion_no_effect += l.deletion_no_effect;
    t.covered_reset += l.covered_reset;
    t.exposed_reset += l.exposed_reset;
    t.recomputes += l.recomputes;
    t.dirty_nodes += l.dirty_nodes;
  }
  std::ostringstream o;
  o << "round=" << round_index << " updates=" << num_updates << " layers=" << layers.size()
    << " events=" << t.events << " targets=" << t.grouped_targets << " user_targets=" << t.user_targets
    << " no_deletion=" << t.no_deletion << " deletion_no_effect=" << t.deletion_no_effect
    << " covered_reset=" << t.covered_reset << " exposed_reset=" << t.exposed_reset
    << " recomputes=" << t.recomputes << " dirty=" << t.dirty_nodes << " ckpt_fetches=" << checkpoint_fetches
    << " feat_fetches=" << feature_fetches;
  if (has_baseline)
    o << " affected_fetches=" << affected_fetches << " full_fetches=" << full_fetches
      << " area_nodes=" << affected_area_nodes;
  for (size_t i = 0; i < layers.size(); ++i) {
    const LayerStats& l = layers[i];
    const std::string p = " l" + std::to_string(i + 1) + ".";
    o << p << "events=" << l.events << p << "targets=" << l.grouped_targets << p << "user_targets=" << l.user_targets
      << p << "no_deletion=" << l.no_deletion << p << "deletion_no_effect=" << l.deletion_no_effect << p
      << "covered_reset=" << l.covered_reset << p << "exposed_reset=" << l.exposed_reset << p
      << "recomputes=" << l.recomputes << p << "dirty=" << l.dirty_nodes << p << "fetch_rows=" << l.fetch_rows;
  }
  return o.str();
}

RoundStats stats_from_line(const std::string& line) {
  RoundStats st;
  std::istringstream in(line);
  std::string tok;
  std::vector<std::pair<std::string, std::string>> kvs;
  while (in >> tok) {
    const size_t eq = tok.find('=');
    if (eq == std::string::npos) fail(Errc::format, "bad stats token: " + tok);
    kvs.emplace_back(tok.substr(0, eq), tok.substr(eq + 1));
  }
  size_t num_layers = 0;
  for (const auto& [key, v] : kvs)
    if (key == "layers") num_layers = std::stoull(v);
  st.layers.resize(num_layers);
  for (const auto& [key, v] : kvs) {
    const uint64_t val = std::stoull(v);
    if (key == "round") {
      st.round_index = val;
    } else if (key == "updates") {
      st.num_updates = val;
    } else if (key == "ckpt_fetches") {
      st.checkpoint_fetches = val;
    } else if (key == "feat_fetches") {
      st.feature_fetches = val;
    } else if (key == "affected_fetches" || key == "full_fetches" || key == "area_nodes") {
      (key == "affected_fetches" ? st.affected_fetches
                                 : (key == "full_fetches" ? st.full_fetches : st.affected_area_nodes)) = val;
      st.has_baseline = true;
    } else if (key.size() > 1 && key[0] == 'l' && key.find('.') != std::string::npos) {
      const size_t dot = key.find('.');
      const size_t idx = std::stoull(key.substr(1, dot - 1));
      if (idx < 1 || idx > num_layers) fail(Errc::format, "bad layer index in stats: " + key);
      LayerStats& l = st.layers[idx - 1];
      const std::string f = key.substr(dot + 1);
      uint64_t LayerStats::* field = nullptr;
      if (f == "events") field = &LayerStats::events;
      else if (f == "targets") field = &LayerStats::grouped_targets;
      else if (f == "user_targets") field = &LayerStats::user_targets;
      else if (f == "no_deletion") field = &LayerStats::no_deletion;
      else if (f == "deletion_no_effect") field = &LayerStats::deletion_no_effect;
      else if (f == "covered_reset") field = &LayerStats::covered_reset;
      else if (f == "exposed_reset") field = &LayerStats::exposed_reset;
      else if (f == "recomputes") field = &LayerStats::recomputes;
      else if (f == "dirty") field = &LayerStats::dirty_nodes;
      else if (f == "fetch_rows") field = &LayerStats::fetch_rows;
      if (field) l.*field = val;
    }
  }
  return st;
}

namespace {

// Whole-round totals a stats file aggregates (streamgnn_cli.cpp:95-103).
struct ReportSums {
  uint64_t rounds = 0, no_deletion = 0, deletion_no_effect = 0, covered_reset = 0, exposed_reset = 0;
  uint64_t engine_fetches = 0, affected_fetches = 0, full_fetches = 0, area_nodes = 0, dirty_nodes = 0;
  bool has_baseline = false;
  std::vector<double> reduction;  // affected / engine, per round with baseline counters
};

template <typename... A>
void appendf(std::string& out, const char* fmt, A... a) {
  char buf[512];
  const int n = std::snprintf(buf, sizeof buf, fmt, a...);
  out.append(buf, static_cast<size_t>(std::max(0, std::min(n, static_cast<int>(sizeof buf) - 1))));
}

}  // namespace

std::string stats_report(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(Errc::io, "cannot open stats file: " + path);
  ReportSums s;
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    // lenient key=value scan: tokens without '=' are skipped, absent keys read 0
    std::map<std::string, uint64_t> kv;
    std::istringstream ls(line);
    std::string tok;
    while (ls >> tok) {
      const size_t eq = tok.find('=');
      if (eq != std::string::npos) kv[tok.substr(0, eq)] = std::stoull(tok.substr(eq + 1));
    }
    if (!kv.count("round")) continue;
    ++s.rounds;
    s.no_deletion += kv["no_deletion"];
    s.deletion_no_effect += kv["deletion_no_effect"];
    s.covered_reset += kv["covered_reset"];
    s.exposed_reset += kv["exposed_reset"];
    const uint64_t engine = kv["ckpt_fetches"] + kv["feat_fetches"];
    s.engine_fetches += engine;
    s.dirty_nodes += kv["dirty"];
    if (kv.count("affected_fetches")) {
      s.has_baseline = true;
      s.affected_fetches += kv["affected_fetches"];
      s.full_fetches += kv["full_fetches"];
      s.area_nodes += kv["area_nodes"];
      s.reduction.push_back(static_cast<double>(kv["affected_fetches"]) / (engine ? static_cast<double>(engine) : 1.0));
    }
  }
  const uint64_t visited = s.no_deletion + s.deletion_no_effect + s.covered_reset + s.exposed_reset;
  auto pct = [&](uint64_t n) { return visited ? 100.0 * static_cast<double>(n) / static_cast<double>(visited) : 0.0; };
  using ull = unsigned long long;
  std::string o;
  appendf(o, "stream %s\n", path.c_str());
  appendf(o, "  rounds                 %llu\n", static_cast<ull>(s.rounds));
  appendf(o, "  visited targets        %llu\n", static_cast<ull>(visited));
  appendf(o, "  no deletion            %6.2f%%\n", pct(s.no_deletion));
  appendf(o, "  deletion no effect     %6.2f%%\n", pct(s.deletion_no_effect));
  appendf(o, "  covered reset          %6.2f%%\n", pct(s.covered_reset));
  appendf(o, "  exposed reset          %6.2f%%\n", pct(s.exposed_reset));
  appendf(o, "  incremental fraction   %6.2f%%\n", pct(s.no_deletion + s.deletion_no_effect + s.covered_reset));
  appendf(o, "  engine fetches         %llu\n", static_cast<ull>(s.engine_fetches));
  if (s.has_baseline) {
    appendf(o, "  affected fetches       %llu\n", static_cast<ull>(s.affected_fetches));
    appendf(o, "  full fetches           %llu\n", static_cast<ull>(s.full_fetches));
    const double overall =
        s.engine_fetches ? static_cast<double>(s.affected_fetches) / static_cast<double>(s.engine_fetches) : 0.0;
    std::vector<double> sorted = s.reduction;
    std::sort(sorted.begin(), sorted.end());
    const double median = sorted.empty() ? 0.0 : sorted[sorted.size() / 2];
    appendf(o, "  fetch reduction        %.2fx overall, %.2fx median per round\n", overall, median);
    if (s.area_nodes)
      appendf(o, "  dirty/theoretical area %6.2f%%\n",
              100.0 * static_cast<double>(s.dirty_nodes) / static_cast<double>(s.area_nodes));
  }
  return o;
}

}  // namespace sgb
