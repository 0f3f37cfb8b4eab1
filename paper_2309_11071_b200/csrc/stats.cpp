#include "stats.hpp"

#include <sstream>

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

}  // namespace sgb
