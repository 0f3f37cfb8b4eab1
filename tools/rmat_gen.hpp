// BENCHMARK / TEST HARNESS — not product code.
//
// Seeded synthetic inputs for the BASELINE.json configurations:
//   * an R-MAT power-law directed graph, (a,b,c,d) = (0.57,0.19,0.19,0.05), ids in
//     a 2^ceil(log2 N) space with rejection of ids >= N, a random relabelling,
//     self-loops and duplicates rejected, exactly E distinct edges sorted by (src,dst);
//   * a 50/50 insert/delete update stream over it (inserts from the same R-MAT
//     distribution, never a live edge; deletes uniform over the live edges);
//   * row-major uniform [0,1) features built like the reference's Rng::unit
//     (proj/src/core/synth.hpp:14-24: std::mt19937_64, top 24 bits / 2^24).
// Candidates are counter-based (splitmix64 of (stream, index)), so the output
// does not depend on the thread count.
//
// This header is compiled into two harness libraries and nowhere else:
//   tools/libsgnn_datagen.so  (bench.py's B200 arm, tests)
//   oracle/_ref/libstreamgnn_ref.so (bench.py's reference arm, via oracle/ref_harness.cpp)
// so both arms of the benchmark build byte-identical inputs without the
// reference arm loading the product library.
#pragma once

#include <algorithm>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <thread>
#include <unordered_set>
#include <utility>
#include <vector>

namespace sgnn_tools {

inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

inline uint64_t edge_key(uint32_t s, uint32_t d) { return (static_cast<uint64_t>(s) << 32) | d; }

struct Rmat {
  uint32_t n;
  int scale = 0;
  uint64_t seed;
  std::vector<uint32_t> perm;  // random relabelling of [0, n)

  Rmat(uint32_t num_nodes, uint64_t s) : n(num_nodes), seed(s) {
    while ((uint64_t(1) << scale) < n) ++scale;
    perm.resize(n);
    for (uint32_t i = 0; i < n; ++i) perm[i] = i;
    std::mt19937_64 eng(seed ^ 0xA5A5F00DULL);
    for (uint32_t i = n; i > 1; --i) std::swap(perm[i - 1], perm[eng() % i]);
  }

  // Candidate i of the counter stream `stream`; false when rejected.
  bool candidate(uint64_t stream, uint64_t i, uint32_t& s, uint32_t& d) const {
    // (a, a+b, a+b+c) = (0.57, 0.76, 0.95) on 16-bit draws
    constexpr uint32_t A = 37355, AB = 49807, ABC = 62259;
    uint64_t st = splitmix64(seed ^ splitmix64(stream * 0x632BE59BD9B4E019ull + i));
    uint64_t bits = st;
    uint32_t u = 0, v = 0;
    for (int l = 0; l < scale; ++l) {
      if (l && (l & 3) == 0) {
        st = splitmix64(st);
        bits = st;
      }
      const uint32_t r = static_cast<uint32_t>(bits & 0xFFFF);
      bits >>= 16;
      const uint32_t ub = r >= AB, vb = (r >= A && r < AB) || r >= ABC;
      u = (u << 1) | ub;
      v = (v << 1) | vb;
    }
    if (u >= n || v >= n || u == v) return false;
    s = perm[u];
    d = perm[v];
    return true;
  }
};

inline unsigned num_threads() { return std::max(1u, std::min(32u, std::thread::hardware_concurrency())); }

// Sorts keys (src << 32 | dst, src < n) by bucketing on src, then sorting buckets.
inline void sort_keys(std::vector<uint64_t>& keys, uint32_t n) {
  const unsigned T = num_threads();
  std::vector<uint64_t> off(static_cast<size_t>(n) + 1, 0);
  for (uint64_t k : keys) ++off[(k >> 32) + 1];
  for (uint32_t v = 0; v < n; ++v) off[v + 1] += off[v];
  std::vector<uint64_t> out(keys.size());
  std::vector<uint64_t> pos(off.begin(), off.end() - 1);
  for (uint64_t k : keys) out[pos[k >> 32]++] = k;
  std::vector<std::thread> th;
  for (unsigned t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      for (uint64_t v = t; v < n; v += T) std::sort(out.begin() + off[v], out.begin() + off[v + 1]);
    });
  for (auto& x : th) x.join();
  keys.swap(out);
}

// Base graph: exactly num_edges distinct (src,dst), sorted by (src,dst).
inline void gen_rmat_graph(uint32_t num_nodes, uint64_t num_edges, uint64_t seed, uint32_t* src, uint32_t* dst) {
  if (num_nodes < 2) throw std::invalid_argument("need at least two nodes");
  if (num_edges > static_cast<uint64_t>(num_nodes) * (num_nodes - 1))
    throw std::invalid_argument("average degree too high for a simple graph");
  Rmat rm(num_nodes, seed);
  std::vector<uint64_t> uniq;
  uint64_t next = 0;
  const unsigned T = num_threads();
  for (int round = 0; uniq.size() < num_edges; ++round) {
    if (round > 64) throw std::invalid_argument("R-MAT generator cannot reach the requested edge count");
    const uint64_t need = num_edges - uniq.size();
    const uint64_t batch = need + need / 3 + 4096;
    std::vector<std::vector<uint64_t>> part(T);
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        const uint64_t b = next + batch * t / T, e = next + batch * (t + 1) / T;
        part[t].reserve(e - b);
        for (uint64_t i = b; i < e; ++i) {
          uint32_t s, d;
          if (rm.candidate(0, i, s, d)) part[t].push_back(edge_key(s, d));
        }
      });
    for (auto& x : th) x.join();
    next += batch;
    std::vector<uint64_t> cand = std::move(uniq);
    for (auto& p : part) cand.insert(cand.end(), p.begin(), p.end());
    sort_keys(cand, num_nodes);
    cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
    uniq.swap(cand);
  }
  if (uniq.size() > num_edges) {
    // Keep a hash-ranked subset so the selection does not depend on key order.
    std::vector<std::pair<uint64_t, uint64_t>> ranked(uniq.size());
    for (size_t i = 0; i < uniq.size(); ++i) ranked[i] = {splitmix64(uniq[i] ^ seed), uniq[i]};
    std::nth_element(ranked.begin(), ranked.begin() + static_cast<long>(num_edges), ranked.end());
    uniq.resize(num_edges);
    for (uint64_t i = 0; i < num_edges; ++i) uniq[i] = ranked[i].second;
    sort_keys(uniq, num_nodes);
  }
  for (uint64_t i = 0; i < num_edges; ++i) {
    src[i] = static_cast<uint32_t>(uniq[i] >> 32);
    dst[i] = static_cast<uint32_t>(uniq[i]);
  }
}

// Update stream over a base graph given as (src,dst) arrays.
inline void gen_rmat_stream(uint32_t num_nodes, const uint32_t* base_src, const uint32_t* base_dst,
                            uint64_t num_edges, uint64_t stream_len, double insert_fraction, uint64_t seed,
                            char* ops, uint32_t* src, uint32_t* dst) {
  Rmat rm(num_nodes, seed);
  std::vector<uint64_t> base(num_edges);
  for (uint64_t i = 0; i < num_edges; ++i) base[i] = edge_key(base_src[i], base_dst[i]);
  if (!std::is_sorted(base.begin(), base.end())) sort_keys(base, num_nodes);
  std::unordered_set<uint64_t> deleted_base;  // indices into base
  std::vector<uint64_t> inserted;              // keys in insertion order
  std::vector<char> inserted_dead;
  std::unordered_set<uint64_t> inserted_live;  // keys
  uint64_t n_deleted = 0, n_live_inserted = 0;
  std::mt19937_64 rng(seed ^ 0x5EEDULL);
  auto unit = [&] { return static_cast<float>(rng() >> 40) * (1.0f / 16777216.0f); };
  uint64_t cand = 0;
  auto base_live = [&](uint64_t key) {
    auto it = std::lower_bound(base.begin(), base.end(), key);
    if (it == base.end() || *it != key) return false;
    return !deleted_base.count(static_cast<uint64_t>(it - base.begin()));
  };
  for (uint64_t i = 0; i < stream_len; ++i) {
    const uint64_t live = num_edges - n_deleted + n_live_inserted;
    const bool insert = live == 0 || unit() < insert_fraction;
    if (insert) {
      for (;;) {
        uint32_t s, d;
        if (!rm.candidate(1, cand++, s, d)) continue;
        const uint64_t key = edge_key(s, d);
        if (base_live(key) || inserted_live.count(key)) continue;
        inserted.push_back(key);
        inserted_dead.push_back(0);
        inserted_live.insert(key);
        ++n_live_inserted;
        ops[i] = '+';
        src[i] = s;
        dst[i] = d;
        break;
      }
    } else {
      for (;;) {
        const uint64_t r = rng() % (num_edges + inserted.size());
        uint64_t key;
        if (r < num_edges) {
          if (deleted_base.count(r)) continue;
          deleted_base.insert(r);
          ++n_deleted;
          key = base[r];
        } else {
          const uint64_t j = r - num_edges;
          if (inserted_dead[j]) continue;
          inserted_dead[j] = 1;
          key = inserted[j];
          inserted_live.erase(key);
          --n_live_inserted;
        }
        ops[i] = '-';
        src[i] = static_cast<uint32_t>(key >> 32);
        dst[i] = static_cast<uint32_t>(key);
        break;
      }
    }
  }
}

// Row-major uniform [0,1) features (reference Rng::unit construction).
inline void gen_features(uint32_t rows, uint32_t cols, uint64_t seed, float* out) {
  std::mt19937_64 rng(seed);
  const size_t n = static_cast<size_t>(rows) * cols;
  for (size_t i = 0; i < n; ++i) out[i] = static_cast<float>(rng() >> 40) * (1.0f / 16777216.0f);
}

}  // namespace sgnn_tools
