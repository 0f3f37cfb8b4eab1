#include "host_graph.hpp"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <thread>

namespace sgb {

namespace {

struct FileCloser {
  void operator()(FILE* f) const {
    if (f) std::fclose(f);
  }
};
using File = std::unique_ptr<FILE, FileCloser>;

// Whitespace set of the "C" locale, as used by operator>> on the reference's
// istringstream tokenisation.
inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

// Up to `max_tok` tokens of [b, e); returns the number found (capped at max_tok+1
// to signal trailing tokens).
int tokenize(const char* b, const char* e, std::pair<const char*, const char*>* tok, int max_tok) {
  int n = 0;
  const char* p = b;
  while (p < e) {
    while (p < e && is_ws(*p)) ++p;
    if (p >= e) break;
    const char* s = p;
    while (p < e && !is_ws(*p)) ++p;
    if (n < max_tok) tok[n] = {s, p};
    ++n;
    if (n > max_tok) break;
  }
  return n;
}

// Decimal digits only, value <= UINT32_MAX (reference parse_node_id, graph.cpp:135-147).
bool parse_node_id(const char* b, const char* e, NodeId& out) {
  if (b == e) return false;
  uint64_t v = 0;
  for (const char* p = b; p < e; ++p) {
    if (*p < '0' || *p > '9') return false;
    v = v * 10 + static_cast<uint64_t>(*p - '0');
    if (v > UINT32_MAX) return false;
  }
  out = static_cast<NodeId>(v);
  return true;
}

std::string read_file(const std::string& path, const char* what) {
  File f(std::fopen(path.c_str(), "rb"));
  if (!f) fail(Errc::io, std::string("cannot open ") + what + ": " + path);
  std::string buf;
  std::fseek(f.get(), 0, SEEK_END);
  long size = std::ftell(f.get());
  std::fseek(f.get(), 0, SEEK_SET);
  if (size > 0) {
    buf.resize(static_cast<size_t>(size));
    size_t got = std::fread(buf.data(), 1, buf.size(), f.get());
    buf.resize(got);
  }
  return buf;
}

template <typename Fn>
void parallel_for(size_t n, Fn&& fn) {
  unsigned t = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (n < 4096 || t == 1) {
    fn(size_t(0), n);
    return;
  }
  std::vector<std::thread> th;
  size_t chunk = (n + t - 1) / t;
  for (unsigned i = 0; i < t; ++i) {
    size_t b = i * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    th.emplace_back([&, b, e] { fn(b, e); });
  }
  for (auto& x : th) x.join();
}

}  // namespace

HostGraph::HostGraph(uint32_t num_nodes) : n_(num_nodes) {
  if (num_nodes == 0) fail(Errc::invalid_argument, "graph must have at least one node");
  out_.resize(num_nodes);
  in_.resize(num_nodes);
}

void HostGraph::check_node(NodeId u) const {
  if (u >= n_) fail(Errc::invalid_argument, "node id out of range: " + std::to_string(u));
}

bool HostGraph::has_edge(NodeId src, NodeId dst) const {
  check_node(src);
  check_node(dst);
  const auto& o = out_[src];
  return std::binary_search(o.begin(), o.end(), dst);
}

void HostGraph::add_edge(NodeId src, NodeId dst) {
  if (has_edge(src, dst))
    fail(Errc::duplicate_edge, "duplicate edge " + std::to_string(src) + "->" + std::to_string(dst));
  auto& o = out_[src];
  o.insert(std::lower_bound(o.begin(), o.end(), dst), dst);
  auto& i = in_[dst];
  i.insert(std::lower_bound(i.begin(), i.end(), src), src);
  ++m_;
}

const std::vector<NodeId>& HostGraph::out(NodeId u) const {
  check_node(u);
  return out_[u];
}

const std::vector<NodeId>& HostGraph::in(NodeId u) const {
  check_node(u);
  return in_[u];
}

HostGraph HostGraph::from_edges(uint32_t num_nodes, const NodeId* src, const NodeId* dst, size_t count,
                                bool symmetrize) {
  HostGraph g(num_nodes);
  // The first failing add_edge in input order decides the error: an
  // out-of-range id, or (without symmetrize) the second occurrence of an edge.
  size_t first_range = count;
  for (size_t i = 0; i < count; ++i)
    if (src[i] >= num_nodes || dst[i] >= num_nodes) {
      first_range = i;
      break;
    }
  size_t valid = first_range;  // edges before the first range error are all well-formed

  // Bucket by source: (dst << 32 | input index) per bucket, sorted.
  std::vector<uint64_t> cnt(num_nodes + 1, 0);
  auto push_count = [&](NodeId s) { ++cnt[s + 1]; };
  for (size_t i = 0; i < valid; ++i) {
    push_count(src[i]);
    if (symmetrize && src[i] != dst[i]) push_count(dst[i]);
  }
  for (uint32_t v = 0; v < num_nodes; ++v) cnt[v + 1] += cnt[v];
  std::vector<uint64_t> pos(cnt.begin(), cnt.end() - 1);
  std::vector<uint64_t> pairs(cnt[num_nodes]);
  for (size_t i = 0; i < valid; ++i) {
    pairs[pos[src[i]]++] = (static_cast<uint64_t>(dst[i]) << 32) | static_cast<uint32_t>(i);
    if (symmetrize && src[i] != dst[i]) pairs[pos[dst[i]]++] = (static_cast<uint64_t>(src[i]) << 32) | static_cast<uint32_t>(i);
  }
  size_t first_dup = count;
  std::vector<size_t> dup_at(16, count);
  std::vector<std::pair<uint32_t, uint32_t>> dup_edge(16);
  {
    // per-thread minimum of the failing index
    std::vector<std::thread> th;
    unsigned t = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    uint32_t chunk = (num_nodes + t - 1) / t;
    for (unsigned ti = 0; ti < t; ++ti) {
      th.emplace_back([&, ti] {
        uint32_t b = ti * chunk, e = std::min<uint64_t>(num_nodes, uint64_t(b) + chunk);
        for (uint32_t u = b; u < e; ++u) {
          uint64_t* p0 = pairs.data() + cnt[u];
          uint64_t* p1 = pairs.data() + cnt[u + 1];
          std::sort(p0, p1);
          if (!symmetrize)
            for (uint64_t* p = p0 + 1; p < p1; ++p)
              if ((*p >> 32) == (p[-1] >> 32) && (p == p0 + 1 || (p[-2] >> 32) != (*p >> 32))) {
                size_t idx = static_cast<uint32_t>(*p);
                if (idx < dup_at[ti]) {
                  dup_at[ti] = idx;
                  dup_edge[ti] = {u, static_cast<uint32_t>(*p >> 32)};
                }
              }
        }
      });
    }
    for (auto& x : th) x.join();
    std::pair<uint32_t, uint32_t> e{0, 0};
    for (unsigned ti = 0; ti < dup_at.size(); ++ti)
      if (dup_at[ti] < first_dup) {
        first_dup = dup_at[ti];
        e = dup_edge[ti];
      }
    if (first_dup < first_range)
      fail(Errc::duplicate_edge, "duplicate edge " + std::to_string(e.first) + "->" + std::to_string(e.second));
  }
  if (first_range < count) {
    NodeId bad = src[first_range] >= num_nodes ? src[first_range] : dst[first_range];
    fail(Errc::invalid_argument, "node id out of range: " + std::to_string(bad));
  }
  // Dedup (symmetrize) and materialise sorted lists.
  std::vector<uint32_t> indeg(num_nodes, 0);
  parallel_for(num_nodes, [&](size_t b, size_t e) {
    for (size_t u = b; u < e; ++u) {
      auto& o = g.out_[u];
      o.reserve(cnt[u + 1] - cnt[u]);
      for (uint64_t k = cnt[u]; k < cnt[u + 1]; ++k) {
        NodeId v = static_cast<NodeId>(pairs[k] >> 32);
        if (o.empty() || o.back() != v) o.push_back(v);
      }
    }
  });
  uint64_t m = 0;
  for (uint32_t u = 0; u < num_nodes; ++u) {
    m += g.out_[u].size();
    for (NodeId v : g.out_[u]) ++indeg[v];
  }
  for (uint32_t v = 0; v < num_nodes; ++v) g.in_[v].reserve(indeg[v]);
  for (uint32_t u = 0; u < num_nodes; ++u)
    for (NodeId v : g.out_[u]) g.in_[v].push_back(u);
  g.m_ = m;
  return g;
}

HostGraph HostGraph::padded(uint32_t num_nodes) const {
  HostGraph g = *this;
  if (num_nodes > n_) {
    g.n_ = num_nodes;
    g.out_.resize(num_nodes);
    g.in_.resize(num_nodes);
  }
  return g;
}

HostGraph load_edge_list(const std::string& path, bool symmetrize) {
  std::string buf = read_file(path, "edge list");
  std::vector<NodeId> src, dst;
  NodeId max_id = 0;
  size_t lineno = 0;
  const char* p = buf.data();
  const char* end = p + buf.size();
  while (p < end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    const char* le = nl ? nl : end;
    ++lineno;
    std::pair<const char*, const char*> tok[2];
    int n = tokenize(p, le, tok, 2);
    p = nl ? nl + 1 : end;
    if (n == 0) continue;
    if (*tok[0].first == '#') continue;
    NodeId s = 0, d = 0;
    if (n != 2 || !parse_node_id(tok[0].first, tok[0].second, s) || !parse_node_id(tok[1].first, tok[1].second, d))
      fail(Errc::format, "bad edge line " + std::to_string(lineno) + " in " + path);
    src.push_back(s);
    dst.push_back(d);
    max_id = std::max({max_id, s, d});
  }
  uint32_t n = src.empty() ? 1u : max_id + 1u;
  return HostGraph::from_edges(n, src.data(), dst.data(), src.size(), symmetrize);
}

namespace {

constexpr char kBinMagic[8] = {'S', 'G', 'N', 'N', 'E', 'D', 'G', '1'};

void read_exact(std::FILE* f, void* dst, size_t bytes, const std::string& path) {
  char* p = static_cast<char*>(dst);
  while (bytes) {
    const size_t want = std::min<size_t>(bytes, 1u << 28);
    const size_t got = std::fread(p, 1, want, f);
    if (got != want) fail(Errc::format, "truncated binary edge list: " + path);
    p += got;
    bytes -= got;
  }
}

}  // namespace

HostGraph load_edge_list_binary(const std::string& path, bool symmetrize) {
  File f(std::fopen(path.c_str(), "rb"));
  if (!f) fail(Errc::io, "cannot open edge list: " + path);
  char magic[8];
  uint32_t hdr[2];
  uint64_t count = 0;
  if (std::fread(magic, 1, 8, f.get()) != 8 || std::memcmp(magic, kBinMagic, 8) != 0 ||
      std::fread(hdr, 4, 2, f.get()) != 2 || std::fread(&count, 8, 1, f.get()) != 1)
    fail(Errc::format, "bad binary edge list header: " + path);
  std::vector<NodeId> src(count), dst(count);
  read_exact(f.get(), src.data(), count * 4, path);
  read_exact(f.get(), dst.data(), count * 4, path);
  NodeId max_id = 0;
  for (uint64_t i = 0; i < count; ++i) max_id = std::max({max_id, src[i], dst[i]});
  if (count && max_id == 0xFFFFFFFFu) fail(Errc::invalid_argument, "node id out of range: 4294967295");
  const uint32_t n = std::max<uint32_t>(hdr[0], count ? max_id + 1u : 1u);
  return HostGraph::from_edges(n, src.data(), dst.data(), count, symmetrize);
}

void save_edge_list_binary(const HostGraph& g, const std::string& path) {
  File f(std::fopen(path.c_str(), "wb"));
  if (!f) fail(Errc::io, "cannot open for write: " + path);
  const uint64_t m = g.num_edges();
  std::vector<NodeId> src, dst;
  src.reserve(m);
  dst.reserve(m);
  for (NodeId u = 0; u < g.num_nodes(); ++u)
    for (NodeId v : g.out(u)) {
      src.push_back(u);
      dst.push_back(v);
    }
  const uint32_t hdr[2] = {g.num_nodes(), 0};
  bool ok = std::fwrite(kBinMagic, 1, 8, f.get()) == 8 && std::fwrite(hdr, 4, 2, f.get()) == 2 &&
            std::fwrite(&m, 8, 1, f.get()) == 1 && std::fwrite(src.data(), 4, m, f.get()) == m &&
            std::fwrite(dst.data(), 4, m, f.get()) == m;
  if (!ok || std::fflush(f.get()) != 0) fail(Errc::io, "write failed: " + path);
}

namespace {

char* put_u32(char* p, uint32_t v) {
  char tmp[12];
  int n = 0;
  do {
    tmp[n++] = static_cast<char>('0' + v % 10);
    v /= 10;
  } while (v);
  while (n) *p++ = tmp[--n];
  return p;
}

}  // namespace

void save_edge_list(const HostGraph& g, const std::string& path) {
  File f(std::fopen(path.c_str(), "wb"));
  if (!f) fail(Errc::io, "cannot open for write: " + path);
  std::vector<char> buf(1 << 20);
  size_t used = 0;
  bool ok = true;
  for (NodeId u = 0; u < g.num_nodes(); ++u)
    for (NodeId v : g.out(u)) {
      if (used + 24 > buf.size()) {
        ok &= std::fwrite(buf.data(), 1, used, f.get()) == used;
        used = 0;
      }
      char* q = buf.data() + used;
      q = put_u32(q, u);
      *q++ = ' ';
      q = put_u32(q, v);
      *q++ = '\n';
      used = static_cast<size_t>(q - buf.data());
    }
  ok &= std::fwrite(buf.data(), 1, used, f.get()) == used;
  if (!ok || std::fflush(f.get()) != 0) fail(Errc::io, "write failed: " + path);
}

void save_edge_list_csr(uint32_t num_nodes, const uint64_t* offsets, const NodeId* targets, const std::string& path) {
  File f(std::fopen(path.c_str(), "wb"));
  if (!f) fail(Errc::io, "cannot open for write: " + path);
  std::vector<char> buf(1 << 20);
  size_t used = 0;
  bool ok = true;
  for (NodeId u = 0; u < num_nodes; ++u)
    for (uint64_t k = offsets[u]; k < offsets[u + 1]; ++k) {
      if (used + 24 > buf.size()) {
        ok &= std::fwrite(buf.data(), 1, used, f.get()) == used;
        used = 0;
      }
      char* q = buf.data() + used;
      q = put_u32(q, u);
      *q++ = ' ';
      q = put_u32(q, targets[k]);
      *q++ = '\n';
      used = static_cast<size_t>(q - buf.data());
    }
  ok &= std::fwrite(buf.data(), 1, used, f.get()) == used;
  if (!ok || std::fflush(f.get()) != 0) fail(Errc::io, "write failed: " + path);
}

std::vector<EdgeDelta> load_update_stream(const std::string& path) {
  std::string buf = read_file(path, "update stream");
  std::vector<EdgeDelta> out;
  size_t lineno = 0;
  const char* p = buf.data();
  const char* end = p + buf.size();
  while (p < end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    const char* le = nl ? nl : end;
    ++lineno;
    std::pair<const char*, const char*> tok[3];
    int n = tokenize(p, le, tok, 3);
    p = nl ? nl + 1 : end;
    if (n == 0) continue;
    if (*tok[0].first == '#') continue;
    NodeId s = 0, d = 0;
    bool op_ok = (tok[0].second - tok[0].first) == 1 && (*tok[0].first == '+' || *tok[0].first == '-');
    if (!op_ok || n != 3 || !parse_node_id(tok[1].first, tok[1].second, s) ||
        !parse_node_id(tok[2].first, tok[2].second, d))
      fail(Errc::format, "bad stream line " + std::to_string(lineno) + " in " + path);
    out.push_back({*tok[0].first == '+' ? EdgeOp::Insert : EdgeOp::Delete, s, d});
  }
  return out;
}

void save_update_stream(const std::vector<EdgeDelta>& s, const std::string& path) {
  File f(std::fopen(path.c_str(), "wb"));
  if (!f) fail(Errc::io, "cannot open for write: " + path);
  bool ok = true;
  for (const EdgeDelta& d : s)
    ok &= std::fprintf(f.get(), "%c %u %u\n", d.op == EdgeOp::Insert ? '+' : '-', d.src, d.dst) > 0;
  if (!ok || std::fflush(f.get()) != 0) fail(Errc::io, "write failed: " + path);
}

}  // namespace sgb
