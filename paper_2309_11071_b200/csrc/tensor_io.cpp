#include "tensor_io.hpp"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>

namespace sgb {

namespace {

constexpr uint32_t kMaxRank = 8;

struct FileCloser {
  void operator()(FILE* f) const {
    if (f) std::fclose(f);
  }
};
using File = std::unique_ptr<FILE, FileCloser>;

}  // namespace

HostTensor read_tensor(const std::string& path) {
  File f(std::fopen(path.c_str(), "rb"));
  if (!f) fail(Errc::io, "cannot open: " + path);
  char magic[4];
  uint32_t rank = 0;
  if (std::fread(magic, 1, 4, f.get()) != 4 || std::fread(&rank, 4, 1, f.get()) != 1 ||
      std::memcmp(magic, "TNSR", 4) != 0)
    fail(Errc::format, "not a tensor file: " + path);
  if (rank == 0 || rank > kMaxRank) fail(Errc::format, "bad tensor rank in " + path);
  HostTensor t;
  t.dims.resize(rank);
  if (std::fread(t.dims.data(), 4, rank, f.get()) != rank) fail(Errc::format, "truncated tensor header: " + path);
  size_t count = 1;
  for (uint32_t d : t.dims) {
    if (d == 0) fail(Errc::format, "zero dimension in " + path);
    count *= d;
  }
  t.data.resize(count);
  if (std::fread(t.data.data(), sizeof(float), count, f.get()) != count)
    fail(Errc::format, "truncated tensor payload: " + path);
  if (std::fgetc(f.get()) != EOF) fail(Errc::format, "trailing bytes in tensor file: " + path);
  for (float v : t.data)
    if (std::isnan(v)) fail(Errc::nan_input, "NaN in tensor file: " + path);
  for (float& v : t.data) v = flush_zero(v);
  return t;
}

void write_tensor(const std::string& path, const std::vector<uint32_t>& dims, const float* data, size_t count) {
  if (dims.empty() || dims.size() > kMaxRank) fail(Errc::invalid_argument, "write_tensor: bad rank");
  size_t expected = 1;
  for (uint32_t d : dims) expected *= d;
  if (expected != count) fail(Errc::dimension, "write_tensor: dims do not match payload");
  File f(std::fopen(path.c_str(), "wb"));
  if (!f) fail(Errc::io, "cannot open for write: " + path);
  uint32_t rank = static_cast<uint32_t>(dims.size());
  bool ok = std::fwrite("TNSR", 1, 4, f.get()) == 4 && std::fwrite(&rank, 4, 1, f.get()) == 1 &&
            std::fwrite(dims.data(), 4, rank, f.get()) == rank &&
            std::fwrite(data, sizeof(float), count, f.get()) == count;
  if (!ok || std::fflush(f.get()) != 0) fail(Errc::io, "write failed: " + path);
}

HostTensor read_matrix(const std::string& path) {
  HostTensor t = read_tensor(path);
  if (t.dims.size() != 2) fail(Errc::format, "expected rank-2 tensor: " + path);
  return t;
}

void write_matrix(const std::string& path, uint32_t rows, uint32_t cols, const float* data) {
  write_tensor(path, {rows, cols}, data, static_cast<size_t>(rows) * cols);
}

}  // namespace sgb
