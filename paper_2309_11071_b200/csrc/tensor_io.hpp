// TNSR tensor files: "TNSR", u32 rank, u32 dims[rank], f32 payload, all
// little-endian. Same format and error behaviour as the reference
// (proj/src/core/tensor_io.cpp:17-90): NaN payloads are rejected and -0 is
// flushed on load.
#pragma once

#include <string>
#include <vector>

#include "common.hpp"

namespace sgb {

struct HostTensor {
  std::vector<uint32_t> dims;
  std::vector<float> data;
};

HostTensor read_tensor(const std::string& path);
void write_tensor(const std::string& path, const std::vector<uint32_t>& dims, const float* data, size_t count);

// Rank-2 helpers (reference read_mat/write_mat, tensor_io.cpp:68-77).
HostTensor read_matrix(const std::string& path);
void write_matrix(const std::string& path, uint32_t rows, uint32_t cols, const float* data);

}  // namespace sgb
