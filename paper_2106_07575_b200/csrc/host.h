// Host-only helpers (partition, rounding, tile lists); see host.cpp.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "ptyger.h"

namespace pty {

// foot: rows a frame's window touches (N; N + 1 for bilinear fractional positions, R#22)
int partition(const int32_t* scan, int64_t n, int64_t H, int N, int P, std::vector<int32_t>& rank,
              std::vector<int64_t>& rows, std::string& err, int foot = -1);
int max_feasible_P(const int32_t* scan, int64_t n, int N, int limit);
void canonical_order(const int32_t* scan, int64_t n, int N, std::vector<int64_t>& idx);
void round_positions(const float* raw, int64_t n, int32_t* out);
void build_tiles(const std::vector<int32_t>& lpos, const std::vector<int32_t>& order, int foot, int64_t SH,
                 int64_t W, int& ntx, int& nty, std::vector<int32_t>& tile_ptr,
                 std::vector<int32_t>& entries);

}  // namespace pty
