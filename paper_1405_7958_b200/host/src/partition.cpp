// Box partitions (see rt/partition.hpp).
#include "rt/partition.hpp"

#include <algorithm>
#include <array>
#include <string>

namespace rt {

std::vector<BoundingBox> partition_regular(const BoundingBox& box,
                                           std::span<const std::int64_t> tile) {
  if (box.empty()) return {};
  const int d = box.dims();
  if (int(tile.size()) != d)
    throw PartitionError("partition of a rank-" + std::to_string(d) + " box with rank-" +
                         std::to_string(tile.size()) + " tiles");
  // tiles per axis, then the total: tile k's grid coordinate is k written in
  // the mixed radix of those counts (last axis fastest)
  std::array<std::int64_t, BoundingBox::kMaxDims> count{};
  std::int64_t total = 1;
  for (int a = 0; a < d; ++a) {
    if (tile[std::size_t(a)] <= 0)
      throw PartitionError("tile extent on axis " + std::to_string(a) + " is not positive");
    count[std::size_t(a)] = (box.extent(a) + tile[std::size_t(a)] - 1) / tile[std::size_t(a)];
    total *= count[std::size_t(a)];
  }
  std::vector<BoundingBox> out;
  out.reserve(std::size_t(total));
  for (std::int64_t k = 0; k < total; ++k) {
    std::int64_t lo[BoundingBox::kMaxDims], hi[BoundingBox::kMaxDims];
    std::int64_t rest = k;
    for (int a = d - 1; a >= 0; --a) {
      const std::int64_t g = rest % count[std::size_t(a)];
      rest /= count[std::size_t(a)];
      lo[a] = box.lo(a) + g * tile[std::size_t(a)];
      hi[a] = std::min(lo[a] + tile[std::size_t(a)] - 1, box.hi(a));
    }
    out.emplace_back(d, lo, hi);
  }
  return out;
}

std::vector<BoundingBox> partition_regular(const BoundingBox& box,
                                           std::initializer_list<std::int64_t> tile) {
  return partition_regular(box, std::span<const std::int64_t>(tile.begin(), tile.size()));
}

std::vector<BoundingBox> partition_custom(const BoundingBox& box, std::vector<BoundingBox> boxes) {
  for (const BoundingBox& b : boxes) {
    // a rank mismatch surfaces as contains()'s DimensionError
    const bool inside = !b.empty() && !box.empty() && box.contains(b);
    if (!inside) throw PartitionError("custom tile " + b.to_string() + " is not inside " + box.to_string());
  }
  return boxes;
}

}  // namespace rt
