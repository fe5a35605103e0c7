// Regular and custom partitions of a box into tiles (reference
// include/rt/partition.hpp:23-41, src/partition.cpp:23-70): how a whole-slide
// image becomes the bag of per-tile stages (the 100k x 100k
// slide in 4096^2 tiles is 625 tiles = 576 full + 48 edge + 1 corner).
#pragma once

#include <cstdint>
#include <initializer_list>
#include <span>
#include <vector>

#include "rt/region.hpp"

namespace rt {

// Row-major (last axis fastest) exact cover of `box` by tiles of the given
// per-axis extents, edge tiles clamped.  Empty box -> no tiles;
// PartitionError when the tile rank differs from the box's or an extent is
// not positive.
std::vector<BoundingBox> partition_regular(const BoundingBox& box,
                                           std::span<const std::int64_t> tile);
std::vector<BoundingBox> partition_regular(const BoundingBox& box,
                                           std::initializer_list<std::int64_t> tile);

// Accepts caller-chosen boxes (overlap allowed) that all lie inside `box`;
// PartitionError for an empty box or one that escapes.
std::vector<BoundingBox> partition_custom(const BoundingBox& box, std::vector<BoundingBox> boxes);

}  // namespace rt
