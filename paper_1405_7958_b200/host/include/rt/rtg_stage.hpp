// The per-tile segmentation + feature stage as a Region Templates stage
// whose task has a B200 variant calling the C-ABI (include/rtg.h).
//
// This fills the slot the reference leaves empty: its simulator materialises
// stage outputs with a constant payload (src/sim.cpp:557-582) and charges
// virtual time in start_task (src/sim.cpp:630-685).  Region naming follows the
// paper's application: "RGB" input, "Mask" output (
// test_runtime.cpp:525-526 uses img::rgb -> img::mask).
#pragma once

#include <memory>
#include <mutex>
#include <vector>

#include "rt/runtime.hpp"
#include "rtg.h"

namespace rt {

// Maps an rtg_status onto the rt::Error taxonomy (the same pattern as the
// reference's throw_wire_error, src/service.cpp:181-219).
[[noreturn]] void throw_rtg_error(int status);
inline void rtg_check(int status) {
  if (status != RTG_OK) throw_rtg_error(status);
}

// RAII owner of one rtg_ctx (device arena + stream) — one per GPU worker.
class GpuDevice {
 public:
  explicit GpuDevice(int device, std::int64_t max_h = 4096, std::int64_t max_w = 4096,
                     std::int32_t max_objects = 1 << 16);
  ~GpuDevice();
  GpuDevice(const GpuDevice&) = delete;
  GpuDevice& operator=(const GpuDevice&) = delete;
  rtg_ctx* ctx() const { return ctx_; }
  int device() const { return device_; }
  std::int32_t max_objects() const { return max_objects_; }
  // A pinned max_objects x RTG_MAX_FEATURE_COLUMNS row buffer for one tile in
  // flight: the stage writes the n live rows straight into it (zero-copy
  // stores); it returns to the device's pool when the last holder drops it.
  std::shared_ptr<float> acquire_staging();
  // Pinned row buffers allocated so far (one per tile ever in flight at once).
  std::size_t staging_buffers() const;

 private:
  rtg_ctx* ctx_ = nullptr;
  int device_ = 0;
  std::int32_t max_objects_ = 0;
  mutable std::mutex mu_;
  std::vector<float*> free_, all_;
};

// Routes Chunk payloads of at least `min_bytes` into pinned host pages
// (rtg_host_alloc), recycling up to `pool_bytes` of them by size, so the GPU
// variant's H2D of the RGB tile and D2H of Mask / Labels are direct DMAs
// from / into the chunks.  At most `live_bytes` are pinned at
// once (a 625-tile slide's staged outputs alone are 50 GB); further payloads
// are plain heap blocks (correct, with a staged copy).  Call once per process
// before the tiles are staged; use_pageable_payloads() undoes it.
void use_pinned_payloads(std::size_t min_bytes = std::size_t(1) << 20,
                         std::size_t pool_bytes = std::size_t(4) << 30,
                         std::size_t live_bytes = std::size_t(16) << 30);
void use_pageable_payloads();

struct SegmentationRegions {
  // The RGB input is lazy by default: the GPU variant DMAs it straight out of
  // the store (view_region, a pitched H2D from the staged slide) and falls
  // back to touch_region when the store cannot provide a view.
  bool lazy_rgb = true;
  DataRegionId rgb{"img", "RGB", "raw", 0, 0};
  DataRegionId mask{"img", "Mask", "label", 0, 0};
  DataRegionId labels{"img", "Labels", "label", 0, 0};
  DataRegionId features{"img", "Features", "table", 0, 0};
  std::string binding = "store";
};

// Task name of the stage's single fine-grain task in a VariantRegistry.
inline constexpr const char* kSegmentFeaturesTask = "segment_features";

// Registers the B200 variant of "segment_features".  The body finds the
// tile (a zero-copy store view for a lazy input, else the local template's
// payload), installs Mask (Dense2D u8) and Labels (Dense2D i32) into the
// local template, enqueues upload / stage / download with
// rtg_process_tile_async on the worker's GpuDevice and defers the rest
// (ticket wait, Features region, Dense2D f32 n x rtg_feature_columns(params))
// to the executor, which meanwhile prepares and starts the next stage.
void register_gpu_segmentation(VariantRegistry& reg, const SegmentationRegions& ids,
                               const rtg_params& params);

// A stage over one tile: descriptors RGB (Dense3D <y0,x0,0;y1,x1,2>) in,
// Mask / Labels / Features out; body expands to one "segment_features" task
// with whatever variants `reg` holds (kGpuOnly for the product registry).
StageInstance make_segmentation_stage(std::uint64_t stage_id, const BoundingBox& tile,
                                      const SegmentationRegions& ids,
                                      std::shared_ptr<const VariantRegistry> reg);

// Resolves the stage's concrete region tuples (timestamp / version are per
// stage) from the local template by (ns, key, type_tag).
SegmentationRegions resolve_regions(const RegionTemplate& local, const SegmentationRegions& names);

// Output installation helper shared by variants: replaces the metadata-only
// shell worker_prepare created with a typed dense region that keeps the
// shell's io mode and storage binding; zero-filled unless the caller writes
// every cell (zero_fill = false skips the pass).
DataRegion& install_output(RegionTemplate& local, const DataRegionId& id, RegionKind kind,
                           ElementKind elem, const BoundingBox& box, bool zero_fill = true);

}  // namespace rt
