// B200 variant of the segmentation + feature stage (see rt/rtg_stage.hpp).
#include "rt/rtg_stage.hpp"

#include <cstring>
#include <string>

namespace rt {

void throw_rtg_error(int status) {
  const std::string msg = std::string("rtg: ") + rtg_last_error();
  switch (status) {
    case RTG_ERR_INVALID_ARG: throw ConfigError(msg);
    case RTG_ERR_DIMENSION: throw DimensionError(msg);
    case RTG_ERR_RANGE:
    case RTG_ERR_OVERFLOW: throw RangeError(msg);
    case RTG_ERR_NOT_FOUND: throw NotFoundError(msg);
    case RTG_ERR_OUT_OF_MEMORY:
    case RTG_ERR_DEVICE:
    case RTG_ERR_NO_DEVICE: throw DeviceError(msg);
    default: throw Error(msg);
  }
}

GpuDevice::GpuDevice(int device, std::int64_t max_h, std::int64_t max_w,
                     std::int32_t max_objects)
    : device_(device), max_objects_(max_objects) {
  rtg_check(rtg_ctx_create(device, max_h, max_w, max_objects, &ctx_));
}

GpuDevice::~GpuDevice() {
  if (ctx_) rtg_ctx_destroy(ctx_);  // waits for the context's streams
  for (float* f : all_) rtg_host_free(f);
}

std::shared_ptr<float> GpuDevice::acquire_staging() {
  float* f = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu_);
    if (!free_.empty()) {
      f = free_.back();
      free_.pop_back();
    }
  }
  if (!f) {
    void* p = nullptr;
    rtg_check(rtg_host_alloc(sizeof(float) * std::size_t(max_objects_) * RTG_MAX_FEATURE_COLUMNS, &p));
    f = static_cast<float*>(p);
    std::lock_guard<std::mutex> lk(mu_);
    all_.push_back(f);
  }
  return std::shared_ptr<float>(f, [this](float* q) {
    std::lock_guard<std::mutex> lk(mu_);
    free_.push_back(q);
  });
}

std::size_t GpuDevice::staging_buffers() const {
  std::lock_guard<std::mutex> lk(mu_);
  return all_.size();
}

namespace {
void* pinned_alloc(std::size_t bytes) {
  void* p = nullptr;
  return rtg_host_alloc(bytes, &p) == RTG_OK ? p : nullptr;
}
void pinned_free(void* p) { rtg_host_free(p); }
}  // namespace

void use_pinned_payloads(std::size_t min_bytes, std::size_t pool_bytes, std::size_t live_bytes) {
  set_payload_allocator(pinned_alloc, pinned_free, min_bytes, pool_bytes, live_bytes);
}

void use_pageable_payloads() { set_payload_allocator(nullptr, nullptr, 0, 0); }

DataRegion& install_output(RegionTemplate& local, const DataRegionId& id, RegionKind kind,
                           ElementKind elem, const BoundingBox& box, bool zero_fill) {
  IoMode mode = IoMode::kOutput;
  std::string binding;
  if (const DataRegion* shell = local.get_data_region(id)) {
    mode = shell->io_mode();
    binding = shell->storage_binding();
    local.remove_data_region(id);
  }
  DataRegion r(id, kind, elem, box);
  const std::size_t n = std::size_t(box.volume()) * element_size(elem);
  r.put_chunk(box, zero_fill ? Bytes(n, 0) : Bytes(n));
  r.set_io_mode(mode);
  r.set_storage_binding(binding);
  return local.insert_data_region(std::move(r));
}

SegmentationRegions resolve_regions(const RegionTemplate& local, const SegmentationRegions& names) {
  SegmentationRegions out = names;
  auto pick = [&](DataRegionId& id) {
    // the stage's own instance of this (ns, key, type) — timestamps and
    // versions are per stage, so look the tuple up in the local template
    if (const DataRegion* r = local.get_newest(id.ns, id.key, id.type_tag)) id = r->id();
  };
  pick(out.rgb);
  pick(out.mask);
  pick(out.labels);
  pick(out.features);
  return out;
}

namespace {

// Where the RGB bytes of the tile come from: a store view (no host copy) or
// the local template's payload.
struct TileSource {
  const std::uint8_t* data = nullptr;
  std::int64_t pitch = 0;
  std::shared_ptr<const void> keep;
};

TileSource tile_source(WorkerContext& wc, RegionTemplate& local, const DataRegionId& id) {
  DataRegion* rgb = local.get_data_region(id);
  if (!rgb) throw NotFoundError("stage input " + id.to_string() + " missing");
  const BoundingBox b3 = rgb->bbox();
  if (b3.dims() != 3 || b3.extent(2) != 3)
    throw DimensionError("RGB tile must be <y0,x0,0;y1,x1,2>, got " + b3.to_string());
  if (rgb->lazy() && !rgb->materialized()) {
    if (!wc.storage) throw ProtocolError("lazy RGB input outside an executor with storage");
    std::optional<PayloadView> v = wc.storage->at(rgb->storage_binding()).view_region(id, b3);
    if (v && v->elem == ElementKind::kU8)
      return TileSource{v->data, v->row_pitch, std::move(v->keep)};
    rgb = &touch_region(local, id, *wc.storage);
  }
  if (rgb->element_kind() != ElementKind::kU8)
    throw DimensionError("RGB tile must be u8");
  const Chunk* c = rgb->find_chunk(b3);
  if (!c) throw NotFoundError("RGB tile has no chunk covering " + b3.to_string());
  return TileSource{c->payload.data(), 3 * b3.extent(1), nullptr};
}

void gpu_segment_features(const SegmentationRegions& names, const rtg_params& params) {
  WorkerContext& wc = worker_context();
  if (!wc.local) throw ProtocolError("segment_features ran outside a worker context");
  if (!wc.gpu) throw DeviceError("segment_features GPU variant scheduled without a GpuDevice");
  RegionTemplate& local = *wc.local;
  const SegmentationRegions ids = resolve_regions(local, names);
  TileSource src = tile_source(wc, local, ids.rgb);  // validates the RGB region
  const BoundingBox b3 = local.get_data_region(ids.rgb)->bbox();
  const std::int64_t h = b3.extent(0), w = b3.extent(1);
  // Outputs are Dense2D with the trailing axis the reference allows
  // (data_region.cpp:152-157), so every region of the stage template has rank
  // 3 like the RGB tile (a rank mix throws in RegionTemplate's box fold).
  const BoundingBox b2({b3.lo(0), b3.lo(1), 0}, {b3.hi(0), b3.hi(1), 0});
  DataRegion& mask = install_output(local, ids.mask, RegionKind::kDense2D, ElementKind::kU8, b2, false);
  DataRegion& labels =
      install_output(local, ids.labels, RegionKind::kDense2D, ElementKind::kI32, b2, false);
  GpuDevice* dev = wc.gpu;
  std::int32_t cols = 0;
  rtg_check(rtg_feature_columns(&params, &cols));
  std::shared_ptr<float> rows = dev->acquire_staging();
  std::uint64_t ticket = 0;
  rtg_check(rtg_process_tile_async(
      dev->ctx(), src.data, h, w, src.pitch, &params, mask.find_chunk(b2)->payload.data(),
      reinterpret_cast<std::int32_t*>(labels.find_chunk(b2)->payload.data()), nullptr, rows.get(),
      dev->max_objects(), &ticket));
  // the device owns the tile's buffers until the ticket is waited; `src.keep`
  // holds a viewed store piece alive for the upload
  defer_completion([dev, ticket, rows, cols, keep = std::move(src.keep), fid = ids.features] {
    std::int32_t n = 0;
    rtg_check(rtg_ticket_wait(dev->ctx(), ticket, &n));
    if (n <= 0) return;
    RegionTemplate& tpl = *worker_context().local;
    const BoundingBox fb({0, 0, 0}, {n - 1, cols - 1, 0});
    DataRegion& f = install_output(tpl, fid, RegionKind::kDense2D, ElementKind::kF32, fb, false);
    std::memcpy(f.find_chunk(fb)->payload.data(), rows.get(),
                sizeof(float) * std::size_t(n) * std::size_t(cols));
  });
}

}  // namespace

void register_gpu_segmentation(VariantRegistry& reg, const SegmentationRegions& ids,
                               const rtg_params& params) {
  reg.register_variant(kSegmentFeaturesTask, DeviceKind::kGpu,
                       [ids, params] { gpu_segment_features(ids, params); });
}

StageInstance make_segmentation_stage(std::uint64_t stage_id, const BoundingBox& tile,
                                      const SegmentationRegions& ids,
                                      std::shared_ptr<const VariantRegistry> reg) {
  if (tile.dims() != 2) throw DimensionError("tile box must be 2-D <y0,x0;y1,x1>");
  const BoundingBox rgb_box({tile.lo(0), tile.lo(1), 0}, {tile.hi(0), tile.hi(1), 2});
  const BoundingBox out_box({tile.lo(0), tile.lo(1), 0}, {tile.hi(0), tile.hi(1), 0});
  StageInstance s;
  s.stage_id = stage_id;
  s.stage_kind = "segmentation";
  s.region_descriptors = {
      RegionDescriptor{ids.rgb, rgb_box, IoMode::kInput, ids.binding, ids.lazy_rgb},
      RegionDescriptor{ids.mask, out_box, IoMode::kOutput, ids.binding, false},
      RegionDescriptor{ids.labels, out_box, IoMode::kOutput, ids.binding, false},
      RegionDescriptor{ids.features, BoundingBox({0, 0, 0}, {0, RTG_NUM_FEATURES - 1, 0}),
                       IoMode::kOutput, ids.binding, false},
  };
  s.body = [reg, stage_id] {
    return std::vector<TaskNode>{reg->make_task(kSegmentFeaturesTask, stage_id, stage_id)};
  };
  return s;
}

}  // namespace rt
