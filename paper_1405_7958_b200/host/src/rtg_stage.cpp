// B200 variant of the segmentation + feature stage (see rt/rtg_stage.hpp).
#include "rt/rtg_stage.hpp"

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
  void* f = nullptr;
  const int st = rtg_host_alloc(sizeof(float) * std::size_t(max_objects) * RTG_NUM_FEATURES, &f);
  if (st != RTG_OK) {
    rtg_ctx_destroy(ctx_);
    throw_rtg_error(st);
  }
  features_ = static_cast<float*>(f);
}

GpuDevice::~GpuDevice() {
  if (features_) rtg_host_free(features_);
  if (ctx_) rtg_ctx_destroy(ctx_);
}

namespace {
void* pinned_alloc(std::size_t bytes) {
  void* p = nullptr;
  return rtg_host_alloc(bytes, &p) == RTG_OK ? p : nullptr;
}
void pinned_free(void* p) { rtg_host_free(p); }
}  // namespace

void use_pinned_payloads(std::size_t min_bytes, std::size_t pool_bytes) {
  set_payload_allocator(pinned_alloc, pinned_free, min_bytes, pool_bytes);
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

void gpu_segment_features(const SegmentationRegions& names, const rtg_params& params) {
  WorkerContext& wc = worker_context();
  if (!wc.local) throw ProtocolError("segment_features ran outside a worker context");
  if (!wc.gpu) throw DeviceError("segment_features GPU variant scheduled without a GpuDevice");
  RegionTemplate& local = *wc.local;
  const SegmentationRegions ids = resolve_regions(local, names);
  const DataRegion* rgb = local.get_data_region(ids.rgb);
  if (!rgb) throw NotFoundError("stage input " + ids.rgb.to_string() + " missing");
  const BoundingBox& b3 = rgb->bbox();
  if (b3.dims() != 3 || b3.extent(2) != 3 || rgb->element_kind() != ElementKind::kU8)
    throw DimensionError("RGB tile must be Dense3D u8 <y0,x0,0;y1,x1,2>, got " + b3.to_string());
  const Chunk* c = rgb->find_chunk(b3);
  if (!c) throw NotFoundError("RGB tile has no chunk covering " + b3.to_string());
  const std::int64_t h = b3.extent(0), w = b3.extent(1);
  // Outputs are Dense2D with the trailing axis the reference allows
  // (data_region.cpp:152-157), so every region of the stage template has rank
  // 3 like the RGB tile (a rank mix throws in RegionTemplate's box fold).
  const BoundingBox b2({b3.lo(0), b3.lo(1), 0}, {b3.hi(0), b3.hi(1), 0});

  DataRegion& mask = install_output(local, ids.mask, RegionKind::kDense2D, ElementKind::kU8, b2, false);
  DataRegion& labels =
      install_output(local, ids.labels, RegionKind::kDense2D, ElementKind::kI32, b2, false);
  const std::int32_t cap = wc.gpu->max_objects();
  float* feats = wc.gpu->feature_staging();
  std::int32_t n = 0;
  rtg_check(rtg_process_tile(wc.gpu->ctx(), c->payload.data(), h, w, 3 * w, &params,
                             mask.find_chunk(b2)->payload.data(),
                             reinterpret_cast<std::int32_t*>(labels.find_chunk(b2)->payload.data()),
                             nullptr, feats, cap, &n));
  if (n > 0) {
    const BoundingBox fb({0, 0, 0}, {n - 1, RTG_NUM_FEATURES - 1, 0});
    DataRegion& f = install_output(local, ids.features, RegionKind::kDense2D, ElementKind::kF32, fb, false);
    std::memcpy(f.find_chunk(fb)->payload.data(), feats,
                sizeof(float) * std::size_t(n) * RTG_NUM_FEATURES);
  }
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
      RegionDescriptor{ids.rgb, rgb_box, IoMode::kInput, ids.binding, false},
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
