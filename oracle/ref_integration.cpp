// Drop-in proof against the REAL reference runtime (TEST INFRASTRUCTURE).
//
// Compiled by oracle/build_ref.sh against the reference's own headers and
// librt_ref.a (built from /root/reference/proj/src, outputs only under
// oracle/_ref/) and linked with this repo's librtg.so.  It runs the
// INTEGRATION.md §2 task body through the reference's ManagerState,
// WrmState, worker_prepare, a 3-D DmsStore and stage_finalize, in the
// run_pipeline pattern of tests/test_acceptance.cpp:546-613, and checks every
// tile's Mask / Labels read back from the reference store against the oracle
// (rtg_oracle.c, compiled in as the checker) bit-exactly and its Features
// within rtol 1e-5.
//
//   ref_integration            GPU body (librtg.so rtg_process_tile)
//   ref_integration --cpu      oracle body (harness self-check, no GPU)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "rt/dataflow.hpp"
#include "rt/dms.hpp"
#include "rt/region_template.hpp"
#include "rt/storage.hpp"
#include "rt/wrm.hpp"
#include "rtg.h"
#include "rtg_oracle.h"

extern "C" int orc_synth_tile_host(uint64_t, int64_t, int64_t, int64_t, int64_t, uint8_t*);

using namespace rt;

namespace {

constexpr int64_t H = 1024, W = 1536, T = 512;
constexpr int32_t kRows = 1 << 15;

[[noreturn]] void die(const std::string& m) {
  std::printf("FAIL %s\n", m.c_str());
  std::exit(1);
}

// Replaces the metadata-only U8 shell worker_prepare made for `id`
// (dataflow.cpp:128) with a typed dense region carrying `bytes`.
void install(RegionTemplate& local, const DataRegionId& id, ElementKind elem,
             const BoundingBox& box, std::vector<std::uint8_t> bytes) {
  IoMode mode = IoMode::kOutput;
  std::string binding = "store";
  if (const DataRegion* shell = local.get_data_region(id)) {
    mode = shell->io_mode();
    binding = shell->storage_binding();
    local.remove_data_region(id);
  }
  DataRegion r(id, RegionKind::kDense2D, elem, box);
  r.put_chunk(box, std::move(bytes));
  r.set_io_mode(mode);
  r.set_storage_binding(binding);
  local.insert_data_region(std::move(r));
}

struct TileIds {
  DataRegionId rgb, mask, labels, features;
};

// The INTEGRATION.md §2 body: RGB from the local template -> rtg_process_tile
// (or the oracle) -> typed Mask / Labels / Features regions.
void segment_body(RegionTemplate& local, const TileIds& ids, rtg_ctx* ctx, bool cpu) {
  const DataRegion* rgb = local.get_data_region(ids.rgb);
  if (!rgb) die("RGB missing from the local template");
  const BoundingBox b = rgb->bbox();
  const int64_t h = b.extent(0), w = b.extent(1);
  std::vector<std::uint8_t> mask(std::size_t(h * w));
  std::vector<std::uint8_t> labels(std::size_t(h * w) * 4);
  std::vector<float> feats(std::size_t(kRows) * RTG_NUM_FEATURES);
  rtg_params p;
  rtg_params_default(&p);
  int32_t n = 0;
  const std::uint8_t* px = rgb->find_chunk(b)->payload.data();
  if (cpu) {
    n = orc_process_tile(px, h, w, 3 * w, &p, mask.data(), reinterpret_cast<int32_t*>(labels.data()),
                         feats.data(), kRows, nullptr);
  } else if (rtg_process_tile(ctx, px, h, w, 3 * w, &p, mask.data(),
                              reinterpret_cast<int32_t*>(labels.data()), nullptr, feats.data(),
                              kRows, &n) != RTG_OK) {
    throw Error(rtg_last_error());
  }
  const BoundingBox b2({b.lo(0), b.lo(1), 0}, {b.hi(0), b.hi(1), 0});
  install(local, ids.mask, ElementKind::kU8, b2, std::move(mask));
  install(local, ids.labels, ElementKind::kI32, b2, std::move(labels));
  if (n > 0) {
    std::vector<std::uint8_t> fb(std::size_t(n) * RTG_NUM_FEATURES * 4);
    std::memcpy(fb.data(), feats.data(), fb.size());
    install(local, ids.features, ElementKind::kF32,
            BoundingBox({0, 0, 0}, {n - 1, RTG_NUM_FEATURES - 1, 0}), std::move(fb));
  }
}

}  // namespace

int main(int argc, char** argv) {
  const bool cpu = argc > 1 && std::strcmp(argv[1], "--cpu") == 0;
  rtg_ctx* ctx = nullptr;
  if (!cpu && rtg_ctx_create(0, T, T, kRows, &ctx) != RTG_OK)
    die(std::string("rtg_ctx_create: ") + rtg_last_error());

  // a 3-D DMS (the RGB tile is Dense3D; SURVEY §7.3 hard part 7)
  StorageRegistry registry;
  DmsConfig cfg;
  cfg.hilbert = sfc::HilbertParams{3, 2};
  cfg.grid_origin = {0, 0, 0};
  cfg.cell_extent = {T, T, 3};
  cfg.occupied = {BoundingBox({0, 0, 0}, {H / T - 1, W / T - 1, 0})};
  cfg.shard_count = 2;
  auto dms = std::make_shared<DmsStore>("store", cfg, registry.sequence());
  registry.add(dms);

  const DataRegionId slide_id{"img", "RGB", "raw", 0, 0};
  std::vector<std::uint8_t> px(std::size_t(H * W * 3));
  if (orc_synth_tile_host(1405795800ULL, 0, 0, H, W, px.data()) != 0) die("synth");
  {
    DataRegion slide(slide_id, RegionKind::kDense3D, ElementKind::kU8,
                     BoundingBox({0, 0, 0}, {H - 1, W - 1, 2}));
    slide.put_chunk(slide.bbox(), px);
    dms->stage_region(slide, 0).wait();
  }

  ManagerState manager;
  WrmState wrm(WrmOptions{SchedulerKind::kPats, false, 0.12});
  std::vector<TileIds> tiles;
  std::vector<BoundingBox> boxes;
  std::uint64_t sid = 1;
  for (int64_t y = 0; y < H; y += T) {
    for (int64_t x = 0; x < W; x += T, ++sid) {
      TileIds ids{slide_id, {"img", "Mask", "label", int64_t(sid), 0},
                  {"img", "Labels", "label", int64_t(sid), 0},
                  {"img", "Features", "table", int64_t(sid), 0}};
      const BoundingBox rgb_box({y, x, 0}, {y + T - 1, x + T - 1, 2});
      const BoundingBox out_box({y, x, 0}, {y + T - 1, x + T - 1, 0});
      StageInstance stage;
      stage.stage_id = sid;
      stage.stage_kind = "segmentation";
      stage.region_descriptors = {
          RegionDescriptor{ids.rgb, rgb_box, IoMode::kInput, "store", false},
          RegionDescriptor{ids.mask, out_box, IoMode::kOutput, "store", false},
          RegionDescriptor{ids.labels, out_box, IoMode::kOutput, "store", false},
          RegionDescriptor{ids.features, BoundingBox({0, 0, 0}, {0, RTG_NUM_FEATURES - 1, 0}),
                           IoMode::kOutput, "store", false}};
      stage.body = [sid] {
        TaskNode node;
        node.task_id = sid;
        node.stage_id = sid;
        node.variants = TaskVariants::kGpuOnly;
        return std::vector<TaskNode>{node};
      };
      manager.add_stage(std::move(stage));
      tiles.push_back(ids);
      boxes.push_back(out_box);
    }
  }

  // run_pipeline (test_acceptance.cpp:546-613), GPU slot instead of CPU
  std::size_t ran = 0;
  while (!manager.all_done()) {
    const auto s = manager.dispatch(0);
    if (!s) die("pipeline wedged");
    const StageInstance& stage = manager.stage(*s);
    RegionTemplate local = worker_prepare(stage, registry);
    const TileIds& ids = tiles[std::size_t(*s - 1)];
    std::vector<TaskNode> tasks = stage.body();
    for (auto& t : tasks) t.body = [&local, &ids, ctx, cpu] { segment_body(local, ids, ctx, cpu); };
    wrm.submit(tasks);
    while (const auto tid = wrm.next(DeviceKind::kGpu)) {
      for (const auto& t : tasks)
        if (t.task_id == *tid && t.body) t.body();
      wrm.complete(*tid);
      ++ran;
    }
    for (auto& c : stage_finalize(local, stage, registry, 0)) c.wait();
    manager.stage_complete(*s);
  }

  // read back through the reference store; compare with the oracle
  rtg_params p;
  rtg_params_default(&p);
  int bad = 0;
  for (std::size_t k = 0; k < tiles.size(); ++k) {
    const BoundingBox& ob = boxes[k];
    const int64_t y0 = ob.lo(0), x0 = ob.lo(1);
    std::vector<std::uint8_t> tile(std::size_t(T * T * 3));
    for (int64_t r = 0; r < T; ++r)
      std::memcpy(tile.data() + r * T * 3, px.data() + ((y0 + r) * W + x0) * 3, std::size_t(T * 3));
    std::vector<std::uint8_t> rm(std::size_t(T * T));
    std::vector<int32_t> rl(std::size_t(T * T));
    std::vector<float> rf(std::size_t(kRows) * RTG_NUM_FEATURES);
    const int32_t rn = orc_process_tile(tile.data(), T, T, 3 * T, &p, rm.data(), rl.data(),
                                        rf.data(), kRows, nullptr);
    const DataRegion m = dms->read_region(tiles[k].mask, ob);
    const DataRegion l = dms->read_region(tiles[k].labels, ob);
    const BoundingBox fb({0, 0, 0}, {rn - 1, RTG_NUM_FEATURES - 1, 0});
    const DataRegion f = dms->read_region(tiles[k].features, fb);
    const auto& mp = m.chunks().begin()->second.payload;
    const auto& lp = l.chunks().begin()->second.payload;
    const auto& fp = f.chunks().begin()->second.payload;
    const bool mask_ok = l.element_kind() == ElementKind::kI32 &&
                         std::memcmp(mp.data(), rm.data(), rm.size()) == 0;
    const bool lab_ok = std::memcmp(lp.data(), rl.data(), rl.size() * 4) == 0;
    bool feat_ok = fp.size() == std::size_t(rn) * RTG_NUM_FEATURES * 4;
    const float* fv = reinterpret_cast<const float*>(fp.data());
    for (std::size_t i = 0; feat_ok && i < std::size_t(rn) * RTG_NUM_FEATURES; ++i)
      feat_ok = std::fabs(fv[i] - rf[i]) <= 1e-6f + 1e-5f * std::fabs(rf[i]);
    std::printf("tile %zu %s objects=%d mask=%d labels=%d features=%d\n", k,
                ob.to_string().c_str(), rn, int(mask_ok), int(lab_ok), int(feat_ok));
    bad += !(mask_ok && lab_ok && feat_ok);
  }
  if (ctx) rtg_ctx_destroy(ctx);
  if (bad || ran != tiles.size()) die(std::to_string(bad) + " tile(s) differ");
  std::printf("OK %zu stages through the reference ManagerState / WrmState / worker_prepare / "
              "DmsStore / stage_finalize (%s body)\n",
              ran, cpu ? "oracle" : "B200 librtg.so");
  return 0;
}
