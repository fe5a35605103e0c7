// Behaviour probe of the Region Templates host API, compiled twice:
//   -DRT_REF : against the REFERENCE library built from /root/reference by
//              oracle/build_ref.sh (outputs only in oracle/_ref/);
//   default  : against this repo's host layer (paper_1405_7958_b200/host).
// Both binaries print one line per observation; tests/test_host_ref.py
// requires identical output.  TEST INFRASTRUCTURE ONLY.
//
// Covered semantics (reference anchors): BoundingBox algebra
// (bounding_box.cpp), copy_box_overlap (data_region.cpp:270-295), put_chunk
// validation (data_region.cpp:171-192), RegionTemplate bbox fold / remove
// (region_template.cpp:19-74), worker_prepare / stage_finalize
// (dataflow.cpp:113-176) incl. sub-box reads (storage.cpp:21-54), WRM FCFS /
// PATS picks (wrm.cpp:246-273), ManagerState FIFO dispatch (dataflow.cpp:73-111).
#include <cstdint>
#include <cstdio>
#include <functional>
#include <memory>
#include <random>
#include <string>
#include <vector>

#ifdef RT_REF
#include "rt/bounding_box.hpp"
#include "rt/data_region.hpp"
#include "rt/dataflow.hpp"
#include "rt/dms.hpp"
#include "rt/region_template.hpp"
#include "rt/wrm.hpp"
#else
#include "rt/region.hpp"
#include "rt/runtime.hpp"
#endif

using namespace rt;

namespace {

std::uint64_t fnv(const std::vector<std::uint8_t>& v) {
  std::uint64_t h = 1469598103934665603ull;
  for (auto b : v) h = (h ^ b) * 1099511628211ull;
  return h;
}

BoundingBox rbox(std::mt19937_64& g, int dims, int span) {
  std::int64_t lo[4], hi[4];
  for (int a = 0; a < dims; ++a) {
    lo[a] = std::int64_t(g() % span) - span / 2;
    hi[a] = lo[a] + std::int64_t(g() % (span / 2 + 1));
  }
  return BoundingBox(dims, lo, hi);
}

std::string s_opt(const std::optional<BoundingBox>& b) { return b ? b->to_string() : "none"; }

template <class F>
std::string outcome(F&& f) {
  try {
    f();
    return "ok";
  } catch (const DimensionError&) {
    return "DimensionError";
  } catch (const NotFoundError&) {
    return "NotFoundError";
  } catch (const DuplicateRegionError&) {
    return "DuplicateRegionError";
  } catch (const ProtocolError&) {
    return "ProtocolError";
  } catch (const ConfigError&) {
    return "ConfigError";
  } catch (const Error&) {
    return "Error";
  }
}

void boxes() {
  std::mt19937_64 g(1405);
  for (int i = 0; i < 200; ++i) {
    const int d = 1 + int(g() % 3);
    BoundingBox a = rbox(g, d, 20), b = rbox(g, d, 20);
    std::printf("box %s %s vol=%lld u=%s i=%s c=%d lt=%d\n", a.to_string().c_str(),
                b.to_string().c_str(), (long long)a.volume(), a.unioned(b).to_string().c_str(),
                s_opt(a.intersected(b)).c_str(), int(a.contains(b)), int(a < b));
  }
  std::printf("empty %s vol=%lld\n", BoundingBox().to_string().c_str(),
              (long long)BoundingBox().volume());
}

void copies() {
  std::mt19937_64 g(7958);
  for (int i = 0; i < 200; ++i) {
    const int d = 2 + int(g() % 2);
    const std::size_t es = (g() % 2) ? 4 : 1;
    BoundingBox s = rbox(g, d, 16), t = rbox(g, d, 16);
    std::vector<std::uint8_t> src(std::size_t(s.volume()) * es), dst(std::size_t(t.volume()) * es, 0);
    for (auto& v : src) v = std::uint8_t(g());
    copy_box_overlap(dst, t, src, s, es);
    std::printf("copy %d %zu %016llx\n", i, es, (unsigned long long)fnv(dst));
  }
}

void regions() {
  RegionTemplate t("probe");
  std::mt19937_64 g(42);
  std::vector<DataRegionId> ids;
  for (int i = 0; i < 30; ++i) {
    DataRegionId id{"p", "r" + std::to_string(g() % 5), "raw", std::int64_t(g() % 3), 0};
    BoundingBox b = rbox(g, 2, 40);
    const std::string o = outcome([&] {
      t.insert_data_region(DataRegion(id, RegionKind::kDense2D, ElementKind::kU8, b));
    });
    if (o == "ok") ids.push_back(id);
    std::printf("insert %s %s -> %s bbox=%s size=%zu\n", id.name().c_str(), b.to_string().c_str(),
                o.c_str(), t.bbox().to_string().c_str(), t.size());
    if (i % 4 == 3 && !ids.empty()) {
      const DataRegionId victim = ids[std::size_t(g() % ids.size())];
      const bool removed = t.remove_data_region(victim);
      std::printf("remove %s -> %d bbox=%s\n", victim.name().c_str(), int(removed),
                  t.bbox().to_string().c_str());
    }
  }
  DataRegion r(DataRegionId{"p", "x", "raw", 0, 0}, RegionKind::kDense2D, ElementKind::kI32,
               BoundingBox({0, 0}, {3, 4}));
  std::printf("put short %s\n", outcome([&] { r.put_chunk(BoundingBox({0, 0}, {3, 4}), std::vector<std::uint8_t>(20)); }).c_str());
  std::printf("put escape %s\n", outcome([&] { r.put_chunk(BoundingBox({0, 0}, {4, 4}), std::vector<std::uint8_t>(100)); }).c_str());
  std::printf("put ok %s bytes=%llu\n",
              outcome([&] { r.put_chunk(BoundingBox({1, 1}, {2, 2}), std::vector<std::uint8_t>(16)); }).c_str(),
              (unsigned long long)r.payload_bytes());
  std::printf("rank %s\n", outcome([] {
                DataRegion(DataRegionId{}, RegionKind::kDense2D, ElementKind::kU8, BoundingBox({0}, {3}));
              }).c_str());
  std::printf("rank3 %s\n", outcome([] {
                DataRegion(DataRegionId{}, RegionKind::kDense2D, ElementKind::kU8,
                           BoundingBox({0, 0, 0}, {3, 3, 2}));
              }).c_str());
}

std::shared_ptr<StorageBackend> make_store(StorageRegistry& reg) {
#ifdef RT_REF
  DmsConfig cfg;
  cfg.hilbert = sfc::HilbertParams{2, 4};
  cfg.grid_origin = {0, 0};
  cfg.cell_extent = {8, 8};
  cfg.occupied = {BoundingBox({0, 0}, {7, 7})};
  cfg.shard_count = 2;
  auto s = std::make_shared<DmsStore>("store", cfg, reg.sequence());
#else
  auto s = std::make_shared<MemoryStore>("store");
#endif
  reg.add(s);
  return s;
}

void dataflow() {
  StorageRegistry reg;
  auto st = make_store(reg);
  const DataRegionId rgb{"img", "rgb", "raw", 0, 0}, mask{"img", "mask", "label", 0, 0};
  DataRegion in(rgb, RegionKind::kDense2D, ElementKind::kU8, BoundingBox({0, 0}, {31, 31}));
  std::vector<std::uint8_t> px(32 * 32);
  for (std::size_t i = 0; i < px.size(); ++i) px[i] = std::uint8_t(i * 7 + 1);
  in.put_chunk(in.bbox(), px);
  st->stage_region(in, 0).wait();
  StageInstance s;
  s.stage_id = 9;
  s.stage_kind = "seg";
  s.region_descriptors = {
      RegionDescriptor{rgb, BoundingBox({4, 6}, {19, 27}), IoMode::kInput, "store", false},
      RegionDescriptor{mask, BoundingBox({4, 6}, {19, 27}), IoMode::kOutput, "store", false}};
  RegionTemplate local = worker_prepare(s, reg);
  const DataRegion* a = local.get_data_region(rgb);
  const DataRegion* b = local.get_data_region(mask);
  std::printf("prepare name=%s bbox=%s in=%d/%s/%016llx out=%d/%s kind=%d elem=%d\n",
              local.name().c_str(), local.bbox().to_string().c_str(), int(a->materialized()),
              a->bbox().to_string().c_str(),
              (unsigned long long)fnv(a->chunks().begin()->second.payload), int(b->materialized()),
              b->bbox().to_string().c_str(), int(b->kind()), int(b->element_kind()));
  local.get_data_region(mask)->put_chunk(BoundingBox({4, 6}, {19, 27}),
                                         std::vector<std::uint8_t>(16 * 22, 5));
  const auto comps = stage_finalize(local, s, reg, 0);
  std::printf("finalize completions=%zu left=%zu\n", comps.size(), local.size());
  DataRegion back = st->read_region(mask, BoundingBox({10, 10}, {12, 20}));
  std::printf("readback %s %016llx\n", back.bbox().to_string().c_str(),
              (unsigned long long)fnv(back.chunks().begin()->second.payload));
  std::printf("read outside %s\n",
              outcome([&] { st->read_region(mask, BoundingBox({0, 0}, {5, 5})); }).c_str());
  s.region_descriptors[0].id.key = "absent";
  std::printf("prepare missing %s\n", outcome([&] { worker_prepare(s, reg); }).c_str());
}

void scheduler() {
  for (int pats = 0; pats < 2; ++pats) {
#ifdef RT_REF
    WrmState w(WrmOptions{pats ? SchedulerKind::kPats : SchedulerKind::kFcfs, false, 0.12});
#else
    WrmState w(pats ? SchedulerKind::kPats : SchedulerKind::kFcfs);
#endif
    std::mt19937_64 g(100 + pats);
    std::vector<TaskNode> ts;
    for (int i = 1; i <= 24; ++i) {
      TaskNode t;
      t.task_id = std::uint64_t(i);
      const int v = int(g() % 3);
      t.variants = v == 0 ? TaskVariants::kCpuOnly : v == 1 ? TaskVariants::kGpuOnly : TaskVariants::kBoth;
      if (v == 2) t.speedup_estimate = double(1 + g() % 20);
      if (i > 4 && g() % 3 == 0) t.deps = {std::uint64_t(1 + g() % (i - 1))};
      ts.push_back(t);
    }
    w.submit(ts);
    std::string seq;
    for (int step = 0; step < 200 && !w.all_done(); ++step) {
      const DeviceKind d = (step % 3 == 0) ? DeviceKind::kGpu : DeviceKind::kCpu;
      auto id = w.next(d);
      if (!id) {
        id = w.next(d == DeviceKind::kGpu ? DeviceKind::kCpu : DeviceKind::kGpu);
        if (!id) break;
      }
      seq += std::to_string(*id) + (d == DeviceKind::kGpu ? "g " : "c ");
      w.complete(*id);
    }
    std::printf("wrm %s %s\n", pats ? "pats" : "fcfs", seq.c_str());
  }
  ManagerState m;
  for (int i = 1; i <= 6; ++i) {
    StageInstance s;
    s.stage_id = std::uint64_t(i);
    if (i % 2 == 0) s.deps = {std::uint64_t(i - 1)};
    m.add_stage(s);
  }
  std::string seq;
  while (auto id = m.dispatch(0)) seq += std::to_string(*id) + " ";
  std::printf("manager %s\n", seq.c_str());
  std::printf("manager complete1 -> %zu\n", m.stage_complete(1).size());
  std::printf("manager double %s\n", outcome([&] { m.stage_complete(1); }).c_str());
}

}  // namespace

int main() {
  boxes();
  copies();
  regions();
  dataflow();
  scheduler();
  return 0;
}
