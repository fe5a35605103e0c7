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
// PATS picks (wrm.cpp:246-273), ManagerState FIFO dispatch (dataflow.cpp:73-111),
// RTP1 pack bytes / unpack round trips / decode errors (pack.cpp:33-133),
// RTS1 session files (disk_store.cpp:150-217).
#include <cstdint>
#include <cstring>
#include <cstdio>
#include <fstream>
#include <functional>
#include <memory>
#include <random>
#include <string>
#include <vector>

#ifdef RT_REF
#include "rt/partition.hpp"
#include "rt/bounding_box.hpp"
#include "rt/data_region.hpp"
#include "rt/pack.hpp"
#include "rt/dataflow.hpp"
#include "rt/dms.hpp"
#include "rt/region_template.hpp"
#include "rt/disk_store.hpp"
#include "rt/wrm.hpp"
#else
#include "rt/partition.hpp"
#include "rt/pack.hpp"
#include "rt/session.hpp"
#include "rt/region.hpp"
#include "rt/runtime.hpp"
#endif

using namespace rt;

namespace {

template <typename V>
std::uint64_t fnv(const V& v) {
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
  } catch (const DecodeError&) {
    return "DecodeError";
  } catch (const IoError&) {
    return "IoError";
  } catch (const PartitionError&) {
    return "PartitionError";
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

// A stage's output template as the hot path leaves it: RGB (Dense3D u8),
// Mask (Dense2D u8), Labels (Dense2D i32), Features (Dense2D f32, n x 20).
RegionTemplate stage_template(std::mt19937_64& g, int h, int w, int nobj) {
  RegionTemplate t("seg_tile");
  auto fill = [&](std::size_t n) {
    std::vector<std::uint8_t> v(n);
    for (auto& b : v) b = std::uint8_t(g());
    return v;
  };
  DataRegion rgb(DataRegionId{"wsi", "RGB", "Dense3D", 3, 1}, RegionKind::kDense3D,
                 ElementKind::kU8, BoundingBox({8, 16, 0}, {8 + h - 1, 16 + w - 1, 2}));
  rgb.put_chunk(rgb.bbox(), fill(std::size_t(3 * h * w)));
  rgb.set_storage_binding("disk");
  t.insert_data_region(std::move(rgb));
  // outputs: Dense2D + trailing axis, so all regions share rank 3
  DataRegion mask(DataRegionId{"seg", "Mask", "Dense2D", 3, 2}, RegionKind::kDense2D,
                  ElementKind::kU8, BoundingBox({8, 16, 0}, {8 + h - 1, 16 + w - 1, 0}));
  mask.put_chunk(mask.bbox(), fill(std::size_t(h * w)));
  mask.set_io_mode(IoMode::kOutput);
  mask.set_roi(BoundingBox({9, 17, 0}, {8 + h - 2, 16 + w - 2, 0}));
  t.insert_data_region(std::move(mask));
  DataRegion labels(DataRegionId{"seg", "Labels", "Dense2D", 3, 2}, RegionKind::kDense2D,
                    ElementKind::kI32, BoundingBox({8, 16, 0}, {8 + h - 1, 16 + w - 1, 0}));
  // two row bands as separate chunks
  const int hh = h / 2;
  labels.put_chunk(BoundingBox({8, 16, 0}, {8 + hh - 1, 16 + w - 1, 0}),
                   fill(std::size_t(4 * hh * w)));
  labels.put_chunk(BoundingBox({8 + hh, 16, 0}, {8 + h - 1, 16 + w - 1, 0}),
                   fill(std::size_t(4 * (h - hh) * w)));
  labels.set_io_mode(IoMode::kInputOutput);
  t.insert_data_region(std::move(labels));
  DataRegion feats(DataRegionId{"seg", "Features", "Dense2D", 3, 2}, RegionKind::kDense2D,
                   ElementKind::kF32, BoundingBox({0, 0, 0}, {nobj - 1, 19, 0}));
  std::vector<std::uint8_t> fp(std::size_t(nobj) * 20 * 4);
  for (int k = 0; k < nobj * 20; ++k) {
    const float v = float(int(g() % 100000)) / 7.0f;
    std::memcpy(fp.data() + 4 * k, &v, 4);
  }
  feats.put_chunk(feats.bbox(), std::move(fp));
  feats.set_io_mode(IoMode::kOutput);
  t.insert_data_region(std::move(feats));
  DataRegion lazy(DataRegionId{"wsi", "Next", "Dense2D", 4, 0}, RegionKind::kDense2D,
                  ElementKind::kU16, BoundingBox({0, 0, 0}, {3, 3, 0}));
  lazy.set_lazy(true);
  t.insert_data_region(std::move(lazy));
  return t;
}

void packs() {
  std::mt19937_64 g(1405795800);
  for (int i = 0; i < 6; ++i) {
    RegionTemplate t = stage_template(g, 6 + 2 * i, 5 + 3 * i, 1 + 5 * i);
    for (int pay = 0; pay < 2; ++pay) {
      const std::vector<std::uint8_t> b = pack_template(t, pay != 0);
      const RegionTemplate u = unpack_template(b);
      const std::vector<std::uint8_t> b2 = pack_template(u, pay != 0);
      std::printf("pack %d %d len=%zu h=%016llx rt=%d regions=%zu box=%s\n", i, pay, b.size(),
                  (unsigned long long)fnv(b), int(b2 == b), u.regions().size(),
                  u.bbox().to_string().c_str());
    }
    // corruptions
    const std::vector<std::uint8_t> b = pack_template(t, true);
    auto bad = [&](const char* what, std::vector<std::uint8_t> v) {
      std::printf("unpack %d %s %s\n", i, what, outcome([&] { unpack_template(v); }).c_str());
    };
    bad("truncated", std::vector<std::uint8_t>(b.begin(), b.end() - 1));
    bad("trailing", [&] { auto v = b; v.push_back(0); return v; }());
    bad("magic", [&] { auto v = b; v[0] ^= 1; return v; }());
    bad("flags", [&] { auto v = b; v[4] = 2; return v; }());
    bad("empty", std::vector<std::uint8_t>());
    bad("cut_half", std::vector<std::uint8_t>(b.begin(), b.begin() + b.size() / 2));
  }
  // a rank mix: the region is inserted, the box fold throws
  {
    RegionTemplate t("mix");
    t.insert_data_region(DataRegion(DataRegionId{"a", "x", "raw", 0, 0}, RegionKind::kDense3D,
                                    ElementKind::kU8, BoundingBox({0, 0, 0}, {3, 3, 2})));
    const std::string o = outcome([&] {
      t.insert_data_region(DataRegion(DataRegionId{"a", "y", "raw", 0, 0}, RegionKind::kDense2D,
                                      ElementKind::kU8, BoundingBox({0, 0}, {3, 3})));
    });
    std::printf("mix %s size=%zu box=%s\n", o.c_str(), t.regions().size(),
                t.bbox().to_string().c_str());
  }
  RegionTemplate empty("none");
  const std::vector<std::uint8_t> e = pack_template(empty, true);
  std::printf("pack empty len=%zu h=%016llx\n", e.size(), (unsigned long long)fnv(e));
}

std::vector<std::uint8_t> file_bytes(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  return std::vector<std::uint8_t>((std::istreambuf_iterator<char>(f)),
                                   std::istreambuf_iterator<char>());
}

void write_bytes(const std::string& path, const std::vector<std::uint8_t>& b) {
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  f.write(reinterpret_cast<const char*>(b.data()), std::streamsize(b.size()));
}

std::uint64_t record_hash(const DiskRecord& r) {
  std::vector<std::uint8_t> v(r.payload.begin(), r.payload.end());
  const std::string s = r.id.ns + "|" + r.id.key + "|" + r.id.type_tag + "|" +
                        std::to_string(r.id.timestamp) + "|" + std::to_string(r.id.version) + "|" +
                        std::to_string(int(r.kind)) + "|" + std::to_string(int(r.element_kind)) +
                        "|" + r.box.to_string() + "|" + std::to_string(r.seq);
  v.insert(v.end(), s.begin(), s.end());
  return fnv(v);
}

void sessions(const char* dir) {
  std::mt19937_64 g(7958);
  for (int i = 0; i < 4; ++i) {
    RegionTemplate t = stage_template(g, 4 + 3 * i, 6 + i, 2 + 4 * i);
    std::vector<DiskRecord> recs;
    std::uint64_t seq = 100 * std::uint64_t(i);
    for (const auto& [id, r] : t.regions()) {
      if (!r.materialized()) continue;
      for (const auto& [box, chunk] : r.chunks())
        recs.push_back(DiskRecord{id, r.kind(), r.element_kind(), box, seq++, chunk.payload});
    }
    const std::string path = std::string(dir) + "/s" + std::to_string(i) + ".rts";
    const std::vector<std::uint64_t> offs = write_session_file(path, 7 + std::uint64_t(i), recs);
    const std::vector<std::uint8_t> bytes = file_bytes(path);
    std::string o;
    for (auto x : offs) o += std::to_string(x) + ",";
    std::printf("session %d n=%zu len=%zu h=%016llx offs=%s\n", i, recs.size(), bytes.size(),
                (unsigned long long)fnv(bytes), o.c_str());
    const std::vector<DiskRecord> back = read_session_file(path);
    for (std::size_t k = 0; k < back.size(); ++k)
      std::printf("record %d %zu %016llx at=%016llx\n", i, k,
                  (unsigned long long)record_hash(back[k]),
                  (unsigned long long)record_hash(read_record_at(path, offs[k])));
    auto bad = [&](const char* what, std::vector<std::uint8_t> v) {
      write_bytes(path, v);
      std::printf("session_bad %d %s %s\n", i, what,
                  outcome([&] { read_session_file(path); }).c_str());
    };
    bad("truncated", std::vector<std::uint8_t>(bytes.begin(), bytes.end() - 1));
    bad("magic", [&] { auto v = bytes; v[0] ^= 4; return v; }());
    bad("end_magic", [&] { auto v = bytes; v[v.size() - 1] ^= 4; return v; }());
    bad("footer", [&] { auto v = bytes; v[v.size() - 12] ^= 0x40; return v; }());
    bad("short", std::vector<std::uint8_t>(bytes.begin(), bytes.begin() + 20));
  }
  std::printf("session_missing %s\n",
              outcome([&] { read_session_file(std::string(dir) + "/nope.rts"); }).c_str());
}

// Edge cases of the box / region / dataflow API the hot path relies on.
void edges() {
  const BoundingBox a({0, 0}, {3, 3}), e;
  std::printf("edge contains_empty %d\n", int(a.contains(e)));
  std::printf("edge empty_contains %s\n", outcome([&] { (void)e.contains(a); }).c_str());
  std::printf("edge empty_contains_empty %d\n", int(e.contains(e)));
  const std::int64_t lo[1] = {0}, hi[1] = {0};
  std::printf("edge rank0 %s\n", outcome([&] { std::printf("edge rank0_box %s vol=%lld\n",
      BoundingBox(0, lo, hi).to_string().c_str(), (long long)BoundingBox(0, lo, hi).volume()); }).c_str());
  std::printf("edge rank5 %s\n", outcome([&] { BoundingBox(5, lo, hi); }).c_str());
  std::printf("edge inverted %s\n", outcome([&] { BoundingBox({3}, {1}); }).c_str());
  // DataRegion equality looks at every attribute
  const DataRegionId id{"e", "r", "raw", 1, 2};
  auto make = [&] {
    DataRegion r(id, RegionKind::kDense2D, ElementKind::kU8, a);
    r.put_chunk(a, std::vector<std::uint8_t>(16, 3));
    return r;
  };
  DataRegion base = make();
  std::printf("edge eq_same %d\n", int(base == make()));
  { DataRegion r = make(); r.set_roi(BoundingBox({1, 1}, {2, 2})); std::printf("edge eq_roi %d\n", int(base == r)); }
  { DataRegion r = make(); r.set_io_mode(IoMode::kOutput); std::printf("edge eq_io %d\n", int(base == r)); }
  { DataRegion r = make(); r.set_storage_binding("x"); std::printf("edge eq_binding %d\n", int(base == r)); }
  { DataRegion r = make(); r.set_lazy(true); std::printf("edge eq_lazy %d\n", int(base == r)); }
  { DataRegion r = make(); r.drop_payload(); std::printf("edge eq_dropped %d\n", int(base == r)); }
  // partitions
  for (const auto& [bx, t] : std::vector<std::pair<BoundingBox, std::vector<std::int64_t>>>{
           {BoundingBox({0, 0}, {99999, 99999}), {4096, 4096}},
           {BoundingBox({5, -3, 0}, {17, 9, 2}), {4, 5, 3}},
           {BoundingBox({0}, {9}), {3}},
           {BoundingBox({0, 0}, {9, 9}), {10, 1}}}) {
    std::string o = outcome([&, bx = bx, t = t] {
      const std::vector<BoundingBox> v = partition_regular(bx, std::span<const std::int64_t>(t));
      std::uint64_t h = 1469598103934665603ull;
      for (const auto& b : v)
        for (char c : b.to_string()) h = (h ^ std::uint8_t(c)) * 1099511628211ull;
      std::printf("partition %s n=%zu first=%s last=%s h=%016llx\n", bx.to_string().c_str(), v.size(),
                  v.front().to_string().c_str(), v.back().to_string().c_str(), (unsigned long long)h);
    });
    if (o != "ok") std::printf("partition %s %s\n", bx.to_string().c_str(), o.c_str());
  }
  std::printf("partition empty n=%zu\n", partition_regular(BoundingBox(), {4}).size());
  std::printf("partition bad_rank %s\n", outcome([] { partition_regular(BoundingBox({0, 0}, {3, 3}), {2}); }).c_str());
  std::printf("partition zero %s\n", outcome([] { partition_regular(BoundingBox({0, 0}, {3, 3}), {2, 0}); }).c_str());
  std::printf("partition custom_ok %s\n", outcome([] {
    partition_custom(BoundingBox({0, 0}, {9, 9}), {BoundingBox({0, 0}, {4, 9}), BoundingBox({3, 0}, {9, 9})}); }).c_str());
  std::printf("partition custom_escape %s\n", outcome([] {
    partition_custom(BoundingBox({0, 0}, {9, 9}), {BoundingBox({0, 0}, {10, 9})}); }).c_str());
  std::printf("partition custom_rank %s\n", outcome([] {
    partition_custom(BoundingBox({0, 0}, {9, 9}), {BoundingBox({0}, {3})}); }).c_str());
}

// Lazy inputs (touch_region), 3-D shells, and a growing stage graph.
void lazy_and_growth() {
  StorageRegistry reg;
  auto st = make_store(reg);
  const DataRegionId src{"img", "rgb", "raw", 0, 0}, out{"img", "mask", "label", 0, 0};
  DataRegion in(src, RegionKind::kDense2D, ElementKind::kU8, BoundingBox({0, 0}, {31, 31}));
  std::vector<std::uint8_t> px(32 * 32);
  for (std::size_t i = 0; i < px.size(); ++i) px[i] = std::uint8_t(i * 5 + 3);
  in.put_chunk(in.bbox(), px);
  st->stage_region(in, 0).wait();
  StageInstance s;
  s.stage_id = 4;
  s.stage_kind = "lazy";
  s.region_descriptors = {
      RegionDescriptor{src, BoundingBox({2, 3}, {20, 30}), IoMode::kInput, "store", true},
      RegionDescriptor{out, BoundingBox({2, 3}, {20, 30}), IoMode::kOutput, "store", true}};
  RegionTemplate local = worker_prepare(s, reg);
  const DataRegion* shell = local.get_data_region(src);
  std::printf("lazy shell mat=%d lazy=%d kind=%d out_lazy=%d\n", int(shell->materialized()),
              int(shell->lazy()), int(shell->kind()), int(local.get_data_region(out)->lazy()));
  DataRegion& t1 = touch_region(local, src, reg);
  std::printf("lazy touch mat=%d lazy=%d kind=%d io=%d bind=%s box=%s h=%016llx\n",
              int(t1.materialized()), int(t1.lazy()), int(t1.kind()), int(t1.io_mode()),
              t1.storage_binding().c_str(), t1.bbox().to_string().c_str(),
              (unsigned long long)fnv(t1.chunks().begin()->second.payload));
  DataRegion& t2 = touch_region(local, src, reg);
  std::printf("lazy retouch same=%d\n", int(&t1 == &t2));
  std::printf("lazy touch_output %s\n", outcome([&] { touch_region(local, out, reg); }).c_str());
  std::printf("lazy touch_absent %s\n",
              outcome([&] { touch_region(local, DataRegionId{"no", "pe", "x", 0, 0}, reg); }).c_str());
  // a 3-D query's output shell
  StageInstance s3;
  s3.stage_id = 5;
  s3.stage_kind = "three";
  s3.region_descriptors = {
      RegionDescriptor{out, BoundingBox({0, 0, 0}, {3, 3, 2}), IoMode::kOutput, "store", false}};
  RegionTemplate l3 = worker_prepare(s3, reg);
  const DataRegion* o3 = l3.get_data_region(out);
  std::printf("shell3 kind=%d elem=%d box=%s\n", int(o3->kind()), int(o3->element_kind()),
              o3->bbox().to_string().c_str());
  // dynamic growth, stuck detection, completion log
  ManagerState m;
  auto stage = [](std::uint64_t id, std::set<std::uint64_t> deps) {
    StageInstance x;
    x.stage_id = id;
    x.deps = std::move(deps);
    return x;
  };
  m.add_stage(stage(1, {}));
  m.add_stage(stage(3, {2}));  // depends on a stage not added yet
  std::printf("grow stuck0=%d eligible=%zu\n", int(m.stuck()), m.eligible_ids().size());
  const auto d1 = m.dispatch(7);
  std::printf("grow dispatch=%llu worker=%d stuck=%d\n", (unsigned long long)*d1,
              *m.assigned_worker(1), int(m.stuck()));
  std::vector<StageInstance> kids;
  kids.push_back(stage(2, {1}));
  kids.push_back(stage(4, {9}));
  const auto now = m.stage_complete(1, std::move(kids));
  std::string ns;
  for (auto x : now) ns += std::to_string(x) + ",";
  std::printf("grow spawned -> %s size=%zu done=%zu\n", ns.c_str(), m.size(), m.done_count());
  while (auto d = m.dispatch(1)) {
    const auto nn = m.stage_complete(*d);
    std::printf("grow done %llu -> %zu\n", (unsigned long long)*d, nn.size());
  }
  std::string log;
  for (auto x : m.completion_log()) log += std::to_string(x) + ",";
  std::printf("grow log=%s all=%d stuck=%d unassigned=%d\n", log.c_str(), int(m.all_done()),
              int(m.stuck()), int(!m.assigned_worker(4).has_value()));
  std::printf("grow unknown %s\n", outcome([&] { m.assigned_worker(99); }).c_str());
  std::printf("grow undispatched %s\n", outcome([&] { m.stage_complete(4); }).c_str());
  std::printf("grow dup_spawn %s\n", outcome([&] {
    ManagerState q;
    q.add_stage(stage(1, {}));
    q.dispatch(0);
    std::vector<StageInstance> k;
    k.push_back(stage(1, {}));
    q.stage_complete(1, std::move(k));
  }).c_str());
}

}  // namespace

int main(int argc, char** argv) {
  boxes();
  copies();
  regions();
  dataflow();
  scheduler();
  packs();
  sessions(argc > 1 ? argv[1] : "/tmp");
  edges();
  lazy_and_growth();
  return 0;
}
