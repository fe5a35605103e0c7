// Framework-free checks of the C++ Region Templates host layer, in the style
// of the reference's acceptance gate (tests/test_acceptance.cpp: one PASS/FAIL
// line per check).  `test_host` runs the CPU checks; `test_host --gpu` adds the
// stage executed through StageInstance -> WRM -> TaskNode::body -> C-ABI on a
// B200, checked bit-exactly against the oracle (linked here as the checker).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include "../../oracle/rtg_oracle.h"
#include "rt/pack.hpp"
#include "rt/region.hpp"
#include "rt/session.hpp"
#include "rt/rtg_stage.hpp"
#include "rt/runtime.hpp"

using namespace rt;

namespace {

int g_fail = 0;

void check(const std::string& name, const std::function<void()>& fn) {
  try {
    fn();
    std::printf("PASS %s\n", name.c_str());
  } catch (const std::exception& e) {
    ++g_fail;
    std::printf("FAIL %s: %s\n", name.c_str(), e.what());
  }
}

void require(bool ok, const std::string& what) {
  if (!ok) throw std::runtime_error(what);
}

template <typename E>
void require_throws(const std::function<void()>& fn, const std::string& what) {
  try {
    fn();
  } catch (const E&) {
    return;
  }
  throw std::runtime_error("expected exception: " + what);
}

BoundingBox box2(std::int64_t a, std::int64_t b, std::int64_t c, std::int64_t d) {
  return BoundingBox({a, b}, {c, d});
}

DataRegion u8_region(const std::string& key, const BoundingBox& b, std::int64_t ts = 0,
                     std::int64_t ver = 0) {
  return DataRegion(DataRegionId{"t", key, "raw", ts, ver}, RegionKind::kDense2D,
                    ElementKind::kU8, b);
}

// ---------------------------------------------------------------- containers

void containers() {
  check("copy_box_overlap KAT (reference test_region.cpp:277-285 restated)", [] {
    std::vector<std::uint8_t> src(25), dst(9, 0);
    for (int i = 0; i < 25; ++i) src[i] = std::uint8_t(i + 1);
    copy_box_overlap(dst, box2(3, 3, 5, 5), src, box2(0, 0, 4, 4), 1);
    require(dst == std::vector<std::uint8_t>{19, 20, 0, 24, 25, 0, 0, 0, 0}, "overlap bytes");
  });
  check("copy_box_overlap / fill_box_overlap match a per-cell walk (200 seeded 1-3-D trials)", [] {
    std::mt19937 rng(7958);
    auto rnd = [&](int lo, int hi) { return int(rng() % unsigned(hi - lo + 1)) + lo; };
    for (int trial = 0; trial < 200; ++trial) {
      const int d = rnd(1, 3);
      std::vector<std::int64_t> l1(d), h1(d), l2(d), h2(d);
      for (int a = 0; a < d; ++a) {
        const bool full = a > 0 && rnd(0, 1);  // trailing axes often identical
        l1[a] = rnd(0, 4); h1[a] = l1[a] + rnd(0, 5);
        l2[a] = full ? l1[a] : rnd(0, 4); h2[a] = full ? h1[a] : l2[a] + rnd(0, 5);
      }
      const BoundingBox db(d, l1.data(), h1.data()), sb(d, l2.data(), h2.data());
      const std::size_t es = std::size_t(rnd(1, 3));
      std::vector<std::uint8_t> src(std::size_t(sb.volume()) * es), dst(std::size_t(db.volume()) * es, 0);
      for (auto& v : src) v = std::uint8_t(rng());
      std::vector<std::uint8_t> want = dst, seen(std::size_t(db.volume()), 0), seen_want = seen;
      for (std::int64_t i = 0; i < db.volume(); ++i) {  // naive: decode every dst cell
        std::vector<std::int64_t> c(d);
        std::int64_t r = i;
        for (int a = d - 1; a >= 0; --a) { c[a] = db.lo(a) + r % db.extent(a); r /= db.extent(a); }
        bool in = true;
        std::int64_t o = 0;
        for (int a = 0; a < d; ++a) {
          in = in && c[a] >= sb.lo(a) && c[a] <= sb.hi(a);
          o = o * sb.extent(a) + (c[a] - sb.lo(a));
        }
        if (!in) continue;
        std::memcpy(want.data() + std::size_t(i) * es, src.data() + std::size_t(o) * es, es);
        seen_want[std::size_t(i)] = 1;
      }
      copy_box_overlap(dst, db, src, sb, es);
      fill_box_overlap(seen, db, sb, 1);
      require(dst == want && seen == seen_want, "trial " + std::to_string(trial));
    }
  });
  check("stage_region_consume moves payloads into the store, region ends unmaterialised", [] {
    MemoryStore st("s");
    const DataRegionId id{"t", "c", "raw", 0, 0};
    DataRegion a(id, RegionKind::kDense2D, ElementKind::kU8, box2(0, 0, 3, 3));
    std::vector<std::uint8_t> v(16);
    for (int i = 0; i < 16; ++i) v[std::size_t(i)] = std::uint8_t(i);
    a.put_chunk(a.bbox(), v);
    const DataRegion copy = a;
    st.stage_region_consume(a, 0).wait();
    require(!a.materialized() && a.chunks().empty(), "region consumed");
    require(st.read_region(id, box2(0, 0, 3, 3)) == copy, "store holds the bytes");
  });
  check("MemoryStore read: a newer partial piece wins over an older exact piece", [] {
    MemoryStore st("s");
    const DataRegionId id{"t", "p", "raw", 0, 0};
    DataRegion a(id, RegionKind::kDense2D, ElementKind::kU8, box2(0, 0, 3, 3));
    a.put_chunk(a.bbox(), std::vector<std::uint8_t>(16, 1));
    DataRegion b(id, RegionKind::kDense2D, ElementKind::kU8, box2(2, 2, 5, 5));
    b.put_chunk(b.bbox(), std::vector<std::uint8_t>(16, 2));
    st.stage_region(a, 0).wait();
    st.stage_region(b, 0).wait();
    const DataRegion r = st.read_region(id, box2(0, 0, 3, 3));
    const Bytes& v = r.chunks().begin()->second.payload;
    require(v[0] == 1 && v[3 * 4 + 3] == 2 && v[2 * 4 + 1] == 1, "last writer wins");
  });
  check("put_chunk validates box and dense payload length", [] {
    DataRegion r = u8_region("a", box2(0, 0, 9, 9));
    require_throws<DimensionError>([&] { r.put_chunk(box2(0, 0, 9, 9), std::vector<std::uint8_t>(99)); },
                                   "short payload");
    require_throws<DimensionError>([&] { r.put_chunk(box2(5, 5, 10, 10), std::vector<std::uint8_t>(36)); },
                                   "escaping chunk");
    r.put_chunk(box2(0, 0, 9, 9), std::vector<std::uint8_t>(100, 3));
    require(r.materialized() && r.payload_bytes() == 100, "materialised");
    DataRegion i32(DataRegionId{"t", "l", "label", 0, 0}, RegionKind::kDense2D, ElementKind::kI32,
                   box2(0, 0, 3, 3));
    require_throws<DimensionError>([&] { i32.put_chunk(box2(0, 0, 3, 3), std::vector<std::uint8_t>(16)); },
                                   "i32 payload needs 4 bytes per element");
  });
  check("template bbox = fold of region boxes (50 seeded trials)", [] {
    std::mt19937_64 rng(20261018);
    for (int trial = 0; trial < 50; ++trial) {
      RegionTemplate t("p");
      std::int64_t a0 = INT64_MAX, a1 = INT64_MAX, b0 = INT64_MIN, b1 = INT64_MIN;
      const int n = 1 + int(rng() % 8);
      for (int i = 0; i < n; ++i) {
        const std::int64_t l0 = std::int64_t(rng() % 100) - 50, l1 = std::int64_t(rng() % 100) - 50;
        const std::int64_t h0 = l0 + std::int64_t(rng() % 40), h1 = l1 + std::int64_t(rng() % 40);
        t.insert_data_region(u8_region("r", box2(l0, l1, h0, h1), i));
        a0 = std::min(a0, l0); a1 = std::min(a1, l1); b0 = std::max(b0, h0); b1 = std::max(b1, h1);
      }
      require(t.bbox() == box2(a0, a1, b0, b1), "fold");
    }
  });
  check("duplicate tuple insert throws, bumped version does not", [] {
    RegionTemplate t("s");
    t.insert_data_region(u8_region("a", box2(0, 0, 9, 9)));
    require_throws<DuplicateRegionError>([&] { t.insert_data_region(u8_region("a", box2(0, 0, 9, 9))); },
                                         "duplicate");
    t.insert_data_region(u8_region("a", box2(0, 0, 9, 9), 0, 1));
    require(t.get_newest("t", "a", "raw")->id().version == 1, "newest");
  });
  check("DenseDataRegion2D typed view", [] {
    DataRegion r = DenseDataRegion2D<std::int32_t>::create(DataRegionId{"t", "l", "label", 0, 0},
                                                           box2(10, 20, 13, 24));
    DenseDataRegion2D<std::int32_t> v(r);
    require(v.height() == 4 && v.width() == 5, "extent");
    v.at(3, 4) = 77;
    require(reinterpret_cast<const std::int32_t*>(r.find_chunk(r.bbox())->payload.data())[19] == 77,
            "row-major, last axis contiguous");
    require_throws<DimensionError>([&] { DenseDataRegion2D<std::uint8_t> bad(r); }, "kind check");
  });
  check("template box fold rejects a rank mix but keeps the region (region_template.cpp:19-29)", [] {
    RegionTemplate t("mix");
    DataRegion rgb(DataRegionId{"img", "RGB", "raw", 0, 0}, RegionKind::kDense3D, ElementKind::kU8,
                   BoundingBox({0, 0, 0}, {7, 7, 2}));
    t.insert_data_region(std::move(rgb));
    require_throws<DimensionError>([&] {
      t.insert_data_region(DataRegion(DataRegionId{"img", "m", "raw", 0, 0}, RegionKind::kDense2D,
                                      ElementKind::kU8, box2(0, 0, 7, 7)));
    }, "rank mismatch");
    require(t.size() == 2 && t.bbox() == BoundingBox({0, 0, 0}, {7, 7, 2}), "inserted, box kept");
    // the same output as Dense2D + trailing axis folds fine
    t.insert_data_region(DataRegion(DataRegionId{"img", "m", "raw", 1, 0}, RegionKind::kDense2D,
                                    ElementKind::kU8, BoundingBox({0, 0, 0}, {9, 7, 0})));
    require(t.bbox() == BoundingBox({0, 0, 0}, {9, 7, 2}), "rank-3 fold");
  });
  check("rank check: Dense3D RGB box and Dense2D+time", [] {
    DataRegion rgb(DataRegionId{"img", "RGB", "raw", 0, 0}, RegionKind::kDense3D, ElementKind::kU8,
                   BoundingBox({0, 0, 0}, {7, 7, 2}));
    rgb.put_chunk(rgb.bbox(), std::vector<std::uint8_t>(8 * 8 * 3));
    require_throws<DimensionError>([] {
      DataRegion(DataRegionId{}, RegionKind::kDense2D, ElementKind::kU8, BoundingBox({0}, {3}));
    }, "1-D box for Dense2D");
  });
}

// ---------------------------------------------------------------- scheduler / dataflow

TaskNode task(std::uint64_t id, TaskVariants v, std::optional<double> s = std::nullopt) {
  TaskNode t;
  t.task_id = id;
  t.variants = v;
  t.speedup_estimate = s;
  return t;
}

void scheduling() {
  check("payload allocator hook: size threshold, recycling by size, per-block free function", [] {
    static int allocs_a = 0, frees_a = 0, frees_b = 0;
    struct H {
      static void* alloc_a(std::size_t n) { ++allocs_a; return std::malloc(n); }
      static void free_a(void* p) { ++frees_a; std::free(p); }
      static void* alloc_b(std::size_t n) { return std::malloc(n); }
      static void free_b(void* p) { ++frees_b; std::free(p); }
    };
    set_payload_allocator(H::alloc_a, H::free_a, 1000, 1 << 20);
    {
      Bytes small(999, 1), big(4096, 2);
      require(!payload_is_hooked(small.data()) && payload_is_hooked(big.data()), "threshold");
      require(reinterpret_cast<std::uintptr_t>(small.data()) % 64 == 0, "heap blocks 64-byte aligned");
      const std::uint8_t* first = big.data();
      big = Bytes();
      Bytes again(4096, 3);  // recycled block, contents value-initialised
      require(again.data() == first && again[4095] == 3 && allocs_a == 1, "recycled by size");
      DataRegion r(DataRegionId{"t", "p", "raw", 0, 0}, RegionKind::kDense2D, ElementKind::kU8,
                   box2(0, 0, 63, 63));
      r.put_chunk(r.bbox(), std::move(again));
      require(payload_is_hooked(r.find_chunk(r.bbox())->payload.data()), "chunk keeps the block");
      set_payload_allocator(H::alloc_b, H::free_b, 1000, 0);  // pool of hook a released
      Bytes b2(8192, 4);
      require(payload_is_hooked(b2.data()), "hook b");
    }  // r's block goes back through free_a, b2 through free_b (pool cap 0)
    require(frees_a == 1 && frees_b == 1, "each block freed by the hook that made it");
    set_payload_allocator(nullptr, nullptr, 0, 0);
    Bytes plain(1 << 16, 0);
    require(!payload_is_hooked(plain.data()), "hook removed");
  });
  check("WRM FCFS takes the first compatible ready task", [] {
    WrmState w(SchedulerKind::kFcfs);
    w.submit({task(1, TaskVariants::kCpuOnly), task(2, TaskVariants::kGpuOnly),
              task(3, TaskVariants::kBoth, 4.0)});
    require(*w.next(DeviceKind::kGpu) == 2, "gpu");
    require(*w.next(DeviceKind::kCpu) == 1, "cpu");
    require(*w.next(DeviceKind::kCpu) == 3, "cpu2");
    require(!w.next(DeviceKind::kGpu), "empty");
  });
  check("WRM PATS: GPU takes max speedup, CPU min (reference wrm.cpp:246-273)", [] {
    WrmState w(SchedulerKind::kPats);
    w.submit({task(1, TaskVariants::kBoth, 2.0), task(2, TaskVariants::kBoth, 9.0),
              task(3, TaskVariants::kBoth, 5.0)});
    require(*w.next(DeviceKind::kGpu) == 2, "gpu max");
    require(*w.next(DeviceKind::kCpu) == 1, "cpu min");
  });
  check("WRM rejects dual-variant tasks without a speedup", [] {
    WrmState w;
    require_throws<ConfigError>([&] { w.submit({task(1, TaskVariants::kBoth)}); }, "speedup");
  });
  check("WRM dependencies gate readiness", [] {
    WrmState w;
    TaskNode b = task(2, TaskVariants::kCpuOnly);
    b.deps = {1};
    w.submit({task(1, TaskVariants::kCpuOnly), b});
    require(*w.next(DeviceKind::kCpu) == 1 && !w.next(DeviceKind::kCpu), "blocked");
    require(w.complete(1) == std::vector<std::uint64_t>{2}, "released");
  });
  check("VariantRegistry derives variants from registered implementations", [] {
    VariantRegistry r;
    r.register_variant("g", DeviceKind::kGpu, [] {});
    r.register_variant("b", DeviceKind::kGpu, [] {});
    r.register_variant("b", DeviceKind::kCpu, [] {});
    r.set_speedup("b", 12.0);
    require(r.make_task("g", 1, 1).variants == TaskVariants::kGpuOnly, "gpu only");
    const TaskNode t = r.make_task("b", 2, 1);
    require(t.variants == TaskVariants::kBoth && *t.speedup_estimate == 12.0, "both");
    require_throws<NotFoundError>([&] { r.make_task("x", 3, 1); }, "unknown");
  });
  check("worker_prepare materialises inputs, outputs are shells; finalize stages outputs", [] {
    StorageRegistry reg;
    auto st = std::make_shared<MemoryStore>("store");
    reg.add(st);
    const DataRegionId rgb{"img", "rgb", "raw", 0, 0}, mask{"img", "mask", "label", 0, 0};
    DataRegion in(rgb, RegionKind::kDense2D, ElementKind::kU8, box2(0, 0, 15, 15));
    in.put_chunk(box2(0, 0, 15, 15), std::vector<std::uint8_t>(256, 9));
    st->stage_region(in, 0).wait();
    StageInstance s;
    s.stage_id = 5;
    s.stage_kind = "seg";
    s.region_descriptors = {RegionDescriptor{rgb, box2(0, 0, 15, 15), IoMode::kInput, "store"},
                            RegionDescriptor{mask, box2(0, 0, 15, 15), IoMode::kOutput, "store"}};
    RegionTemplate local = worker_prepare(s, reg);
    require(local.get_data_region(rgb)->materialized(), "input read");
    require(!local.get_data_region(mask)->materialized(), "output shell");
    local.get_data_region(mask)->put_chunk(box2(0, 0, 15, 15), std::vector<std::uint8_t>(256, 1));
    stage_finalize(local, s, reg, 0);
    require(!local.get_data_region(rgb), "input dropped");
    require(st->read_region(mask, box2(4, 4, 7, 7)).payload_bytes() == 16, "staged sub-box read");
    s.region_descriptors[0].id.key = "absent";
    require_throws<NotFoundError>([&] { worker_prepare(s, reg); }, "missing input");
  });
  check("ManagerState dispatches FIFO among dependency-satisfied stages", [] {
    ManagerState m;
    StageInstance a, b, c;
    a.stage_id = 1;
    b.stage_id = 2;
    b.deps = {1};
    c.stage_id = 3;
    m.add_stage(a);
    m.add_stage(b);
    m.add_stage(c);
    require(*m.dispatch(0) == 1 && *m.dispatch(0) == 3 && !m.dispatch(0), "fifo + gating");
    require(m.stage_complete(1) == std::vector<std::uint64_t>{2}, "release");
  });
  check("MemoryStore views: every row of a viewed sub-box equals read_region's bytes", [] {
    MemoryStore st("s");
    const DataRegionId id{"img", "RGB", "raw", 0, 0};
    DataRegion slide(id, RegionKind::kDense3D, ElementKind::kU8, BoundingBox({0, 0, 0}, {63, 95, 2}));
    std::vector<std::uint8_t> px(64 * 96 * 3);
    for (std::size_t i = 0; i < px.size(); ++i) px[i] = std::uint8_t(i * 31 + 7);
    slide.put_chunk(slide.bbox(), px);
    st.stage_region(slide, 0).wait();
    const BoundingBox q({8, 16, 0}, {39, 79, 2});
    const auto v = st.view_region(id, q);
    require(v && v->row_pitch == 96 * 3, "view with the slide's row pitch");
    const DataRegion r = st.read_region(id, q);
    const Bytes& want = r.chunks().begin()->second.payload;
    for (std::int64_t y = 0; y < q.extent(0); ++y)
      require(std::memcmp(v->data + y * v->row_pitch, want.data() + y * 64 * 3, 64 * 3) == 0,
              "row " + std::to_string(y));
    require(!st.view_region(id, BoundingBox({8, 16, 1}, {39, 79, 2})), "partial channel axis: no view");
    DataRegion patch(id, RegionKind::kDense3D, ElementKind::kU8, BoundingBox({30, 30, 0}, {33, 33, 2}));
    patch.put_chunk(patch.bbox(), std::vector<std::uint8_t>(48, 9));
    st.stage_region(patch, 0).wait();
    require(!st.view_region(id, q), "a newer partial piece hides the old one: no view");
  });
  check("MemoryStore views of 2-D / 1-D pieces; defer_completion runs in place on CPU workers", [] {
    MemoryStore st("s");
    const DataRegionId id{"t", "lab", "label", 0, 0};
    DataRegion lab(id, RegionKind::kDense2D, ElementKind::kI32, box2(10, 20, 49, 99));
    std::vector<std::uint8_t> px(40 * 80 * 4);
    for (std::size_t i = 0; i < px.size(); ++i) px[i] = std::uint8_t(i * 13 + 5);
    lab.put_chunk(lab.bbox(), px);
    st.stage_region(lab, 0).wait();
    const BoundingBox q = box2(15, 30, 24, 59);
    const auto v = st.view_region(id, q);
    require(v && v->row_pitch == 80 * 4 && v->elem == ElementKind::kI32, "2-D view");
    const DataRegion r = st.read_region(id, q);
    for (std::int64_t y = 0; y < 10; ++y)
      require(std::memcmp(v->data + y * v->row_pitch,
                          r.chunks().begin()->second.payload.data() + y * 30 * 4, 30 * 4) == 0,
              "2-D row " + std::to_string(y));
    const DataRegionId id1{"t", "vec", "raw", 0, 0};
    DataRegion one(id1, RegionKind::kDense1D, ElementKind::kU16, BoundingBox({0}, {99}));
    std::vector<std::uint8_t> b1(200);
    for (std::size_t i = 0; i < b1.size(); ++i) b1[i] = std::uint8_t(i);
    one.put_chunk(one.bbox(), b1);
    st.stage_region(one, 0).wait();
    const auto v1 = st.view_region(id1, BoundingBox({40}, {59}));
    require(v1 && v1->data[0] == 80 && v1->data[39] == 119, "1-D view");
    require(!st.view_region(DataRegionId{"t", "none", "x", 0, 0}, q), "no data: no view");
    int ran = 0;
    defer_completion([&] { ++ran; });
    require(ran == 1, "no pipelining executor: the completion runs at once");
  });
  check("executor: spawned stages run, lazy inputs are touched, a wedged graph throws", [] {
    StorageRegistry reg;
    auto st = std::make_shared<MemoryStore>("store");
    reg.add(st);
    const DataRegionId src{"t", "src", "raw", 0, 0};
    DataRegion in(src, RegionKind::kDense2D, ElementKind::kU8, box2(0, 0, 7, 7));
    in.put_chunk(in.bbox(), std::vector<std::uint8_t>(64, 5));
    st->stage_region(in, 0).wait();
    auto seen = std::make_shared<std::vector<int>>();
    auto mu = std::make_shared<std::mutex>();
    std::function<StageInstance(std::uint64_t, int)> make = [&](std::uint64_t id, int depth) {
      StageInstance s;
      s.stage_id = id;
      s.stage_kind = "grow";
      s.region_descriptors = {RegionDescriptor{src, box2(0, 0, 7, 7), IoMode::kInput, "store", true}};
      s.body = [id, depth, seen, mu, &make, src] {
        TaskNode t;
        t.task_id = 1;
        t.variants = TaskVariants::kCpuOnly;
        t.body = [id, depth, seen, mu, &make, src] {
          WorkerContext& wc = worker_context();
          const DataRegion& r = touch_region(*wc.local, src, *wc.storage);
          require(r.materialized() && r.chunks().begin()->second.payload[63] == 5, "touched");
          {
            std::lock_guard<std::mutex> lk(*mu);
            seen->push_back(int(id));
          }
          if (depth < 3) {
            spawn_stage(make(id * 10 + 1, depth + 1));
            spawn_stage(make(id * 10 + 2, depth + 1));
          }
        };
        return std::vector<TaskNode>{t};
      };
      return s;
    };
    ManagerState m;
    m.add_stage(make(1, 0));
    ExecutorConfig cfg;
    cfg.cpu_workers = 3;
    const ExecutorStats s = run_stages(m, reg, cfg);
    require(s.stages == 15 && seen->size() == 15 && m.all_done(), "1 + 2 + 4 + 8 stages");
    ManagerState w;
    StageInstance a;
    a.stage_id = 1;
    a.deps = {7};  // never added
    w.add_stage(a);
    require_throws<ProtocolError>([&] { run_stages(w, reg, cfg); }, "wedge detected");
  });
}

// ---------------------------------------------------------------- the GPU stage

extern "C" int rtg_synth_tile_host(uint64_t, int64_t, int64_t, int64_t, int64_t, uint8_t*);

// The oracle as the CPU variant of "segment_features" (test-only drop-in twin).
void cpu_segment_features(const SegmentationRegions& names, const rtg_params& p) {
  WorkerContext& wc = worker_context();
  RegionTemplate& local = *wc.local;
  const SegmentationRegions ids = resolve_regions(local, names);
  // a lazy input is read on first touch (reference dataflow.cpp:137-154)
  const DataRegion* rgb = &touch_region(local, ids.rgb, *wc.storage);
  const BoundingBox& b3 = rgb->bbox();
  const std::int64_t h = b3.extent(0), w = b3.extent(1);
  const BoundingBox b2({b3.lo(0), b3.lo(1), 0}, {b3.hi(0), b3.hi(1), 0});
  DataRegion& mask = install_output(local, ids.mask, RegionKind::kDense2D, ElementKind::kU8, b2);
  DataRegion& lab = install_output(local, ids.labels, RegionKind::kDense2D, ElementKind::kI32, b2);
  std::vector<float> f(std::size_t(1 << 16) * RTG_NUM_FEATURES);
  const std::int32_t n = orc_process_tile(
      rgb->find_chunk(b3)->payload.data(), h, w, 3 * w, &p, mask.find_chunk(b2)->payload.data(),
      reinterpret_cast<std::int32_t*>(lab.find_chunk(b2)->payload.data()), f.data(), 1 << 16,
      nullptr);
  if (n > 0) {
    const BoundingBox fb({0, 0, 0}, {n - 1, RTG_NUM_FEATURES - 1, 0});
    DataRegion& fr = install_output(local, ids.features, RegionKind::kDense2D, ElementKind::kF32, fb);
    std::memcpy(fr.find_chunk(fb)->payload.data(), f.data(), sizeof(float) * n * RTG_NUM_FEATURES);
  }
}

// Slide of 2x2 tiles staged as one Dense3D region; one stage per tile.
struct Run {
  std::vector<DataRegion> masks, labels, feats;
};

double g_last_run_ms = 0;  // run_stages wall time of the last run_slide

struct SlideOpts {
  bool use_gpu = true, register_cpu = false;
  int cpu_workers = 0;
  std::int64_t H = 1024, W = 1024, T = 512;
  int gpu_inflight = 3;
  bool lazy_rgb = true;
  const Bytes* pixels = nullptr;  // pre-synthesised slide (H x W x 3), else generated
  GpuDevice* gpu = nullptr;       // a warm device to reuse, else a fresh one
};

// A synthetic slide staged as one Dense3D region, one segmentation stage per
// tile, run through run_stages; returns every tile's staged outputs.
Run run_slide(const SlideOpts& o, ExecutorStats* stats) {
  const std::int64_t H = o.H, W = o.W, T = o.T;
  rtg_params p;
  rtg_check(rtg_params_default(&p));
  StorageRegistry reg;
  auto st = std::make_shared<MemoryStore>("store");
  reg.add(st);
  SegmentationRegions ids;
  ids.lazy_rgb = o.lazy_rgb;
  {
    DataRegion slide(ids.rgb, RegionKind::kDense3D, ElementKind::kU8, BoundingBox({0, 0, 0}, {H - 1, W - 1, 2}));
    Bytes px(std::size_t(H * W * 3));
    if (o.pixels)
      std::memcpy(px.data(), o.pixels->data(), px.size());
    else
      rtg_check(rtg_synth_tile_host(1405795800ULL, 0, 0, H, W, px.data()));
    slide.put_chunk(slide.bbox(), std::move(px));
    st->stage_region_consume(slide, 0).wait();
  }

  auto vr = std::make_shared<VariantRegistry>();
  if (o.use_gpu) register_gpu_segmentation(*vr, ids, p);
  if (o.register_cpu) {
    vr->register_variant(kSegmentFeaturesTask, DeviceKind::kCpu, [ids, p] { cpu_segment_features(ids, p); });
    vr->set_speedup(kSegmentFeaturesTask, 100.0);
  }
  ManagerState m;
  std::uint64_t sid = 1;
  std::vector<SegmentationRegions> tile_ids;
  for (std::int64_t y = 0; y < H; y += T) {
    for (std::int64_t x = 0; x < W; x += T) {
      SegmentationRegions t = ids;
      t.mask.timestamp = t.labels.timestamp = t.features.timestamp = std::int64_t(sid);
      tile_ids.push_back(t);
      m.add_stage(make_segmentation_stage(sid++, box2(y, x, y + T - 1, x + T - 1), t, vr));
    }
  }
  std::unique_ptr<GpuDevice> gpu;
  ExecutorConfig cfg;
  cfg.cpu_workers = o.cpu_workers;
  cfg.gpu_inflight = o.gpu_inflight;
  if (o.use_gpu) {
    if (!o.gpu) gpu = std::make_unique<GpuDevice>(0, T, T, T >= 2048 ? 1 << 16 : 1 << 14);
    cfg.gpus = {o.gpu ? o.gpu : gpu.get()};
  }
  const auto t0 = std::chrono::steady_clock::now();
  *stats = run_stages(m, reg, cfg);
  g_last_run_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  Run out;
  std::int64_t k = 0;
  for (std::int64_t y = 0; y < H; y += T) {
    for (std::int64_t x = 0; x < W; x += T, ++k) {
      const auto& t = tile_ids[std::size_t(k)];
      // stage outputs carry a trailing singleton axis (rank 3 like the RGB tile)
      const BoundingBox tb({y, x, 0}, {y + T - 1, x + T - 1, 0});
      out.masks.push_back(st->read_region(t.mask, tb));
      out.labels.push_back(st->read_region(t.labels, tb));
      out.feats.push_back(
          st->read_region(t.features, BoundingBox({0, 0, 0}, {0, RTG_NUM_FEATURES - 1, 0})));
    }
  }
  return out;
}

bool same_outputs(const Run& a, const Run& b) {
  if (a.masks.size() != b.masks.size()) return false;
  for (std::size_t i = 0; i < a.masks.size(); ++i) {
    if (!(a.masks[i].chunks().begin()->second.payload == b.masks[i].chunks().begin()->second.payload) ||
        !(a.labels[i].chunks().begin()->second.payload == b.labels[i].chunks().begin()->second.payload))
      return false;
  }
  return true;
}

void gpu_stage() {
  check("GPU variant through StageInstance/WRM/TaskNode matches the CPU variant bit-exactly", [] {
    ExecutorStats sg, sc;
    const Run g = run_slide(SlideOpts{}, &sg);
    require(sg.stages == 4 && sg.gpu_tasks == 4 && sg.cpu_tasks == 0, "all tasks on the GPU");
    SlideOpts co;
    co.use_gpu = false;
    co.register_cpu = true;
    const Run c = run_slide(co, &sc);
    require(sc.cpu_tasks == 4, "all tasks on the CPU variant");
    require(same_outputs(g, c), "masks / labels equal");
    for (std::size_t i = 0; i < 4; ++i) {
      require(g.labels[i].element_kind() == ElementKind::kI32, "labels are I32");
      require(g.feats[i].payload_bytes() == c.feats[i].payload_bytes(), "feature table sizes");
    }
  });
  check("pipelined executor (3 stages in flight, async bodies) = one stage at a time = eager reads", [] {
    SlideOpts o;
    o.H = 1536;
    o.W = 2048;
    o.T = 512;
    ExecutorStats s3, s1, se;
    const Run a = run_slide(o, &s3);
    require(s3.stages == 12 && s3.deferred_tasks == 12, "every GPU completion deferred");
    require(s3.max_inflight >= 2, "stages overlapped (max in flight " + std::to_string(s3.max_inflight) + ")");
    o.gpu_inflight = 1;
    const Run b = run_slide(o, &s1);
    require(s1.deferred_tasks == 0 && s1.max_inflight == 0, "depth 1 runs in place");
    o.gpu_inflight = 3;
    o.lazy_rgb = false;  // worker_prepare copies the tile out of the slide
    const Run c = run_slide(o, &se);
    require(same_outputs(a, b) && same_outputs(a, c), "identical outputs");
  });
  check("GPU stage outputs persist as RTP1 packs and RTS1 sessions and read back intact", [] {
    ExecutorStats st;
    const Run g = run_slide(SlideOpts{}, &st);
    RegionTemplate t("seg_out");
    t.insert_data_region(g.masks[0]);
    t.insert_data_region(g.labels[0]);
    t.insert_data_region(g.feats[0]);
    const std::vector<std::uint8_t> b = pack_template(t, true);
    const RegionTemplate u = unpack_template(b);
    require(pack_template(u, true) == b, "pack round trip");
    const std::string path = "test_host_session.rts";
    const std::vector<DiskRecord> recs = template_records(t, 1);
    const std::vector<std::uint64_t> offs = write_session_file(path, 1, recs);
    const std::vector<DiskRecord> back = read_session_file(path);
    require(back.size() == recs.size() && offs.size() == recs.size(), "record count");
    for (std::size_t k = 0; k < recs.size(); ++k)
      require(back[k].payload == recs[k].payload && back[k].box == recs[k].box, "record");
    std::remove(path.c_str());
  });
  check("cooperative CPU+GPU workers: both pull tiles, outputs bit-identical", [] {
    ExecutorStats sg, sm;
    SlideOpts o;
    o.W = 1536;
    o.T = 256;
    const Run g = run_slide(o, &sg);
    o.register_cpu = true;
    o.cpu_workers = 3;
    const Run m = run_slide(o, &sm);
    require(sm.stages == 24 && sm.gpu_tasks + sm.cpu_tasks == 24, "all 24 tiles");
    require(sm.gpu_tasks > 0 && sm.cpu_tasks > 0, "both device kinds used");
    require(same_outputs(g, m), "masks / labels equal");
  });
  check("pinned Chunk payloads (f1): stage reads/writes pinned chunks, outputs bit-identical", [] {
    ExecutorStats sp, sq;
    const Run q = run_slide(SlideOpts{}, &sq);
    use_pinned_payloads(std::size_t(64) << 10, std::size_t(256) << 20);
    {
      const Run p = run_slide(SlideOpts{}, &sp);
      require(sp.gpu_tasks == 4, "all tasks on the GPU");
      for (std::size_t i = 0; i < 4; ++i) {
        const Bytes& pm = p.masks[i].chunks().begin()->second.payload;
        const Bytes& pl = p.labels[i].chunks().begin()->second.payload;
        require(payload_is_hooked(pm.data()) && payload_is_hooked(pl.data()), "outputs pinned");
      }
      require(same_outputs(p, q), "masks / labels equal");
    }
    use_pageable_payloads();
  });
  check("pinned budget exceeded: outputs fall back to heap payloads, results unchanged", [] {
    ExecutorStats sp, sq;
    const Run q = run_slide(SlideOpts{}, &sq);
    // room for the slide and one tile's outputs only
    use_pinned_payloads(std::size_t(64) << 10, 0, std::size_t(4) << 20);
    {
      const Run p = run_slide(SlideOpts{}, &sp);
      const PayloadStats ps = payload_stats();
      require(ps.fallbacks > 0, "some payloads fell back");
      int hooked = 0;
      for (const auto& r : p.labels) hooked += payload_is_hooked(r.chunks().begin()->second.payload.data());
      require(hooked < 4, "not every output pinned");
      require(same_outputs(p, q), "masks / labels equal");
    }
    use_pageable_payloads();
  });
  check("PATS sends a dual-variant task to the GPU worker", [] {
    ExecutorStats s;
    SlideOpts o;
    o.register_cpu = true;
    run_slide(o, &s);
    require(s.gpu_tasks == 4, "gpu picked");
  });
}

// f1 / f3 evidence: wall time per 4096^2 tile of a 16-tile (16384^2) slide
// through the executor (store view -> H2D -> stage -> D2H -> finalize, three
// stages in flight on one GPU worker), next to the direct C-ABI pipeline on
// the same tiles (rtg_process_tile_async over pitched views of the pinned
// slide into pinned outputs, three in flight): the runtime-path / direct
// ratio the reference gates at <= 1.05 (tests/test_acceptance.cpp:641).
// Cold = first run (pinned payload blocks are page-locked as they are first
// allocated); warm = best of the remaining reps (blocks come from the pool).
void bench_f1(int reps) {
  using clk = std::chrono::steady_clock;
  auto ms_since = [](clk::time_point a) {
    return std::chrono::duration<double, std::milli>(clk::now() - a).count();
  };
  const std::int64_t H = 16384, W = 16384, T = 4096;
  const int tiles = int((H / T) * (W / T));
  rtg_params p;
  rtg_check(rtg_params_default(&p));
  Bytes pixels(std::size_t(H * W * 3));
  auto t = clk::now();
  rtg_check(rtg_synth_tile_host(1405795800ULL, 0, 0, H, W, pixels.data()));
  std::printf("synth slide %lldx%lld %.1f ms\n", (long long)H, (long long)W, ms_since(t));

  double direct_ms = 0;
  {  // direct C-ABI pipeline
    void* sp = nullptr;
    rtg_check(rtg_host_alloc(pixels.size(), &sp));
    std::memcpy(sp, pixels.data(), pixels.size());
    const std::uint8_t* slide = static_cast<const std::uint8_t*>(sp);
    GpuDevice g(0, T, T, 1 << 16);
    std::vector<void*> outs;
    for (int k = 0; k < tiles; ++k) {
      void* o = nullptr;
      rtg_check(rtg_host_alloc(std::size_t(T * T) * 5 + sizeof(float) * (std::size_t(1) << 16) * RTG_NUM_FEATURES, &o));
      outs.push_back(o);
    }
    double best = 1e30;
    for (int r = 0; r < reps; ++r) {
      t = clk::now();
      std::vector<std::uint64_t> tk;
      std::size_t waited = 0;
      for (int k = 0; k < tiles; ++k) {
        const std::int64_t y = (k / (W / T)) * T, x = (k % (W / T)) * T;
        std::uint8_t* o = static_cast<std::uint8_t*>(outs[std::size_t(k)]);
        std::uint64_t ticket = 0;
        rtg_check(rtg_process_tile_async(g.ctx(), slide + (y * W + x) * 3, T, T, 3 * W, &p, o,
                                         reinterpret_cast<std::int32_t*>(o + T * T), nullptr,
                                         reinterpret_cast<float*>(o + 5 * T * T), 1 << 16, &ticket));
        tk.push_back(ticket);
        if (tk.size() - waited == RTG_ASYNC_SLOTS) {
          std::int32_t n = 0;
          rtg_check(rtg_ticket_wait(g.ctx(), tk[waited++], &n));
        }
      }
      for (; waited < tk.size(); ++waited) {
        std::int32_t n = 0;
        rtg_check(rtg_ticket_wait(g.ctx(), tk[waited], &n));
      }
      const double ms = ms_since(t) / tiles;
      std::printf("direct rep %d: %.3f ms/tile\n", r, ms);
      best = std::min(best, ms);
    }
    direct_ms = best;
    for (void* o : outs) rtg_host_free(o);
    rtg_host_free(sp);
  }

  struct Mode {
    const char* name;
    bool pinned;
    int inflight;
  };
  std::string json;
  double exec_warm = 0;
  for (const Mode m : {Mode{"pinned_pipelined", true, 3}, Mode{"pinned_serial", true, 1},
                       Mode{"pageable_pipelined", false, 3}}) {
    if (m.pinned) use_pinned_payloads();
    // one device for every rep, as a long-running worker has: the first rep
    // also pays the context's slot allocation and CUDA-graph captures
    GpuDevice dev(0, T, T, 1 << 16);
    SlideOpts o;
    o.H = H;
    o.W = W;
    o.T = T;
    o.gpu_inflight = m.inflight;
    o.pixels = &pixels;
    o.gpu = &dev;
    double cold = 0, warm = 1e30;
    for (int r = 0; r < std::max(reps, 2); ++r) {
      ExecutorStats st;
      run_slide(o, &st);
      const double ms = g_last_run_ms / tiles;
      std::printf("%s rep %d: %.3f ms/tile (max in flight %zu)\n", m.name, r, ms, st.max_inflight);
      if (r == 0) cold = ms;
      else warm = std::min(warm, ms);
    }
    const PayloadStats ps = payload_stats();
    if (m.pinned) use_pageable_payloads();
    if (std::string(m.name) == "pinned_pipelined") exec_warm = warm;
    char buf[400];
    std::snprintf(buf, sizeof buf,
                  "\"%s\": {\"cold_ms\": %.3f, \"warm_ms\": %.3f, \"pool_hits\": %zu, "
                  "\"pinned_allocs\": %zu, \"fallbacks\": %zu}, ",
                  m.name, cold, warm, ps.pool_hits, ps.hook_allocs, ps.fallbacks);
    json += buf;
  }
  std::printf("{\"bench\": \"f1/f3 executor ms per 4096^2 tile\", \"tiles\": %d, \"reps\": %d, %s"
              "\"direct_ms\": %.3f, \"runtime_over_direct\": %.3f, \"reference_gate\": 1.05}\n",
              tiles, reps, json.c_str(), direct_ms, exec_warm / direct_ms);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "--bench-f1") == 0) {
    bench_f1(argc > 2 ? std::atoi(argv[2]) : 3);
    return 0;
  }
  const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
  containers();
  scheduling();
  if (gpu) gpu_stage();
  std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail ? 1 : 0;
}
