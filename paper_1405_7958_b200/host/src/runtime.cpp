// Storage, WRM variant surface, dataflow and executor (see rt/runtime.hpp).
#include "rt/runtime.hpp"

#include <algorithm>
#include <deque>
#include <limits>
#include <thread>

namespace rt {

// ---- MemoryStore -------------------------------------------------------------

Completion MemoryStore::stage_region(const DataRegion& region, int /*origin_node*/) {
  std::vector<std::shared_ptr<const Piece>> fresh;
  for (const auto& [box, c] : region.chunks())  // copies outside the lock
    fresh.push_back(std::make_shared<const Piece>(
        Piece{box, region.kind(), region.element_kind(), c.payload}));
  std::lock_guard<std::mutex> lk(mu_);
  auto& v = pieces_[region.id()];
  v.insert(v.end(), fresh.begin(), fresh.end());
  return Completion();
}

Completion MemoryStore::stage_region_consume(DataRegion& region, int /*origin_node*/) {
  std::vector<std::shared_ptr<const Piece>> fresh;
  for (const auto& [box, c] : region.chunks())
    fresh.push_back(std::make_shared<const Piece>(
        Piece{box, region.kind(), region.element_kind(),
              std::move(region.find_chunk(box)->payload)}));
  region.drop_payload();
  std::lock_guard<std::mutex> lk(mu_);
  auto& v = pieces_[region.id()];
  v.insert(v.end(), fresh.begin(), fresh.end());
  return Completion();
}

DataRegion MemoryStore::read_region(const DataRegionId& id, const BoundingBox& query) {
  std::vector<std::shared_ptr<const Piece>> ps;
  {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = pieces_.find(id);
    if (it == pieces_.end() || it->second.empty())
      throw NotFoundError("no staged data for " + id.to_string());
    ps = it->second;  // a snapshot: the copies below run without the lock
  }
  const Piece& last = *ps.back();
  const std::size_t es = element_size(last.elem);
  DataRegion out(id, last.kind, last.elem, query);
  // Fast path: one piece exactly covering the query (the tile case) moves
  // no canvas/coverage buffers (contrast: reference assemble_read,
  // src/storage.cpp:21-54, which allocates canvas + mask + ones per piece).
  for (auto p = ps.rbegin(); p != ps.rend(); ++p) {
    if ((*p)->box == query) {
      out.put_chunk(query, (*p)->payload);
      return out;
    }
    if ((*p)->box.intersects(query)) break;  // a newer piece overwrites part of it
  }
  // every cell is written below (or the read throws), so no zero pass
  Bytes canvas(std::size_t(query.volume()) * es);
  // one piece containing the query proves coverage without a per-cell map
  bool covered = false;
  for (const auto& p : ps) covered = covered || p->box.contains(query);
  std::vector<std::uint8_t> seen(covered ? 0 : std::size_t(query.volume()), 0);
  for (const auto& p : ps) {  // staging order: last writer wins
    if (!p->box.intersects(query)) continue;
    copy_box_overlap(canvas, query, p->payload, p->box, es);
    if (!covered) fill_box_overlap(seen, query, p->box, 1);
  }
  if (!covered && std::find(seen.begin(), seen.end(), 0) != seen.end())
    throw NotFoundError("query " + query.to_string() + " has cells never written for " +
                        id.to_string());
  out.put_chunk(query, std::move(canvas));
  return out;
}

std::optional<PayloadView> MemoryStore::view_region(const DataRegionId& id,
                                                    const BoundingBox& query) {
  std::shared_ptr<const Piece> hit;
  {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = pieces_.find(id);
    if (it == pieces_.end()) return std::nullopt;
    // the newest piece touching the query must hold all of it
    for (auto p = it->second.rbegin(); p != it->second.rend(); ++p) {
      if (!(*p)->box.intersects(query)) continue;
      if ((*p)->box.contains(query)) hit = *p;
      break;
    }
  }
  if (!hit || query.empty() || !is_dense(hit->kind)) return std::nullopt;
  const BoundingBox& pb = hit->box;
  // rows (axis-0 steps) are contiguous when every axis after the first
  // non-leading one spans the piece fully
  const int d = query.dims();
  for (int a = 2; a < d; ++a)
    if (query.lo(a) != pb.lo(a) || query.hi(a) != pb.hi(a)) return std::nullopt;
  const std::int64_t es = std::int64_t(element_size(hit->elem));
  std::int64_t inner = es;  // bytes per step of the last axes below axis 1
  for (int a = 2; a < d; ++a) inner *= pb.extent(a);
  const std::int64_t pitch = d >= 2 ? inner * pb.extent(1) : es;
  std::int64_t off = (query.lo(0) - pb.lo(0)) * pitch;
  if (d >= 2) off += (query.lo(1) - pb.lo(1)) * inner;
  PayloadView v;
  v.data = hit->payload.data() + off;
  v.row_pitch = pitch;
  v.kind = hit->kind;
  v.elem = hit->elem;
  v.keep = hit;
  return v;
}

void StorageRegistry::add(std::shared_ptr<StorageBackend> b) {
  const std::string n = b->name();
  if (backends_.count(n)) throw ConfigError("duplicate storage backend " + n);
  backends_[n] = std::move(b);
}

StorageBackend& StorageRegistry::at(const std::string& name) const {
  auto it = backends_.find(name);
  if (it == backends_.end()) throw NotFoundError("no storage backend named " + name);
  return *it->second;
}

// ---- WRM -----------------------------------------------------------------------

double effective_speedup(const TaskNode& t) {
  switch (t.variants) {
    case TaskVariants::kCpuOnly: return 0.0;
    case TaskVariants::kGpuOnly: return std::numeric_limits<double>::infinity();
    case TaskVariants::kBoth: return t.speedup_estimate.value_or(1.0);
  }
  return 1.0;
}

bool device_compatible(const TaskNode& t, DeviceKind d) {
  if (t.variants == TaskVariants::kBoth) return true;
  return (t.variants == TaskVariants::kCpuOnly) == (d == DeviceKind::kCpu);
}

void WrmState::submit(std::vector<TaskNode> tasks) {
  for (const auto& t : tasks) {
    if (tasks_.count(t.task_id)) throw ProtocolError("duplicate task id " + std::to_string(t.task_id));
    if ((t.variants == TaskVariants::kBoth) != t.speedup_estimate.has_value())
      throw ConfigError("speedup_estimate must be set exactly for dual-variant tasks");
  }
  std::set<std::uint64_t> batch;
  for (const auto& t : tasks) batch.insert(t.task_id);
  for (const auto& t : tasks)
    for (auto d : t.deps)
      if (!batch.count(d) && !tasks_.count(d))
        throw ConfigError("unknown dependency " + std::to_string(d));
  std::vector<std::uint64_t> fresh;
  for (auto& t : tasks) {
    Entry e;
    e.seq = seq_++;
    e.node = std::move(t);
    const auto id = e.node.task_id;
    for (auto d : e.node.deps) {
      auto it = tasks_.find(d);
      if (it != tasks_.end() && it->second.state == 3) continue;
      ++e.remaining;
      dependents_[d].push_back(id);
    }
    tasks_.emplace(id, std::move(e));
    fresh.push_back(id);
  }
  for (auto id : fresh) {
    auto& e = tasks_.at(id);
    if (e.remaining == 0) {
      e.state = 1;
      ready_.push_back(id);
    }
  }
}

std::optional<std::uint64_t> WrmState::next(DeviceKind device) {
  std::optional<std::size_t> pick;
  for (std::size_t k = 0; k < ready_.size(); ++k) {
    const TaskNode& t = tasks_.at(ready_[k]).node;
    if (!device_compatible(t, device)) continue;
    if (sched_ == SchedulerKind::kFcfs) {
      pick = k;
      break;
    }
    // PATS: the GPU takes the largest speedup, a CPU core the smallest;
    // ties go to the earliest submission (not the earliest readiness).
    if (!pick) {
      pick = k;
      continue;
    }
    const Entry& pe = tasks_.at(ready_[*pick]);
    const double s = effective_speedup(t);
    const double b = effective_speedup(pe.node);
    const bool better = device == DeviceKind::kGpu ? s > b : s < b;
    if (better || (s == b && tasks_.at(ready_[k]).seq < pe.seq)) pick = k;
  }
  if (!pick) return std::nullopt;
  const auto id = ready_[*pick];
  ready_.erase(ready_.begin() + std::ptrdiff_t(*pick));
  tasks_.at(id).state = 2;
  return id;
}

std::vector<std::uint64_t> WrmState::complete(std::uint64_t id) {
  auto it = tasks_.find(id);
  if (it == tasks_.end() || it->second.state != 2)
    throw ProtocolError("completing task " + std::to_string(id) + " that is not running");
  it->second.state = 3;
  std::vector<std::uint64_t> now;
  for (auto d : dependents_[id]) {
    auto& e = tasks_.at(d);
    if (--e.remaining == 0 && e.state == 0) {
      e.state = 1;
      ready_.push_back(d);
      now.push_back(d);
    }
  }
  return now;
}

const TaskNode& WrmState::task(std::uint64_t id) const {
  auto it = tasks_.find(id);
  if (it == tasks_.end()) throw ProtocolError("unknown task " + std::to_string(id));
  return it->second.node;
}

bool WrmState::all_done() const {
  return std::all_of(tasks_.begin(), tasks_.end(),
                     [](const auto& kv) { return kv.second.state == 3; });
}

// ---- variants ---------------------------------------------------------------------

void VariantRegistry::register_variant(const std::string& name, DeviceKind d, Fn fn) {
  auto& e = entries_[name];
  (d == DeviceKind::kCpu ? e.cpu : e.gpu) = std::move(fn);
}

void VariantRegistry::set_speedup(const std::string& name, double s) {
  if (!(s > 0.0)) throw ConfigError("speedup must be positive");
  entries_[name].speedup = s;
}

bool VariantRegistry::has(const std::string& name, DeviceKind d) const {
  auto it = entries_.find(name);
  if (it == entries_.end()) return false;
  return bool(d == DeviceKind::kCpu ? it->second.cpu : it->second.gpu);
}

TaskNode VariantRegistry::make_task(const std::string& name, std::uint64_t task_id,
                                    std::uint64_t stage_id) const {
  auto it = entries_.find(name);
  if (it == entries_.end() || (!it->second.cpu && !it->second.gpu))
    throw NotFoundError("no variant registered for task " + name);
  const Entry e = it->second;
  TaskNode t;
  t.task_id = task_id;
  t.stage_id = stage_id;
  if (e.cpu && e.gpu) {
    t.variants = TaskVariants::kBoth;
    t.speedup_estimate = e.speedup.value_or(1.0);
  } else {
    t.variants = e.cpu ? TaskVariants::kCpuOnly : TaskVariants::kGpuOnly;
  }
  t.body = [e, name] {
    const DeviceKind d = worker_context().device;
    const Fn& fn = d == DeviceKind::kGpu ? e.gpu : e.cpu;
    if (!fn) throw ProtocolError("task " + name + " has no variant for the assigned device");
    fn();
  };
  return t;
}

WorkerContext& worker_context() {
  thread_local WorkerContext wc;
  return wc;
}

// ---- dataflow ---------------------------------------------------------------------

void ManagerState::add_stage(StageInstance stage) {
  const std::uint64_t id = stage.stage_id;
  const bool fresh = stages_.try_emplace(id, Slot{std::move(stage), std::nullopt, false}).second;
  if (!fresh) throw ProtocolError("stage id " + std::to_string(id) + " is already in the graph");
  insertion_.push_back(id);
}

const ManagerState::Slot& ManagerState::slot(std::uint64_t id) const {
  auto it = stages_.find(id);
  if (it == stages_.end()) throw ProtocolError("no stage " + std::to_string(id) + " in the graph");
  return it->second;
}

bool ManagerState::ready(const Slot& s) const {
  if (s.done || s.worker) return false;
  for (const std::uint64_t d : s.stage.deps) {
    auto it = stages_.find(d);
    if (it == stages_.end() || !it->second.done) return false;
  }
  return true;
}

std::vector<std::uint64_t> ManagerState::eligible_ids() const {
  std::vector<std::uint64_t> out;
  for (const std::uint64_t id : insertion_)
    if (ready(stages_.at(id))) out.push_back(id);
  return out;
}

std::optional<std::uint64_t> ManagerState::dispatch(int worker) {
  for (const std::uint64_t id : insertion_) {  // FIFO among eligible stages
    Slot& s = stages_.at(id);
    if (!ready(s)) continue;
    s.worker = worker;
    return id;
  }
  return std::nullopt;
}

std::vector<std::uint64_t> ManagerState::stage_complete(std::uint64_t id,
                                                        std::vector<StageInstance> spawned) {
  auto it = stages_.find(id);
  if (it == stages_.end())
    throw ProtocolError("completing stage " + std::to_string(id) + ", which is not in the graph");
  if (!it->second.worker)
    throw ProtocolError("completing stage " + std::to_string(id) + " before it was dispatched");
  if (it->second.done)
    throw ProtocolError("stage " + std::to_string(id) + " completed a second time");
  const std::vector<std::uint64_t> before = eligible_ids();
  it->second.done = true;
  log_.push_back(id);
  for (StageInstance& child : spawned) add_stage(std::move(child));
  std::vector<std::uint64_t> now;
  for (const std::uint64_t e : eligible_ids())
    if (std::find(before.begin(), before.end(), e) == before.end()) now.push_back(e);
  return now;
}

bool ManagerState::stuck() const {
  if (all_done()) return false;
  for (const auto& [id, s] : stages_)
    if (s.worker && !s.done) return false;  // something is still running
  return eligible_ids().empty();
}

std::optional<int> ManagerState::assigned_worker(std::uint64_t id) const { return slot(id).worker; }

const StageInstance& ManagerState::stage(std::uint64_t id) const { return slot(id).stage; }

RegionTemplate worker_prepare(const StageInstance& stage, StorageRegistry& storage) {
  RegionTemplate local(stage.stage_kind + "#" + std::to_string(stage.stage_id));
  for (const auto& d : stage.region_descriptors) {
    if (d.io_mode != IoMode::kOutput && !d.lazy) {
      DataRegion r = storage.at(d.storage_binding).read_region(d.id, d.query);
      r.set_io_mode(d.io_mode);
      r.set_storage_binding(d.storage_binding);
      local.insert_data_region(std::move(r));
      continue;
    }
    // shells carry shape only (Dense2D / U8 whatever the rank, as the
    // reference's dataflow.cpp:128); touch_region or the body replaces them
    DataRegion r(d.id, RegionKind::kDense2D, ElementKind::kU8, d.query);
    r.set_io_mode(d.io_mode);
    r.set_storage_binding(d.storage_binding);
    r.set_lazy(d.lazy && d.io_mode != IoMode::kOutput);
    local.insert_data_region(std::move(r));
  }
  return local;
}

DataRegion& touch_region(RegionTemplate& local, const DataRegionId& id, StorageRegistry& storage) {
  DataRegion* shell = local.get_data_region(id);
  if (!shell) throw NotFoundError("touch of " + id.to_string() + ": not in template " + local.name());
  if (!shell->lazy() || shell->materialized()) return *shell;
  DataRegion full = storage.at(shell->storage_binding()).read_region(id, shell->bbox());
  full.set_io_mode(shell->io_mode());
  full.set_storage_binding(shell->storage_binding());
  full.set_lazy(true);
  local.remove_data_region(id);
  return local.insert_data_region(std::move(full));
}

std::vector<Completion> stage_finalize(RegionTemplate& local, const StageInstance& stage,
                                       StorageRegistry& storage, int origin_node, bool consume) {
  std::vector<Completion> out;
  for (const auto& d : stage.region_descriptors) {
    const DataRegion* r = local.get_data_region(d.id);
    if (!r) continue;
    if (d.io_mode == IoMode::kInput) {
      local.remove_data_region(d.id);
      continue;
    }
    if (!r->materialized()) continue;
    StorageBackend& s = storage.at(d.storage_binding);
    out.push_back(consume ? s.stage_region_consume(*local.get_data_region(d.id), origin_node)
                          : s.stage_region(*r, origin_node));
  }
  return out;
}

// ---- executor ------------------------------------------------------------------------

void defer_completion(std::function<void()> finish) {
  WorkerContext& wc = worker_context();
  if (wc.deferred) {
    wc.deferred->push_back(std::move(finish));
    return;
  }
  finish();  // no pipelining executor: complete in place
}

void spawn_stage(StageInstance stage) {
  WorkerContext& wc = worker_context();
  if (!wc.spawned) throw ProtocolError("spawn_stage outside an executor-run task body");
  wc.spawned->push_back(std::move(stage));
}

namespace {

// One dispatched stage on a worker: its local template, its task graph and
// the task completions its bodies deferred to the device.
struct Flight {
  std::uint64_t sid = 0;
  StageInstance stage;
  RegionTemplate local;
  WrmState wrm;
  std::map<std::uint64_t, std::function<void()>> bodies;
  std::vector<std::pair<std::uint64_t, std::function<void()>>> pending;
  std::vector<StageInstance> spawned;
  std::size_t ng = 0, nc = 0, deferred = 0;
  explicit Flight(SchedulerKind s) : wrm(s) {}
  bool finished() const { return pending.empty() && wrm.all_done(); }
};

}  // namespace

ExecutorStats run_stages(ManagerState& manager, StorageRegistry& storage,
                         const ExecutorConfig& cfg) {
  ExecutorStats stats;
  std::mutex mu;  // guards manager + stats + failure
  std::exception_ptr failure;
  const int ngpu = int(cfg.gpus.size());
  const int workers = ngpu + std::max(cfg.cpu_workers, ngpu == 0 ? 1 : 0);

  auto worker = [&](int w) {
    WorkerContext& wc = worker_context();
    std::deque<std::unique_ptr<Flight>> flights;  // dispatch order
    // Device work still in flight writes into the flights' host buffers:
    // run (wait for) every deferred completion before the flights go away.
    auto settle = [&] {
      for (auto& f : flights)
        for (auto& [tid, fn] : f->pending) {
          try {
            wc.local = &f->local;
            fn();
          } catch (...) {
          }
        }
      flights.clear();
      wc = WorkerContext{};
    };
    try {
      wc = WorkerContext{};
      wc.worker = w;
      wc.gpu = w < ngpu ? cfg.gpus[std::size_t(w)] : nullptr;
      wc.storage = &storage;
      const std::size_t depth = wc.gpu ? std::size_t(std::max(cfg.gpu_inflight, 1)) : 1;

      // Runs every task of `f` that is ready on this worker's devices; a
      // body that defers leaves its task running until the completion ran.
      auto advance = [&](Flight& f) {
        for (;;) {
          DeviceKind dev = DeviceKind::kGpu;
          std::optional<std::uint64_t> tid;
          if (wc.gpu) tid = f.wrm.next(DeviceKind::kGpu);
          if (!tid) {
            tid = f.wrm.next(DeviceKind::kCpu);
            dev = DeviceKind::kCpu;
          }
          if (!tid) {
            if (f.pending.empty() && !f.wrm.all_done())
              throw ProtocolError("stage " + std::to_string(f.sid) +
                                  " has tasks no device of this worker can run");
            return;
          }
          std::vector<std::function<void()>> later;
          wc.local = &f.local;
          wc.device = dev;
          wc.deferred = depth > 1 ? &later : nullptr;
          wc.spawned = &f.spawned;
          if (f.bodies[*tid]) f.bodies[*tid]();
          wc.deferred = nullptr;
          (dev == DeviceKind::kGpu ? f.ng : f.nc) += 1;
          if (later.empty()) {
            f.wrm.complete(*tid);
            continue;
          }
          f.deferred += 1;
          f.pending.emplace_back(*tid, [later = std::move(later)] {
            for (const auto& fn : later) fn();
          });
        }
      };
      // Finishes the oldest deferred work of `f` (waits on the device).
      auto drain = [&](Flight& f) {
        while (!f.pending.empty()) {
          wc.local = &f.local;
          wc.spawned = &f.spawned;
          f.pending.front().second();
          const std::uint64_t tid = f.pending.front().first;
          f.pending.erase(f.pending.begin());
          f.wrm.complete(tid);
        }
      };
      auto finish = [&](Flight& f) {
        wc.local = nullptr;
        for (auto& c : stage_finalize(f.local, f.stage, storage, w, /*consume=*/true)) c.wait();
        std::lock_guard<std::mutex> lk(mu);
        manager.stage_complete(f.sid, std::move(f.spawned));
        stats.stages += 1;
        stats.gpu_tasks += f.ng;
        stats.cpu_tasks += f.nc;
        stats.deferred_tasks += f.deferred;
      };

      for (;;) {
        std::unique_ptr<Flight> f;
        bool done = false, wedged = false;
        if (flights.size() < depth) {
          std::unique_lock<std::mutex> lk(mu);
          if (failure) {
            lk.unlock();
            settle();
            return;
          }
          if (auto sid = manager.dispatch(w)) {
            f = std::make_unique<Flight>(cfg.scheduler);
            f->sid = *sid;
            f->stage = manager.stage(*sid);
          } else {
            done = manager.all_done();
            wedged = flights.empty() && manager.stuck();
          }
        }
        if (f) {
          // host work of the next stage (store reads / views) overlaps the
          // device work of the stages already in flight
          f->local = worker_prepare(f->stage, storage);
          std::vector<TaskNode> tasks = f->stage.body ? f->stage.body() : std::vector<TaskNode>{};
          for (const auto& t : tasks) f->bodies[t.task_id] = t.body;
          f->wrm.submit(std::move(tasks));
          advance(*f);
          if (f->finished()) {
            finish(*f);
          } else {
            flights.push_back(std::move(f));
            std::lock_guard<std::mutex> lk(mu);
            stats.max_inflight = std::max(stats.max_inflight, flights.size());
          }
          continue;
        }
        if (!flights.empty()) {
          Flight& old = *flights.front();
          drain(old);
          advance(old);
          if (old.finished()) {
            finish(old);
            flights.pop_front();
          }
          continue;
        }
        if (done) {
          wc = WorkerContext{};
          return;
        }
        if (wedged)
          throw ProtocolError("stage graph is wedged: " + std::to_string(manager.size() -
                                                                         manager.done_count()) +
                              " stages can never become eligible");
        std::this_thread::yield();
      }
    } catch (...) {
      {
        std::lock_guard<std::mutex> lk(mu);
        if (!failure) failure = std::current_exception();
      }
      settle();
    }
  };
  if (workers == 1) {
    worker(0);
  } else {
    std::vector<std::thread> th;
    for (int w = 0; w < workers; ++w) th.emplace_back(worker, w);
    for (auto& t : th) t.join();
  }
  if (failure) std::rethrow_exception(failure);
  return stats;
}

}  // namespace rt
