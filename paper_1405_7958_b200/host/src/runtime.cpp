// Storage, WRM variant surface, dataflow and executor (see rt/runtime.hpp).
#include "rt/runtime.hpp"

#include <algorithm>
#include <limits>
#include <thread>

namespace rt {

// ---- MemoryStore -------------------------------------------------------------

Completion MemoryStore::stage_region(const DataRegion& region, int /*origin_node*/) {
  std::lock_guard<std::mutex> lk(mu_);
  auto& v = pieces_[region.id()];
  for (const auto& [box, c] : region.chunks())
    v.push_back(Piece{box, region.kind(), region.element_kind(), c.payload});
  return Completion();
}

Completion MemoryStore::stage_region_consume(DataRegion& region, int /*origin_node*/) {
  std::vector<BoundingBox> boxes;
  for (const auto& [box, c] : region.chunks()) boxes.push_back(box);
  {
    std::lock_guard<std::mutex> lk(mu_);
    auto& v = pieces_[region.id()];
    for (const auto& box : boxes)
      v.push_back(Piece{box, region.kind(), region.element_kind(),
                        std::move(region.find_chunk(box)->payload)});
  }
  region.drop_payload();
  return Completion();
}

DataRegion MemoryStore::read_region(const DataRegionId& id, const BoundingBox& query) {
  std::lock_guard<std::mutex> lk(mu_);
  auto it = pieces_.find(id);
  if (it == pieces_.end() || it->second.empty())
    throw NotFoundError("no staged data for " + id.to_string());
  const Piece& last = it->second.back();
  const std::size_t es = element_size(last.elem);
  DataRegion out(id, last.kind, last.elem, query);
  // Fast path: one piece exactly covering the query (the tile case) moves
  // no canvas/coverage buffers (contrast: reference assemble_read,
  // src/storage.cpp:21-54, which allocates canvas + mask + ones per piece).
  for (auto p = it->second.rbegin(); p != it->second.rend(); ++p) {
    if (p->box == query) {
      out.put_chunk(query, p->payload);
      return out;
    }
    if (p->box.intersects(query)) break;  // a newer piece overwrites part of it
  }
  // every cell is written below (or the read throws), so no zero pass
  Bytes canvas(std::size_t(query.volume()) * es);
  // one piece containing the query proves coverage without a per-cell map
  bool covered = false;
  for (const auto& p : it->second) covered = covered || p.box.contains(query);
  std::vector<std::uint8_t> seen(covered ? 0 : std::size_t(query.volume()), 0);
  for (const auto& p : it->second) {  // staging order: last writer wins
    if (!p.box.intersects(query)) continue;
    copy_box_overlap(canvas, query, p.payload, p.box, es);
    if (!covered) fill_box_overlap(seen, query, p.box, 1);
  }
  if (!covered && std::find(seen.begin(), seen.end(), 0) != seen.end())
    throw NotFoundError("query " + query.to_string() + " has cells never written for " +
                        id.to_string());
  out.put_chunk(query, std::move(canvas));
  return out;
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
  const auto id = stage.stage_id;
  if (stages_.count(id)) throw ProtocolError("duplicate stage id " + std::to_string(id));
  stages_.emplace(id, E{std::move(stage)});
  order_.push_back(id);
}

bool ManagerState::eligible(const E& e) const {
  if (e.assigned || e.done) return false;
  for (auto d : e.stage.deps) {
    auto it = stages_.find(d);
    if (it == stages_.end() || !it->second.done) return false;
  }
  return true;
}

std::optional<std::uint64_t> ManagerState::dispatch(int /*worker*/) {
  for (auto id : order_) {  // FIFO among eligible stages
    auto& e = stages_.at(id);
    if (eligible(e)) {
      e.assigned = true;
      return id;
    }
  }
  return std::nullopt;
}

std::vector<std::uint64_t> ManagerState::stage_complete(std::uint64_t id) {
  auto it = stages_.find(id);
  if (it == stages_.end() || !it->second.assigned || it->second.done)
    throw ProtocolError("stage " + std::to_string(id) + " is not running");
  it->second.done = true;
  ++done_;
  std::vector<std::uint64_t> now;
  for (auto sid : order_)
    if (eligible(stages_.at(sid))) now.push_back(sid);
  return now;
}

const StageInstance& ManagerState::stage(std::uint64_t id) const {
  auto it = stages_.find(id);
  if (it == stages_.end()) throw ProtocolError("unknown stage " + std::to_string(id));
  return it->second.stage;
}

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
    const RegionKind kind = d.query.dims() == 3 ? RegionKind::kDense3D : RegionKind::kDense2D;
    DataRegion r(d.id, kind, ElementKind::kU8, d.query);
    r.set_io_mode(d.io_mode);
    r.set_storage_binding(d.storage_binding);
    r.set_lazy(d.lazy && d.io_mode != IoMode::kOutput);
    local.insert_data_region(std::move(r));
  }
  return local;
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

ExecutorStats run_stages(ManagerState& manager, StorageRegistry& storage,
                         const ExecutorConfig& cfg) {
  ExecutorStats stats;
  std::mutex mu;  // guards manager + stats
  std::exception_ptr failure;
  const int ngpu = int(cfg.gpus.size());
  const int workers = ngpu + std::max(cfg.cpu_workers, ngpu == 0 ? 1 : 0);

  auto worker = [&](int w) {
    try {
      WorkerContext& wc = worker_context();
      wc.worker = w;
      wc.gpu = w < ngpu ? cfg.gpus[std::size_t(w)] : nullptr;
      for (;;) {
        std::optional<std::uint64_t> sid;
        StageInstance stage;
        {
          std::lock_guard<std::mutex> lk(mu);
          if (failure || manager.all_done()) return;
          sid = manager.dispatch(w);
          if (sid) stage = manager.stage(*sid);
        }
        if (!sid) {
          std::this_thread::yield();
          continue;
        }
        RegionTemplate local = worker_prepare(stage, storage);
        WrmState wrm(cfg.scheduler);
        std::vector<TaskNode> tasks = stage.body ? stage.body() : std::vector<TaskNode>{};
        std::map<std::uint64_t, std::function<void()>> bodies;
        for (const auto& t : tasks) bodies[t.task_id] = t.body;
        wrm.submit(std::move(tasks));
        std::size_t ng = 0, nc = 0;
        while (!wrm.all_done()) {
          DeviceKind dev = DeviceKind::kCpu;
          std::optional<std::uint64_t> tid;
          if (wc.gpu) {
            tid = wrm.next(DeviceKind::kGpu);
            dev = DeviceKind::kGpu;
          }
          if (!tid) {
            tid = wrm.next(DeviceKind::kCpu);
            dev = DeviceKind::kCpu;
          }
          if (!tid) throw ProtocolError("stage " + std::to_string(*sid) +
                                        " has tasks no device of this worker can run");
          wc.local = &local;
          wc.device = dev;
          if (bodies[*tid]) bodies[*tid]();
          (dev == DeviceKind::kGpu ? ng : nc) += 1;
          wrm.complete(*tid);
        }
        wc.local = nullptr;
        for (auto& c : stage_finalize(local, stage, storage, w, /*consume=*/true)) c.wait();
        std::lock_guard<std::mutex> lk(mu);
        manager.stage_complete(*sid);
        stats.stages += 1;
        stats.gpu_tasks += ng;
        stats.cpu_tasks += nc;
      }
    } catch (...) {
      std::lock_guard<std::mutex> lk(mu);
      if (!failure) failure = std::current_exception();
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
