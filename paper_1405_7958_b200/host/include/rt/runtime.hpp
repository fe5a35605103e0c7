// Stage/task dataflow, worker scheduler (variant surface), storage and the
// executor that runs stage bodies on CPU slots or B200 contexts.
//
// API mirror of the reference's runtime surface (re-implemented):
//   StorageBackend / StorageRegistry / Completion  include/rt/storage.hpp:34-162
//   TaskNode / TaskVariants / DeviceKind / WrmState  include/rt/wrm.hpp:29-137
//     (FCFS and PATS device picks, src/wrm.cpp:246-273; DL reuse / prefetch
//     model are out of scope for this hot-path build)
//   RegionDescriptor / StageInstance / ManagerState / worker_prepare /
//   stage_finalize                                   include/rt/dataflow.hpp:33-114
// New here: VariantRegistry (function-variant registration by name) and
// WorkerContext (what a TaskNode::body reaches while it runs: the stage's
// local RegionTemplate and the device the WRM picked).
#pragma once

#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <set>
#include <string>
#include <vector>

#include "rt/region.hpp"

namespace rt {

// ---- storage ------------------------------------------------------------------
// A read-only window onto staged bytes (no copy): `data` is the query box's
// first cell and consecutive steps of axis 0 are `row_pitch` bytes apart;
// within one step the query's remaining axes are contiguous.  `keep` holds
// the stored piece alive while the view is in use (e.g. by a DMA).
struct PayloadView {
  const std::uint8_t* data = nullptr;
  std::int64_t row_pitch = 0;
  RegionKind kind = RegionKind::kDense2D;
  ElementKind elem = ElementKind::kU8;
  std::shared_ptr<const void> keep;
};

// Completion of a staging operation (always complete for the in-memory store).
class Completion {
 public:
  Completion() = default;
  void wait() const {}
  bool ready() const { return true; }
};

class StorageBackend {
 public:
  virtual ~StorageBackend() = default;
  virtual const std::string& name() const = 0;
  // Persists every chunk of a materialised region (last writer wins).
  virtual Completion stage_region(const DataRegion& region, int origin_node) = 0;
  // Same, for a region the caller is done with: a backend may take the
  // payloads instead of copying them; the region ends unmaterialised.
  virtual Completion stage_region_consume(DataRegion& region, int origin_node) {
    Completion c = stage_region(region, origin_node);
    region.drop_payload();
    return c;
  }
  // Assembles the query box from staged chunks; NotFoundError when any cell
  // was never written.
  virtual DataRegion read_region(const DataRegionId& id, const BoundingBox& query) = 0;
  // Zero-copy alternative to read_region when one stored piece holds the
  // whole query and the query is row-contiguous in it (a tile
  // of a staged slide DMAs straight from the slide).  nullopt otherwise.
  virtual std::optional<PayloadView> view_region(const DataRegionId& /*id*/,
                                                 const BoundingBox& /*query*/) {
    return std::nullopt;
  }
};

// Process-local store keyed by region tuple; thread-safe.
class MemoryStore : public StorageBackend {
 public:
  explicit MemoryStore(std::string name) : name_(std::move(name)) {}
  const std::string& name() const override { return name_; }
  Completion stage_region(const DataRegion& region, int origin_node) override;
  Completion stage_region_consume(DataRegion& region, int origin_node) override;
  DataRegion read_region(const DataRegionId& id, const BoundingBox& query) override;
  std::optional<PayloadView> view_region(const DataRegionId& id, const BoundingBox& query) override;

 private:
  struct Piece {
    BoundingBox box;
    RegionKind kind;
    ElementKind elem;
    Bytes payload;
  };
  std::string name_;
  std::mutex mu_;
  // staging order per region; shared so a view outlives later stagings
  std::map<DataRegionId, std::vector<std::shared_ptr<const Piece>>> pieces_;
};

class StorageRegistry {
 public:
  void add(std::shared_ptr<StorageBackend> b);
  StorageBackend& at(const std::string& name) const;

 private:
  std::map<std::string, std::shared_ptr<StorageBackend>> backends_;
};

// ---- tasks and the worker scheduler ------------------------------------------------
enum class DeviceKind : std::uint8_t { kCpu = 0, kGpu = 1 };
enum class TaskVariants : std::uint8_t { kCpuOnly = 0, kGpuOnly = 1, kBoth = 2 };
enum class SchedulerKind : std::uint8_t { kFcfs = 0, kPats = 1 };

struct TaskNode {
  std::uint64_t task_id = 0;
  std::set<std::uint64_t> deps;
  TaskVariants variants = TaskVariants::kBoth;
  // GPU acceleration vs one CPU core; required exactly when variants == kBoth.
  std::optional<double> speedup_estimate;
  double cost_cpu = 1.0;
  std::uint64_t stage_id = 0;
  // Runs the task; reaches its data through worker_context().
  std::function<void()> body;
};

double effective_speedup(const TaskNode& t);
bool device_compatible(const TaskNode& t, DeviceKind d);

class WrmState {
 public:
  explicit WrmState(SchedulerKind s = SchedulerKind::kFcfs) : sched_(s) {}
  void submit(std::vector<TaskNode> tasks);
  std::optional<std::uint64_t> next(DeviceKind device);
  std::vector<std::uint64_t> complete(std::uint64_t task_id);
  const TaskNode& task(std::uint64_t id) const;
  bool all_done() const;
  std::size_t ready_count() const { return ready_.size(); }

 private:
  struct Entry {
    TaskNode node;
    int state = 0;  // 0 pending, 1 ready, 2 running, 3 done
    std::size_t remaining = 0;
    std::uint64_t seq = 0;
  };
  SchedulerKind sched_;
  std::uint64_t seq_ = 0;
  std::map<std::uint64_t, Entry> tasks_;
  std::map<std::uint64_t, std::vector<std::uint64_t>> dependents_;
  std::vector<std::uint64_t> ready_;  // readiness order
};

// ---- function variants ----------------------------------------------------------------
// name -> {CPU implementation, GPU implementation, speedup estimate}.
// make_task() derives TaskNode::variants from which implementations exist
// and dispatches body() on the device the executor assigned.
class VariantRegistry {
 public:
  using Fn = std::function<void()>;
  void register_variant(const std::string& name, DeviceKind device, Fn fn);
  void set_speedup(const std::string& name, double s);
  bool has(const std::string& name, DeviceKind device) const;
  TaskNode make_task(const std::string& name, std::uint64_t task_id, std::uint64_t stage_id) const;

 private:
  struct Entry {
    Fn cpu, gpu;
    std::optional<double> speedup;
  };
  std::map<std::string, Entry> entries_;
};

class GpuDevice;  // rt/rtg_stage.hpp

struct StageInstance;

// What a running TaskNode::body can see (set by the executor per task).
struct WorkerContext {
  RegionTemplate* local = nullptr;
  DeviceKind device = DeviceKind::kCpu;
  GpuDevice* gpu = nullptr;
  int worker = 0;
  StorageRegistry* storage = nullptr;  // for touch_region / view_region in bodies
  // Set by a pipelining executor while a body runs: completions the body
  // deferred (defer_completion) and stages it spawned (spawn_stage).
  std::vector<std::function<void()>>* deferred = nullptr;
  std::vector<StageInstance>* spawned = nullptr;
};
WorkerContext& worker_context();

// A body that enqueued asynchronous device work hands the rest of its work
// (wait for the device, install outputs) to the executor: the task counts
// as complete only after `finish` ran, and the executor may prepare and
// start other stages meanwhile (the paper's 3-phase pipeline, PAPER.md:
// 687-700; reference wrm.cpp:385-415).  Without a pipelining executor
// `finish` runs at once.
void defer_completion(std::function<void()> finish);
// Adds a stage to the manager when the running stage completes (reference
// ManagerState::stage_complete(id, spawned), dataflow.cpp:84-111).
void spawn_stage(StageInstance stage);

// ---- dataflow ---------------------------------------------------------------------------
struct RegionDescriptor {
  DataRegionId id;
  BoundingBox query;
  IoMode io_mode = IoMode::kInput;
  std::string storage_binding;
  bool lazy = false;
};

struct StageInstance {
  std::uint64_t stage_id = 0;
  std::string stage_kind;
  std::vector<RegionDescriptor> region_descriptors;
  std::set<std::uint64_t> deps;
  std::function<std::vector<TaskNode>()> body;
};

// Manager-side stage graph (reference dataflow.hpp:51-99): demand-driven
// dispatch of the first eligible stage in insertion order; completing a
// stage may spawn new ones (the graph grows while it runs).
class ManagerState {
 public:
  // ProtocolError on a duplicate id.  Dependencies may name stages that are
  // added later; they stay unsatisfied until that stage completes.
  void add_stage(StageInstance stage);
  std::optional<std::uint64_t> dispatch(int worker);
  // Marks an assigned stage done, adds the stages it spawned and returns the
  // ids that became eligible because of it (insertion order).  ProtocolError
  // for unknown, undispatched or already completed stages.
  std::vector<std::uint64_t> stage_complete(std::uint64_t stage_id,
                                            std::vector<StageInstance> spawned = {});
  const StageInstance& stage(std::uint64_t id) const;
  std::size_t size() const { return stages_.size(); }
  std::size_t done_count() const { return log_.size(); }
  bool all_done() const { return done_count() == size(); }
  // No stage is running or dispatchable but some are not done: a wedge
  // (unsatisfiable or cyclic dependencies).
  bool stuck() const;
  std::vector<std::uint64_t> eligible_ids() const;
  std::optional<int> assigned_worker(std::uint64_t id) const;
  const std::vector<std::uint64_t>& completion_log() const { return log_; }

 private:
  struct Slot {
    StageInstance stage;
    std::optional<int> worker;  // set by dispatch
    bool done = false;
  };
  const Slot& slot(std::uint64_t id) const;
  bool ready(const Slot& s) const;
  std::map<std::uint64_t, Slot> stages_;
  std::vector<std::uint64_t> insertion_;
  std::vector<std::uint64_t> log_;
};

// Reads non-lazy inputs into a fresh local template; outputs are created
// metadata-only (Dense2D/U8 shells, as the reference does) — stage bodies
// replace them with correctly typed regions.
RegionTemplate worker_prepare(const StageInstance& stage, StorageRegistry& storage);
// Read-on-touch for a lazy region of the local template (reference
// dataflow.cpp:137-154): the first touch replaces the metadata-only shell by
// the stored payload (keeping io mode, binding and the lazy flag), later
// touches return the region as is.  NotFoundError when `id` is not in the
// template or the store has no data for it.
DataRegion& touch_region(RegionTemplate& local, const DataRegionId& id, StorageRegistry& storage);

// Stages materialised outputs and drops inputs; completions in descriptor order.
// consume = true (the executor, which discards `local` next) lets the store
// take the output payloads instead of copying them.
std::vector<Completion> stage_finalize(RegionTemplate& local, const StageInstance& stage,
                                       StorageRegistry& storage, int origin_node,
                                       bool consume = false);

// ---- executor ------------------------------------------------------------------------------
// Demand-driven loop over the manager's stages (the real counterpart of the
// simulator's start_task slot, /root/reference/proj/src/sim.cpp:630-685):
// prepare -> expand body -> WRM picks device per task -> run -> finalize.
// Cooperative CPU+GPU execution: one
// worker thread per GPU plus cpu_workers CPU worker threads pull stages
// demand-driven from the manager; inside a stage the WRM picks each task's
// device (PATS: the GPU worker takes the highest-speedup variant first).
struct ExecutorConfig {
  SchedulerKind scheduler = SchedulerKind::kPats;
  std::vector<GpuDevice*> gpus;  // one worker each
  int cpu_workers = 0;           // additional CPU-only workers (>= 1 when no GPU)
  // Stages a GPU worker keeps in flight: while the device runs stage k
  // (asynchronous bodies, defer_completion) the worker prepares and starts
  // stage k+1.  1 = one stage at a time; 3 = the C-ABI's slots per context
  // (RTG_ASYNC_SLOTS: upload, compute and download of three tiles overlap).
  int gpu_inflight = 3;
};
struct ExecutorStats {
  std::size_t stages = 0, cpu_tasks = 0, gpu_tasks = 0;
  std::size_t deferred_tasks = 0;  // GPU tasks whose completion overlapped other stages
  std::size_t max_inflight = 0;    // most stages one worker had in flight
};
ExecutorStats run_stages(ManagerState& manager, StorageRegistry& storage,
                         const ExecutorConfig& cfg);

}  // namespace rt
