// Region Templates containers for the B200 stage host layer.
//
// API mirror (names, argument meaning, error behaviour) of the reference's
// region model, re-implemented from its documented semantics:
//   rt::Error taxonomy            /root/reference/proj/include/rt/error.hpp:24-100
//   BoundingBox                   include/rt/bounding_box.hpp:33-90
//   DataRegionId / RegionKind /
//   ElementKind / Chunk / DataRegion  include/rt/data_region.hpp:34-159
//   RegionTemplate                include/rt/region_template.hpp:30-74
// plus DenseDataRegion2D<T>, the typed dense view the paper's API names
// (the reference spells it DataRegion with RegionKind::kDense2D).
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <map>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

namespace rt {

// ---- errors (error.hpp:24-100) + DeviceError for CUDA faults ---------------
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
#define RT_ERROR_KIND(Name) \
  class Name : public Error { \
   public:                    \
    using Error::Error;       \
  }
RT_ERROR_KIND(DimensionError);
RT_ERROR_KIND(DuplicateRegionError);
RT_ERROR_KIND(PartitionError);
RT_ERROR_KIND(EmptyRoiError);
RT_ERROR_KIND(DecodeError);
RT_ERROR_KIND(RangeError);
RT_ERROR_KIND(NotFoundError);
RT_ERROR_KIND(IoError);
RT_ERROR_KIND(CycleError);
RT_ERROR_KIND(ProtocolError);
RT_ERROR_KIND(ConfigError);
// Not in the reference: raised when the GPU variant's C-ABI reports a CUDA
// fault, an allocation failure or a missing device.
RT_ERROR_KIND(DeviceError);
#undef RT_ERROR_KIND

// ---- bounding boxes -----------------------------------------------------------
// Inclusive integer box of up to four axes; the default box (dims 0) is the
// empty sentinel and the identity of unioned().
class BoundingBox {
 public:
  static constexpr int kMaxDims = 4;
  BoundingBox() = default;
  BoundingBox(std::initializer_list<std::int64_t> lo, std::initializer_list<std::int64_t> hi);
  BoundingBox(int dims, const std::int64_t* lo, const std::int64_t* hi);

  int dims() const { return dims_; }
  bool empty() const { return dims_ == 0; }
  std::int64_t lo(int a) const { return lo_[axis(a)]; }
  std::int64_t hi(int a) const { return hi_[axis(a)]; }
  std::int64_t extent(int a) const { return hi_[axis(a)] - lo_[axis(a)] + 1; }
  std::int64_t volume() const;
  bool contains(const BoundingBox& o) const;
  bool intersects(const BoundingBox& o) const { return intersected(o).has_value(); }
  BoundingBox unioned(const BoundingBox& o) const;
  std::optional<BoundingBox> intersected(const BoundingBox& o) const;
  bool operator==(const BoundingBox& o) const;
  bool operator!=(const BoundingBox& o) const { return !(*this == o); }
  bool operator<(const BoundingBox& o) const;
  std::string to_string() const;

 private:
  int axis(int a) const;
  void same_dims(const BoundingBox& o) const;
  int dims_ = 0;
  std::array<std::int64_t, kMaxDims> lo_{}, hi_{};
};

// ---- data regions ------------------------------------------------------------
struct DataRegionId {
  std::string ns, key, type_tag;
  std::int64_t timestamp = 0, version = 0;
  std::string name() const { return ns + "::" + key; }
  bool operator==(const DataRegionId&) const = default;
  bool operator<(const DataRegionId& o) const {
    return std::tie(ns, key, type_tag, timestamp, version) <
           std::tie(o.ns, o.key, o.type_tag, o.timestamp, o.version);
  }
  std::string to_string() const;
};

enum class RegionKind : std::uint8_t { kDense1D = 0, kDense2D = 1, kDense3D = 2, kSparse = 3, kPolygon = 4 };
enum class ElementKind : std::uint8_t { kU8 = 0, kU16 = 1, kI32 = 2, kF32 = 3, kF64 = 4 };
enum class IoMode : std::uint8_t { kInput = 0, kOutput = 1, kInputOutput = 2 };

std::size_t element_size(ElementKind k);
bool is_dense(RegionKind k);
int dense_rank(RegionKind k);

template <typename T> struct element_of;
template <> struct element_of<std::uint8_t> { static constexpr ElementKind value = ElementKind::kU8; };
template <> struct element_of<std::uint16_t> { static constexpr ElementKind value = ElementKind::kU16; };
template <> struct element_of<std::int32_t> { static constexpr ElementKind value = ElementKind::kI32; };
template <> struct element_of<float> { static constexpr ElementKind value = ElementKind::kF32; };
template <> struct element_of<double> { static constexpr ElementKind value = ElementKind::kF64; };

// ---- payload memory -----------------------------------------
// Chunk payloads are byte vectors whose allocator routes blocks of at least
// `min_bytes` through a process-wide hook, so a GPU worker can put them in
// pinned pages (rtg_host_alloc) and the stage DMAs straight from / into the
// chunk (the reference's payload is a plain std::vector<uint8_t>,
// data_region.hpp:87-92, which forces a staged pageable copy).  Every block
// records the free function it came from, so changing the hook never
// mismatches alloc and free; hooked blocks are recycled by exact size up to
// `pool_bytes` (tiles repeat sizes; page-locking costs ms per call).
using PayloadAllocFn = void* (*)(std::size_t bytes);
using PayloadFreeFn = void (*)(void* p);
// alloc == nullptr restores plain heap payloads (and releases the pool).
// `live_bytes` caps the hook's blocks in use (pinned pages are a scarce
// host resource: a whole slide of staged outputs must not page-lock the
// host); beyond it, and whenever the hook fails, payloads fall back to
// plain heap blocks.
void set_payload_allocator(PayloadAllocFn alloc, PayloadFreeFn free, std::size_t min_bytes,
                           std::size_t pool_bytes,
                           std::size_t live_bytes = std::size_t(-1));
// True when `p` (a payload's data()) lives in a block from the hook.
bool payload_is_hooked(const void* p);
struct PayloadStats {
  std::size_t live_bytes = 0;    // hook blocks in use
  std::size_t pooled_bytes = 0;  // hook blocks parked for reuse
  std::size_t pool_hits = 0, hook_allocs = 0, fallbacks = 0;
};
PayloadStats payload_stats();

namespace detail {
void* payload_allocate(std::size_t bytes);
void payload_deallocate(void* p) noexcept;
}  // namespace detail

template <typename T>
struct PayloadAllocator {
  using value_type = T;
  PayloadAllocator() noexcept = default;
  template <typename U>
  PayloadAllocator(const PayloadAllocator<U>&) noexcept {}
  T* allocate(std::size_t n) { return static_cast<T*>(detail::payload_allocate(n * sizeof(T))); }
  // Default-initialises: Bytes(n) / resize(n) leave the bytes unwritten (a
  // payload the next step overwrites whole costs no zero pass); spell the
  // value, Bytes(n, 0), when zeros are meant.
  template <typename U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <typename U, typename... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
  void deallocate(T* p, std::size_t) noexcept { detail::payload_deallocate(p); }
  template <typename U>
  bool operator==(const PayloadAllocator<U>&) const noexcept { return true; }
};

using Bytes = std::vector<std::uint8_t, PayloadAllocator<std::uint8_t>>;

// One stored piece: dense payloads are row-major, last axis contiguous, with
// length volume(bbox) * element_size.
struct Chunk {
  std::uint64_t chunk_id = 0;
  BoundingBox bbox;
  ElementKind element_kind = ElementKind::kU8;
  Bytes payload;
};

class DataRegion {
 public:
  DataRegion() = default;
  DataRegion(DataRegionId id, RegionKind kind, ElementKind element_kind, BoundingBox bbox);

  const DataRegionId& id() const { return id_; }
  RegionKind kind() const { return kind_; }
  ElementKind element_kind() const { return element_kind_; }
  const BoundingBox& bbox() const { return bbox_; }
  const BoundingBox& roi() const { return roi_; }
  IoMode io_mode() const { return io_mode_; }
  const std::string& storage_binding() const { return storage_binding_; }
  bool lazy() const { return lazy_; }
  bool materialized() const { return materialized_; }
  void set_io_mode(IoMode m) { io_mode_ = m; }
  void set_storage_binding(std::string s) { storage_binding_ = std::move(s); }
  void set_lazy(bool l) { lazy_ = l; }
  void set_roi(const BoundingBox& roi);

  const std::map<BoundingBox, Chunk>& chunks() const { return chunks_; }
  // Inserts or replaces (equal box) a chunk; validates box and dense length.
  Chunk& put_chunk(const BoundingBox& box, Bytes payload);
  Chunk& put_chunk(const BoundingBox& box, const std::vector<std::uint8_t>& payload) {
    return put_chunk(box, Bytes(payload.begin(), payload.end()));
  }
  const Chunk* find_chunk(const BoundingBox& box) const;
  Chunk* find_chunk(const BoundingBox& box);
  void drop_payload();
  std::uint64_t payload_bytes() const;
  bool operator==(const DataRegion& o) const;

 private:
  DataRegionId id_;
  RegionKind kind_ = RegionKind::kDense2D;
  ElementKind element_kind_ = ElementKind::kU8;
  BoundingBox bbox_, roi_;
  IoMode io_mode_ = IoMode::kInput;
  std::string storage_binding_;
  bool lazy_ = false, materialized_ = false;
  std::uint64_t next_chunk_id_ = 0;
  std::map<BoundingBox, Chunk> chunks_;
};

// Row-major, last-axis-contiguous copy of the overlap of two boxes.
void copy_box_overlap(std::span<std::uint8_t> dst, const BoundingBox& dst_box,
                      std::span<const std::uint8_t> src, const BoundingBox& src_box,
                      std::size_t elem_size);
// Sets the cells of `dst` (laid out over dst_box, one byte each) that `box`
// covers to `value`.
void fill_box_overlap(std::span<std::uint8_t> dst, const BoundingBox& dst_box,
                      const BoundingBox& box, std::uint8_t value);

// Typed 2-D dense view of a DataRegion whose single chunk covers its bbox
// (the hot path's tile / mask / label containers).
template <typename T>
class DenseDataRegion2D {
 public:
  explicit DenseDataRegion2D(DataRegion& r) : r_(&r) {
    if (r.element_kind() != element_of<T>::value) throw DimensionError("element kind mismatch");
    if (!is_dense(r.kind())) throw DimensionError("not a dense region");
  }
  // Materialises a zero payload over the whole bbox.
  static DataRegion create(DataRegionId id, const BoundingBox& box, RegionKind kind = RegionKind::kDense2D) {
    DataRegion r(std::move(id), kind, element_of<T>::value, box);
    r.put_chunk(box, Bytes(std::size_t(box.volume()) * sizeof(T), 0));
    return r;
  }
  std::int64_t height() const { return r_->bbox().extent(0); }
  std::int64_t width() const { return r_->bbox().extent(1); }
  T* data() { return reinterpret_cast<T*>(chunk().payload.data()); }
  const T* data() const { return reinterpret_cast<const T*>(const_cast<DenseDataRegion2D*>(this)->chunk().payload.data()); }
  T& at(std::int64_t y, std::int64_t x) { return data()[y * width() + x]; }

 private:
  Chunk& chunk() {
    Chunk* c = r_->find_chunk(r_->bbox());
    if (!c) throw NotFoundError("dense view needs one chunk covering " + r_->bbox().to_string());
    return *c;
  }
  DataRegion* r_;
};

// ---- region templates ------------------------------------------------------
class RegionTemplate {
 public:
  RegionTemplate() = default;
  explicit RegionTemplate(std::string name) : name_(std::move(name)) {}
  const std::string& name() const { return name_; }
  const BoundingBox& bbox() const { return bbox_; }
  std::size_t size() const { return regions_.size(); }
  bool empty() const { return regions_.empty(); }
  DataRegion& insert_data_region(DataRegion region);
  const DataRegion* get_data_region(const DataRegionId& id) const;
  DataRegion* get_data_region(const DataRegionId& id);
  const DataRegion* get_newest(const std::string& ns, const std::string& key,
                               const std::string& type_tag) const;
  bool remove_data_region(const DataRegionId& id);
  const std::map<DataRegionId, DataRegion>& regions() const { return regions_; }

 private:
  void refold();
  std::string name_;
  BoundingBox bbox_;
  std::map<DataRegionId, DataRegion> regions_;
};

}  // namespace rt
