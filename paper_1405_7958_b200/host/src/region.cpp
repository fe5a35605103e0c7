// Region Templates containers (see rt/region.hpp for the reference anchors).
#include "rt/region.hpp"

#include <algorithm>
#include <mutex>
#include <new>
#include <sstream>
#include <unordered_map>

namespace rt {

// ---- payload memory ----------------------------------------------------------

namespace {

// 64-byte prefix in front of every payload block: who frees it and its size.
struct alignas(64) BlockHeader {
  PayloadFreeFn free;  // nullptr: aligned operator new
  std::size_t bytes;
};
static_assert(sizeof(BlockHeader) == 64);

struct PayloadHooks {
  std::mutex mu;
  PayloadAllocFn alloc = nullptr;
  PayloadFreeFn free = nullptr;
  std::size_t min_bytes = 0;
  std::size_t pool_cap = 0;
  std::size_t pooled = 0;
  std::size_t live_cap = std::size_t(-1);
  std::size_t live = 0;
  std::size_t hits = 0, allocs = 0, fallbacks = 0;
  std::unordered_map<std::size_t, std::vector<BlockHeader*>> pool;  // hook blocks by size

  void release_pool_locked() {
    for (auto& [n, v] : pool)
      for (BlockHeader* h : v) h->free(h);
    pool.clear();
    pooled = 0;
  }
};

PayloadHooks& hooks() {
  static PayloadHooks* h = new PayloadHooks();  // outlives static payloads
  return *h;
}

BlockHeader* header_of(const void* p) {
  return reinterpret_cast<BlockHeader*>(const_cast<char*>(static_cast<const char*>(p)) -
                                        sizeof(BlockHeader));
}

}  // namespace

void set_payload_allocator(PayloadAllocFn alloc, PayloadFreeFn free, std::size_t min_bytes,
                           std::size_t pool_bytes, std::size_t live_bytes) {
  if ((alloc == nullptr) != (free == nullptr))
    throw ProtocolError("payload allocator needs both alloc and free");
  PayloadHooks& h = hooks();
  std::lock_guard<std::mutex> lk(h.mu);
  h.release_pool_locked();
  h.alloc = alloc;
  h.free = free;
  h.min_bytes = min_bytes;
  h.pool_cap = alloc ? pool_bytes : 0;
  h.live_cap = live_bytes;
}

PayloadStats payload_stats() {
  PayloadHooks& h = hooks();
  std::lock_guard<std::mutex> lk(h.mu);
  return PayloadStats{h.live, h.pooled, h.hits, h.allocs, h.fallbacks};
}

bool payload_is_hooked(const void* p) { return p && header_of(p)->free != nullptr; }

namespace detail {

void* payload_allocate(std::size_t bytes) {
  PayloadHooks& h = hooks();
  const std::size_t total = bytes + sizeof(BlockHeader);
  {
    std::lock_guard<std::mutex> lk(h.mu);
    if (h.alloc && bytes >= h.min_bytes) {
      BlockHeader* b = nullptr;
      auto it = h.pool.find(bytes);
      if (it != h.pool.end() && !it->second.empty()) {
        b = it->second.back();
        it->second.pop_back();
        h.pooled -= total;
        ++h.hits;
      } else if (h.live + total <= h.live_cap) {
        b = static_cast<BlockHeader*>(h.alloc(total));
        if (b) ++h.allocs;
      }
      if (b) {
        b->free = h.free;
        b->bytes = bytes;
        h.live += total;
        return b + 1;
      }
      ++h.fallbacks;  // over the live budget, or the hook failed: heap block
    }
  }
  auto* b = static_cast<BlockHeader*>(::operator new(total, std::align_val_t(64)));
  b->free = nullptr;
  b->bytes = bytes;
  return b + 1;
}

void payload_deallocate(void* p) noexcept {
  if (!p) return;
  BlockHeader* b = header_of(p);
  if (!b->free) {
    ::operator delete(b, std::align_val_t(64));
    return;
  }
  PayloadHooks& h = hooks();
  const std::size_t total = b->bytes + sizeof(BlockHeader);
  {
    std::lock_guard<std::mutex> lk(h.mu);
    h.live -= std::min(h.live, total);  // every hooked block counts, whichever hook made it
    if (b->free == h.free && h.pooled + total <= h.pool_cap) {
      try {
        h.pool[b->bytes].push_back(b);
        h.pooled += total;
        return;
      } catch (...) {
      }
    }
  }
  b->free(b);
}

}  // namespace detail

// ---- BoundingBox ------------------------------------------------------------

BoundingBox::BoundingBox(std::initializer_list<std::int64_t> lo,
                         std::initializer_list<std::int64_t> hi) {
  if (lo.size() != hi.size()) throw DimensionError("lo/hi rank mismatch");
  // rank 0 is the empty box (the reference builds it through the same path)
  if (lo.size() > kMaxDims) throw DimensionError("box rank must be 0..4");
  dims_ = int(lo.size());
  std::copy(lo.begin(), lo.end(), lo_.begin());
  std::copy(hi.begin(), hi.end(), hi_.begin());
  for (int a = 0; a < dims_; ++a)
    if (lo_[a] > hi_[a]) throw DimensionError("box lo exceeds hi on axis " + std::to_string(a));
}

BoundingBox::BoundingBox(int dims, const std::int64_t* lo, const std::int64_t* hi) {
  if (dims < 0 || dims > kMaxDims) throw DimensionError("box rank must be 0..4");
  dims_ = dims;
  for (int a = 0; a < dims; ++a) {
    lo_[a] = lo[a];
    hi_[a] = hi[a];
    if (lo_[a] > hi_[a]) throw DimensionError("box lo exceeds hi on axis " + std::to_string(a));
  }
}

int BoundingBox::axis(int a) const {
  if (a < 0 || a >= dims_) throw DimensionError("axis out of range");
  return a;
}

void BoundingBox::same_dims(const BoundingBox& o) const {
  if (dims_ != o.dims_) throw DimensionError("combining boxes of different rank");
}

std::int64_t BoundingBox::volume() const {
  if (empty()) return 0;
  std::int64_t v = 1;
  for (int a = 0; a < dims_; ++a) v *= hi_[a] - lo_[a] + 1;
  return v;
}

bool BoundingBox::contains(const BoundingBox& o) const {
  // every box contains the empty box; a rank mismatch (including an empty
  // box asked about a non-empty one) is a DimensionError, as in the reference
  if (o.empty()) return true;
  same_dims(o);
  for (int a = 0; a < dims_; ++a)
    if (o.lo_[a] < lo_[a] || o.hi_[a] > hi_[a]) return false;
  return true;
}

BoundingBox BoundingBox::unioned(const BoundingBox& o) const {
  if (empty()) return o;
  if (o.empty()) return *this;
  same_dims(o);
  BoundingBox r = *this;
  for (int a = 0; a < dims_; ++a) {
    r.lo_[a] = std::min(lo_[a], o.lo_[a]);
    r.hi_[a] = std::max(hi_[a], o.hi_[a]);
  }
  return r;
}

std::optional<BoundingBox> BoundingBox::intersected(const BoundingBox& o) const {
  if (empty() || o.empty()) return std::nullopt;
  same_dims(o);
  BoundingBox r = *this;
  for (int a = 0; a < dims_; ++a) {
    r.lo_[a] = std::max(lo_[a], o.lo_[a]);
    r.hi_[a] = std::min(hi_[a], o.hi_[a]);
    if (r.lo_[a] > r.hi_[a]) return std::nullopt;
  }
  return r;
}

bool BoundingBox::operator==(const BoundingBox& o) const {
  if (dims_ != o.dims_) return false;
  for (int a = 0; a < dims_; ++a)
    if (lo_[a] != o.lo_[a] || hi_[a] != o.hi_[a]) return false;
  return true;
}

bool BoundingBox::operator<(const BoundingBox& o) const {
  // rank first, then axis by axis (lo, hi) — the reference's map-key order
  if (dims_ != o.dims_) return dims_ < o.dims_;
  for (int a = 0; a < dims_; ++a) {
    if (lo_[a] != o.lo_[a]) return lo_[a] < o.lo_[a];
    if (hi_[a] != o.hi_[a]) return hi_[a] < o.hi_[a];
  }
  return false;
}

std::string BoundingBox::to_string() const {
  if (empty()) return "<empty>";
  std::ostringstream s;
  s << '<';
  for (int a = 0; a < dims_; ++a) s << (a ? "," : "") << lo_[a];
  s << ';';
  for (int a = 0; a < dims_; ++a) s << (a ? "," : "") << hi_[a];
  s << '>';
  return s.str();
}

// ---- element kinds ------------------------------------------------------------

std::size_t element_size(ElementKind k) {
  switch (k) {
    case ElementKind::kU8: return 1;
    case ElementKind::kU16: return 2;
    case ElementKind::kI32: return 4;
    case ElementKind::kF32: return 4;
    case ElementKind::kF64: return 8;
  }
  throw ConfigError("unknown element kind");
}

bool is_dense(RegionKind k) {
  return k == RegionKind::kDense1D || k == RegionKind::kDense2D || k == RegionKind::kDense3D;
}

int dense_rank(RegionKind k) {
  switch (k) {
    case RegionKind::kDense1D: return 1;
    case RegionKind::kDense2D: return 2;
    case RegionKind::kDense3D: return 3;
    default: return 0;
  }
}

std::string DataRegionId::to_string() const {
  return name() + "[" + type_tag + ",t=" + std::to_string(timestamp) + ",v=" +
         std::to_string(version) + "]";
}

// ---- DataRegion ---------------------------------------------------------------

DataRegion::DataRegion(DataRegionId id, RegionKind kind, ElementKind element_kind,
                       BoundingBox bbox)
    : id_(std::move(id)), kind_(kind), element_kind_(element_kind), bbox_(bbox), roi_(bbox) {
  // dense boxes carry the kind's rank, optionally plus a trailing time axis
  if (is_dense(kind_) && !bbox_.empty() && bbox_.dims() != dense_rank(kind_) &&
      bbox_.dims() != dense_rank(kind_) + 1)
    throw DimensionError("region box rank " + std::to_string(bbox_.dims()) +
                         " does not match its kind");
}

void DataRegion::set_roi(const BoundingBox& roi) {
  if (!roi.empty() && (bbox_.empty() || !bbox_.contains(roi)))
    throw DimensionError("roi must lie inside the region box");
  roi_ = roi;
}

Chunk& DataRegion::put_chunk(const BoundingBox& box, Bytes payload) {
  if (box.empty()) throw DimensionError("empty chunk box");
  if (bbox_.empty() || !bbox_.contains(box))
    throw DimensionError("chunk " + box.to_string() + " escapes region " + bbox_.to_string());
  if (is_dense(kind_) &&
      payload.size() != std::uint64_t(box.volume()) * element_size(element_kind_))
    throw DimensionError("dense chunk payload length " + std::to_string(payload.size()) +
                         " != volume * element size");
  auto [it, fresh] = chunks_.try_emplace(box);
  if (fresh) it->second.chunk_id = next_chunk_id_++;
  it->second.bbox = box;
  it->second.element_kind = element_kind_;
  it->second.payload = std::move(payload);
  materialized_ = true;
  return it->second;
}

const Chunk* DataRegion::find_chunk(const BoundingBox& box) const {
  auto it = chunks_.find(box);
  return it == chunks_.end() ? nullptr : &it->second;
}

Chunk* DataRegion::find_chunk(const BoundingBox& box) {
  auto it = chunks_.find(box);
  return it == chunks_.end() ? nullptr : &it->second;
}

void DataRegion::drop_payload() {
  chunks_.clear();
  materialized_ = false;
}

std::uint64_t DataRegion::payload_bytes() const {
  std::uint64_t n = 0;
  for (const auto& [b, c] : chunks_) n += c.payload.size();
  return n;
}

bool DataRegion::operator==(const DataRegion& o) const {
  if (!(id_ == o.id_) || kind_ != o.kind_ || element_kind_ != o.element_kind_ ||
      bbox_ != o.bbox_ || roi_ != o.roi_ || io_mode_ != o.io_mode_ ||
      storage_binding_ != o.storage_binding_ || lazy_ != o.lazy_ ||
      materialized_ != o.materialized_ || chunks_.size() != o.chunks_.size())
    return false;
  auto a = chunks_.begin();
  auto b = o.chunks_.begin();
  for (; a != chunks_.end(); ++a, ++b)
    if (a->first != b->first || a->second.payload != b->second.payload) return false;
  return true;
}

namespace {

// Walks the overlap of `dst_box` and `src_box` as contiguous runs: trailing
// axes both boxes span completely fold into one run (a Dense3D RGB tile read
// from a slide moves whole 3*w-byte rows, not 3-byte channel triples).
// fn(dst_offset, src_offset, run_bytes).
template <typename Fn>
void walk_overlap(const BoundingBox& dst_box, const BoundingBox& src_box, std::size_t elem, Fn fn) {
  const auto ov = dst_box.intersected(src_box);
  if (!ov) return;
  const int d = ov->dims();
  int first = d - 1;  // runs span axes first..d-1
  while (first > 0 && ov->extent(first) == dst_box.extent(first) &&
         ov->extent(first) == src_box.extent(first))
    --first;
  std::size_t run = elem;
  for (int a = first; a < d; ++a) run *= std::size_t(ov->extent(a));
  std::array<std::int64_t, BoundingBox::kMaxDims> p{};
  for (int a = 0; a < d; ++a) p[a] = ov->lo(a);
  auto offset = [&](const BoundingBox& b) {
    std::int64_t o = 0;
    for (int a = 0; a < d; ++a) o = o * b.extent(a) + (p[a] - b.lo(a));
    return std::size_t(o) * elem;
  };
  for (;;) {
    fn(offset(dst_box), offset(src_box), run);
    int a = first - 1;
    while (a >= 0 && ++p[a] > ov->hi(a)) {
      p[a] = ov->lo(a);
      --a;
    }
    if (a < 0) break;
  }
}

}  // namespace

void copy_box_overlap(std::span<std::uint8_t> dst, const BoundingBox& dst_box,
                      std::span<const std::uint8_t> src, const BoundingBox& src_box,
                      std::size_t elem) {
  walk_overlap(dst_box, src_box, elem, [&](std::size_t od, std::size_t os, std::size_t n) {
    std::memcpy(dst.data() + od, src.data() + os, n);
  });
}

void fill_box_overlap(std::span<std::uint8_t> dst, const BoundingBox& dst_box,
                      const BoundingBox& box, std::uint8_t value) {
  walk_overlap(dst_box, box, 1, [&](std::size_t od, std::size_t, std::size_t n) {
    std::memset(dst.data() + od, value, n);
  });
}

// ---- RegionTemplate -------------------------------------------------------------

DataRegion& RegionTemplate::insert_data_region(DataRegion region) {
  // region_template.cpp:19-29: the region goes in first, then the template box
  // is folded — a box of another rank throws DimensionError from the union
  // and leaves the region inserted (the reference's observable behaviour)
  const DataRegionId id = region.id();
  if (regions_.count(id)) throw DuplicateRegionError("duplicate region " + id.to_string());
  DataRegion& r = regions_.emplace(id, std::move(region)).first->second;
  if (!r.bbox().empty()) bbox_ = bbox_.empty() ? r.bbox() : bbox_.unioned(r.bbox());
  return r;
}

const DataRegion* RegionTemplate::get_data_region(const DataRegionId& id) const {
  auto it = regions_.find(id);
  return it == regions_.end() ? nullptr : &it->second;
}

DataRegion* RegionTemplate::get_data_region(const DataRegionId& id) {
  auto it = regions_.find(id);
  return it == regions_.end() ? nullptr : &it->second;
}

const DataRegion* RegionTemplate::get_newest(const std::string& ns, const std::string& key,
                                             const std::string& type_tag) const {
  const DataRegion* best = nullptr;
  for (const auto& [id, r] : regions_) {
    if (id.ns != ns || id.key != key || id.type_tag != type_tag) continue;
    if (!best || std::tie(id.timestamp, id.version) >
                     std::tie(best->id().timestamp, best->id().version))
      best = &r;
  }
  return best;
}

bool RegionTemplate::remove_data_region(const DataRegionId& id) {
  if (!regions_.erase(id)) return false;
  refold();
  return true;
}

void RegionTemplate::refold() {
  bbox_ = BoundingBox();
  for (const auto& [id, r] : regions_) {
    if (r.bbox().empty()) continue;
    bbox_ = bbox_.empty() ? r.bbox() : bbox_.unioned(r.bbox());
  }
}

}  // namespace rt
