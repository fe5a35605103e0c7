// RTP1 pack / unpack (see rt/pack.hpp; reference pack.cpp:33-121 defines the
// same byte layout through its wire::Writer / wire::Reader).
#include "rt/pack.hpp"

#include <cstring>
#include <string>

namespace rt {
namespace {

class Out {
 public:
  void u8(std::uint8_t v) { b_.push_back(v); }
  void le(std::uint64_t v, int n) {
    for (int i = 0; i < n; ++i) b_.push_back(std::uint8_t(v >> (8 * i)));
  }
  void u32(std::uint32_t v) { le(v, 4); }
  void u64(std::uint64_t v) { le(v, 8); }
  void i64(std::int64_t v) { le(std::uint64_t(v), 8); }
  void str(const std::string& s) {
    u32(std::uint32_t(s.size()));
    b_.insert(b_.end(), s.begin(), s.end());
  }
  void raw(const Bytes& p) { b_.insert(b_.end(), p.begin(), p.end()); }
  void box(const BoundingBox& b) {
    u8(std::uint8_t(b.dims()));
    for (int a = 0; a < b.dims(); ++a) i64(b.lo(a));
    for (int a = 0; a < b.dims(); ++a) i64(b.hi(a));
  }
  std::vector<std::uint8_t> take() { return std::move(b_); }

 private:
  std::vector<std::uint8_t> b_;
};

class In {
 public:
  explicit In(std::span<const std::uint8_t> s) : s_(s) {}
  bool at_end() const { return pos_ == s_.size(); }
  std::uint64_t le(int n) {
    need(std::uint64_t(n));
    std::uint64_t v = 0;
    for (int i = 0; i < n; ++i) v |= std::uint64_t(s_[pos_++]) << (8 * i);
    return v;
  }
  std::uint8_t u8() { return std::uint8_t(le(1)); }
  std::uint32_t u32() { return std::uint32_t(le(4)); }
  std::uint64_t u64() { return le(8); }
  std::int64_t i64() { return std::int64_t(le(8)); }
  std::string str() {
    const std::uint32_t n = u32();
    need(n);
    std::string out(reinterpret_cast<const char*>(s_.data() + pos_), n);
    pos_ += n;
    return out;
  }
  Bytes raw(std::uint64_t n) {
    need(n);
    Bytes out(s_.begin() + std::ptrdiff_t(pos_),
                                  s_.begin() + std::ptrdiff_t(pos_ + n));
    pos_ += n;
    return out;
  }
  BoundingBox box() {
    const int dims = u8();
    if (dims == 0) return BoundingBox();
    if (dims > BoundingBox::kMaxDims) throw DecodeError("bounding box rank out of range");
    std::int64_t lo[BoundingBox::kMaxDims], hi[BoundingBox::kMaxDims];
    for (int a = 0; a < dims; ++a) lo[a] = i64();
    for (int a = 0; a < dims; ++a) hi[a] = i64();
    return BoundingBox(dims, lo, hi);
  }

 private:
  void need(std::uint64_t n) const {
    if (n > s_.size() - pos_) throw DecodeError("buffer truncated");
  }
  std::span<const std::uint8_t> s_;
  std::size_t pos_ = 0;
};

std::uint8_t enum_byte(std::uint8_t raw, std::uint8_t max, const char* what) {
  if (raw > max) throw DecodeError(std::string("bad enum value for ") + what);
  return raw;
}

RegionTemplate decode(std::span<const std::uint8_t> bytes) {
  In in(bytes);
  if (in.u32() != kPackMagic) throw DecodeError("bad magic");
  const std::uint8_t flags = in.u8();
  if (flags > 1) throw DecodeError("bad flags");
  RegionTemplate t(in.str());
  const BoundingBox declared = in.box();
  const std::uint32_t nregions = in.u32();
  for (std::uint32_t k = 0; k < nregions; ++k) {
    DataRegionId id;
    id.ns = in.str();
    id.key = in.str();
    id.type_tag = in.str();
    id.timestamp = in.i64();
    id.version = in.i64();
    const auto kind = RegionKind(enum_byte(in.u8(), 4, "region kind"));
    const auto elem = ElementKind(enum_byte(in.u8(), 4, "element kind"));
    const auto io = IoMode(enum_byte(in.u8(), 2, "io mode"));
    const bool lazy = in.u8() != 0;
    const bool materialized = in.u8() != 0;
    const BoundingBox box = in.box();
    const BoundingBox roi = in.box();
    std::string binding = in.str();
    DataRegion r(std::move(id), kind, elem, box);
    r.set_roi(roi);
    r.set_io_mode(io);
    r.set_lazy(lazy);
    r.set_storage_binding(std::move(binding));
    const std::uint32_t nchunks = in.u32();
    for (std::uint32_t c = 0; c < nchunks; ++c) {
      const std::uint64_t wire_id = in.u64();
      const BoundingBox cbox = in.box();
      const std::uint64_t len = in.u64();
      r.put_chunk(cbox, in.raw(len)).chunk_id = wire_id;  // keep the sender's id
    }
    if (materialized != r.materialized())
      throw DecodeError("materialized flag disagrees with chunk payload");
    t.insert_data_region(std::move(r));
  }
  if (!in.at_end()) throw DecodeError("trailing bytes after template");
  if (!(t.bbox() == declared)) throw DecodeError("declared template box disagrees with regions");
  return t;
}

}  // namespace

std::vector<std::uint8_t> pack_template(const RegionTemplate& t, bool include_payload) {
  Out out;
  out.u32(kPackMagic);
  out.u8(include_payload ? 1 : 0);
  out.str(t.name());
  out.box(t.bbox());
  out.u32(std::uint32_t(t.regions().size()));
  for (const auto& [id, r] : t.regions()) {
    out.str(id.ns);
    out.str(id.key);
    out.str(id.type_tag);
    out.i64(id.timestamp);
    out.i64(id.version);
    out.u8(std::uint8_t(r.kind()));
    out.u8(std::uint8_t(r.element_kind()));
    out.u8(std::uint8_t(r.io_mode()));
    out.u8(r.lazy() ? 1 : 0);
    out.u8(include_payload && r.materialized() ? 1 : 0);
    out.box(r.bbox());
    out.box(r.roi());
    out.str(r.storage_binding());
    if (!include_payload) {
      out.u32(0);
      continue;
    }
    out.u32(std::uint32_t(r.chunks().size()));
    for (const auto& [cbox, chunk] : r.chunks()) {
      out.u64(chunk.chunk_id);
      out.box(cbox);
      out.u64(chunk.payload.size());
      out.raw(chunk.payload);
    }
  }
  return out.take();
}

RegionTemplate unpack_template(std::span<const std::uint8_t> bytes) {
  try {
    return decode(bytes);
  } catch (const DecodeError&) {
    throw;
  } catch (const Error& e) {
    // a structural violation reached through decoded bytes is corruption
    throw DecodeError(std::string("corrupt template buffer: ") + e.what());
  }
}

}  // namespace rt
