// Little-endian field codec shared by the two byte formats the host layer
// persists stage outputs in: RTP1 template packs (pack.cpp) and RTS1 write
// sessions (session.cpp).  The field tables are in DESIGN.md §8; the reference
// fixes the same bytes in its pack.cpp:33-132 and disk_store.cpp:150-217.
//
// Sink appends fields to a byte vector.  Source walks a bounded byte window
// and names the format and the field in every DecodeError it raises, so a
// corrupt file reports where it broke ("RTS1 record 3: payload: needs 4096
// bytes, 17 left").
#pragma once

#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <string_view>
#include <type_traits>
#include <vector>

#include "rt/region.hpp"

namespace rt::wire {

template <typename T, bool IsEnum>
struct Repr {
  using type = T;
};
template <typename T>
struct Repr<T, true> {
  using type = std::underlying_type_t<T>;
};

class Sink {
 public:
  template <typename T>
  void put(T v) {
    static_assert(std::is_integral_v<T> || std::is_enum_v<T>);
    using U = std::make_unsigned_t<typename Repr<T, std::is_enum_v<T>>::type>;
    const U u = static_cast<U>(v);
    std::uint8_t le[sizeof(U)];
    for (std::size_t i = 0; i < sizeof(U); ++i) le[i] = std::uint8_t(std::uint64_t(u) >> (8 * i));
    bytes_.insert(bytes_.end(), le, le + sizeof(U));
  }
  void put_text(std::string_view s) {
    put(std::uint32_t(s.size()));
    bytes_.insert(bytes_.end(), s.begin(), s.end());
  }
  // rank u8, then every lower corner, then every upper corner (i64 each)
  void put_extent(const BoundingBox& b) {
    put(std::uint8_t(b.dims()));
    for (int a = 0; a < b.dims(); ++a) put(b.lo(a));
    for (int a = 0; a < b.dims(); ++a) put(b.hi(a));
  }
  void put_blob(const std::uint8_t* p, std::size_t n) { bytes_.insert(bytes_.end(), p, p + n); }
  std::size_t size() const { return bytes_.size(); }
  std::vector<std::uint8_t>& bytes() { return bytes_; }

 private:
  std::vector<std::uint8_t> bytes_;
};

class Source {
 public:
  Source(std::span<const std::uint8_t> window, std::string where)
      : w_(window), where_(std::move(where)) {}

  std::size_t offset() const { return at_; }
  std::size_t left() const { return w_.size() - at_; }
  void relabel(std::string where) { where_ = std::move(where); }

  template <typename T>
  T get(const char* field) {
    static_assert(std::is_integral_v<T>);
    take(sizeof(T), field);
    std::uint64_t v = 0;
    for (std::size_t i = 0; i < sizeof(T); ++i) v |= std::uint64_t(w_[at_ - sizeof(T) + i]) << (8 * i);
    return static_cast<T>(v);
  }
  // An enum stored as one byte whose largest legal value is `last`.
  template <typename E>
  E get_enum(const char* field, E last) {
    const std::uint8_t raw = get<std::uint8_t>(field);
    if (raw > std::uint8_t(last))
      fail(std::string(field) + ": value " + std::to_string(raw) + " is not defined (max " +
           std::to_string(int(last)) + ")");
    return E(raw);
  }
  std::string get_text(const char* field) {
    const std::uint32_t n = get<std::uint32_t>(field);
    const std::uint8_t* p = take(n, field);
    return std::string(reinterpret_cast<const char*>(p), n);
  }
  BoundingBox get_extent(const char* field) {
    const int rank = get<std::uint8_t>(field);
    if (rank > BoundingBox::kMaxDims)
      fail(std::string(field) + ": rank " + std::to_string(rank) + " exceeds " +
           std::to_string(BoundingBox::kMaxDims));
    if (rank == 0) return BoundingBox();
    std::int64_t corner[2][BoundingBox::kMaxDims];
    for (auto& c : corner)
      for (int a = 0; a < rank; ++a) c[a] = get<std::int64_t>(field);
    return BoundingBox(rank, corner[0], corner[1]);
  }
  // A view of the next n bytes (no copy).
  std::span<const std::uint8_t> get_blob(std::uint64_t n, const char* field) {
    const std::uint8_t* p = take(n, field);
    return {p, std::size_t(n)};
  }
  void jump(std::uint64_t off, const char* what) {
    if (off > w_.size())
      fail(std::string(what) + ": offset " + std::to_string(off) + " lies beyond the " +
           std::to_string(w_.size()) + "-byte window");
    at_ = std::size_t(off);
  }
  [[noreturn]] void fail(const std::string& msg) const { throw DecodeError(where_ + ": " + msg); }

 private:
  const std::uint8_t* take(std::uint64_t n, const char* field) {
    if (n > left())
      fail(std::string(field) + ": needs " + std::to_string(n) + " bytes, " +
           std::to_string(left()) + " left");
    const std::uint8_t* p = w_.data() + at_;
    at_ += std::size_t(n);
    return p;
  }
  std::span<const std::uint8_t> w_;
  std::size_t at_ = 0;
  std::string where_;
};

// The identity prefix both formats open a region record with:
// ns, key, type_tag (text) | timestamp, version (i64) | kind, element (u8).
struct Identity {
  DataRegionId id;
  RegionKind kind = RegionKind::kDense2D;
  ElementKind element = ElementKind::kU8;
};

inline void put_identity(Sink& s, const DataRegionId& id, RegionKind kind, ElementKind element) {
  s.put_text(id.ns);
  s.put_text(id.key);
  s.put_text(id.type_tag);
  s.put(id.timestamp);
  s.put(id.version);
  s.put(kind);
  s.put(element);
}

inline Identity get_identity(Source& in) {
  Identity r;
  r.id.ns = in.get_text("namespace");
  r.id.key = in.get_text("key");
  r.id.type_tag = in.get_text("type tag");
  r.id.timestamp = in.get<std::int64_t>("timestamp");
  r.id.version = in.get<std::int64_t>("version");
  r.kind = in.get_enum("region kind", RegionKind::kPolygon);
  r.element = in.get_enum("element kind", ElementKind::kF64);
  return r;
}

}  // namespace rt::wire
