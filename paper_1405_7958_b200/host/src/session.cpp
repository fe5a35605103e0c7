// RTS1 session files (see rt/session.hpp).
#include "rt/session.hpp"

#include <fstream>

namespace rt {
namespace {

void le(std::string& o, std::uint64_t v, int n) {
  for (int i = 0; i < n; ++i) o.push_back(char(v >> (8 * i)));
}
void put_str(std::string& o, const std::string& s) {
  le(o, s.size(), 4);
  o += s;
}
void put_box(std::string& o, const BoundingBox& b) {
  o.push_back(char(b.dims()));
  for (int a = 0; a < b.dims(); ++a) le(o, std::uint64_t(b.lo(a)), 8);
  for (int a = 0; a < b.dims(); ++a) le(o, std::uint64_t(b.hi(a)), 8);
}

// Whole file in memory; every read is bounds-checked against it.
class FileBytes {
 public:
  explicit FileBytes(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open session file: " + path);
    f.seekg(0, std::ios::end);
    data_.resize(std::size_t(f.tellg()));
    f.seekg(0);
    if (!data_.empty()) f.read(data_.data(), std::streamsize(data_.size()));
  }
  std::uint64_t size() const { return data_.size(); }
  void seek(std::uint64_t off) {
    if (off > data_.size()) throw DecodeError("session file offset out of range");
    pos_ = off;
  }
  std::uint64_t get(int n) {
    if (std::uint64_t(n) > data_.size() - pos_) throw DecodeError("session file truncated");
    std::uint64_t v = 0;
    for (int i = 0; i < n; ++i) v |= std::uint64_t(std::uint8_t(data_[pos_++])) << (8 * i);
    return v;
  }
  std::string str() {
    const std::uint64_t n = get(4);
    if (n > data_.size()) throw DecodeError("session file string overruns");
    if (n > data_.size() - pos_) throw DecodeError("session file truncated");
    std::string s(data_.data() + pos_, n);
    pos_ += n;
    return s;
  }
  Bytes raw(std::uint64_t n) {
    if (n > data_.size()) throw DecodeError("session file payload overruns");
    if (n > data_.size() - pos_) throw DecodeError("session file truncated");
    Bytes b(data_.begin() + std::ptrdiff_t(pos_),
                                data_.begin() + std::ptrdiff_t(pos_ + n));
    pos_ += n;
    return b;
  }
  BoundingBox box() {
    const int dims = int(get(1));
    if (dims == 0) return BoundingBox();
    if (dims > BoundingBox::kMaxDims) throw DecodeError("session file box rank out of range");
    std::int64_t lo[BoundingBox::kMaxDims], hi[BoundingBox::kMaxDims];
    for (int a = 0; a < dims; ++a) lo[a] = std::int64_t(get(8));
    for (int a = 0; a < dims; ++a) hi[a] = std::int64_t(get(8));
    return BoundingBox(dims, lo, hi);
  }

 private:
  std::string data_;
  std::uint64_t pos_ = 0;
};

DiskRecord record(FileBytes& in) {
  DiskRecord r;
  r.id.ns = in.str();
  r.id.key = in.str();
  r.id.type_tag = in.str();
  r.id.timestamp = std::int64_t(in.get(8));
  r.id.version = std::int64_t(in.get(8));
  const auto kind = std::uint8_t(in.get(1)), elem = std::uint8_t(in.get(1));
  if (kind > 4 || elem > 4) throw DecodeError("session record bad enum");
  r.kind = RegionKind(kind);
  r.element_kind = ElementKind(elem);
  r.box = in.box();
  r.seq = in.get(8);
  r.payload = in.raw(in.get(8));
  return r;
}

}  // namespace

std::vector<std::uint64_t> write_session_file(const std::string& path, std::uint64_t session_seq,
                                              const std::vector<DiskRecord>& records) {
  std::string o;
  le(o, kSessionMagic, 4);
  le(o, session_seq, 8);
  le(o, records.size(), 4);
  std::vector<std::uint64_t> offsets;
  offsets.reserve(records.size());
  for (const DiskRecord& r : records) {
    offsets.push_back(o.size());
    put_str(o, r.id.ns);
    put_str(o, r.id.key);
    put_str(o, r.id.type_tag);
    le(o, std::uint64_t(r.id.timestamp), 8);
    le(o, std::uint64_t(r.id.version), 8);
    o.push_back(char(r.kind));
    o.push_back(char(r.element_kind));
    put_box(o, r.box);
    le(o, r.seq, 8);
    le(o, r.payload.size(), 8);
    o.append(reinterpret_cast<const char*>(r.payload.data()), r.payload.size());
  }
  const std::uint64_t footer = o.size();
  for (std::uint64_t off : offsets) le(o, off, 8);
  le(o, footer, 8);
  le(o, kSessionEndMagic, 4);
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f || !f.write(o.data(), std::streamsize(o.size())))
    throw IoError("cannot write session file: " + path);
  return offsets;
}

std::vector<DiskRecord> read_session_file(const std::string& path) {
  FileBytes in(path);
  if (in.size() < 4 + 8 + 4 + 8 + 4) throw DecodeError("session file too short: " + path);
  if (in.get(4) != kSessionMagic) throw DecodeError("session file bad magic");
  in.get(8);  // session seq
  const std::uint32_t count = std::uint32_t(in.get(4));
  in.seek(in.size() - 12);
  const std::uint64_t footer = in.get(8);
  if (in.get(4) != kSessionEndMagic) throw DecodeError("session file bad end magic");
  in.seek(footer);
  std::vector<std::uint64_t> offsets(count);
  for (auto& off : offsets) off = in.get(8);
  std::vector<DiskRecord> out;
  out.reserve(count);
  for (std::uint64_t off : offsets) {
    in.seek(off);
    out.push_back(record(in));
  }
  return out;
}

DiskRecord read_record_at(const std::string& path, std::uint64_t offset) {
  FileBytes in(path);
  in.seek(offset);
  return record(in);
}

std::vector<DiskRecord> template_records(const RegionTemplate& t, std::uint64_t seq0) {
  std::vector<DiskRecord> out;
  for (const auto& [id, r] : t.regions()) {
    if (!r.materialized()) continue;
    for (const auto& [box, chunk] : r.chunks())
      out.push_back(DiskRecord{id, r.kind(), r.element_kind(), box, seq0++, chunk.payload});
  }
  return out;
}

}  // namespace rt
