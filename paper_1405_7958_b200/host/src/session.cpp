// RTS1 write-session files (rt/session.hpp; field table in DESIGN.md §8).
//
// The file is loaded whole and decoded trailer-first: the trailer fixes the
// record area [16, index) and the index of record offsets; every record is
// then decoded inside the record area only, so a corrupt offset can never
// read the index or the trailer as record bytes.  The byte layout is the
// reference's (disk_store.cpp:150-217); the code structure is not.
#include "rt/session.hpp"

#include <fstream>
#include <iterator>

#include "wire_codec.hpp"

namespace rt {
namespace {

constexpr std::size_t kHeaderBytes = 4 + 8 + 4;  // magic, session seq, record count
constexpr std::size_t kTrailerBytes = 8 + 4;     // index offset, end magic

std::vector<std::uint8_t> load(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw IoError("session file " + path + " could not be opened for reading");
  return std::vector<std::uint8_t>(std::istreambuf_iterator<char>(f), {});
}

void put_record(wire::Sink& out, const DiskRecord& r) {
  wire::put_identity(out, r.id, r.kind, r.element_kind);
  out.put_extent(r.box);
  out.put(r.seq);
  out.put(std::uint64_t(r.payload.size()));
  out.put_blob(r.payload.data(), r.payload.size());
}

DiskRecord get_record(wire::Source& in) {
  const wire::Identity ident = wire::get_identity(in);
  DiskRecord r;
  r.id = ident.id;
  r.kind = ident.kind;
  r.element_kind = ident.element;
  r.box = in.get_extent("box");
  r.seq = in.get<std::uint64_t>("sequence");
  const std::span<const std::uint8_t> p = in.get_blob(in.get<std::uint64_t>("payload length"), "payload");
  r.payload.assign(p.begin(), p.end());
  return r;
}

// Where the records of a decoded file lie.
struct Layout {
  std::span<const std::uint8_t> records;  // bytes [0, index): offsets index into this window
  std::vector<std::uint64_t> offsets;
};

Layout layout(std::span<const std::uint8_t> file, const std::string& path) {
  if (file.size() < kHeaderBytes + kTrailerBytes)
    throw DecodeError("RTS1 file " + path + " holds " + std::to_string(file.size()) +
                      " bytes, fewer than an empty session");
  wire::Source head(file.first(kHeaderBytes), "RTS1 header of " + path);
  if (head.get<std::uint32_t>("magic") != kSessionMagic) head.fail("not an RTS1 session file");
  head.get<std::uint64_t>("session sequence");
  const auto count = head.get<std::uint32_t>("record count");

  wire::Source tail(file.last(kTrailerBytes), "RTS1 trailer of " + path);
  const auto index = tail.get<std::uint64_t>("index offset");
  if (tail.get<std::uint32_t>("end magic") != kSessionEndMagic) tail.fail("end marker missing");
  const std::uint64_t body_end = file.size() - kTrailerBytes;
  if (index < kHeaderBytes || index > body_end || (body_end - index) / 8 < count)
    tail.fail("index of " + std::to_string(count) + " offsets at " + std::to_string(index) +
              " does not fit between the header and the trailer");

  Layout out;
  out.records = file.first(std::size_t(index));
  wire::Source idx(file.subspan(std::size_t(index), std::size_t(body_end - index)),
                   "RTS1 index of " + path);
  out.offsets.resize(count);
  for (auto& off : out.offsets) off = idx.get<std::uint64_t>("record offset");
  return out;
}

}  // namespace

std::vector<std::uint64_t> write_session_file(const std::string& path, std::uint64_t session_seq,
                                              const std::vector<DiskRecord>& records) {
  wire::Sink out;
  out.put(kSessionMagic);
  out.put(session_seq);
  out.put(std::uint32_t(records.size()));
  std::vector<std::uint64_t> offsets;
  offsets.reserve(records.size());
  for (const DiskRecord& r : records) {
    offsets.push_back(out.size());
    put_record(out, r);
  }
  const std::uint64_t index = out.size();
  for (const std::uint64_t off : offsets) out.put(off);
  out.put(index);
  out.put(kSessionEndMagic);

  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  const auto& b = out.bytes();
  f.write(reinterpret_cast<const char*>(b.data()), std::streamsize(b.size()));
  if (!f.flush()) throw IoError("session file " + path + " could not be written");
  return offsets;
}

std::vector<DiskRecord> read_session_file(const std::string& path) {
  const std::vector<std::uint8_t> file = load(path);
  const Layout lay = layout(file, path);
  std::vector<DiskRecord> out;
  out.reserve(lay.offsets.size());
  wire::Source in(lay.records, "");
  for (std::size_t k = 0; k < lay.offsets.size(); ++k) {
    in.relabel("RTS1 record " + std::to_string(k) + " of " + path);
    in.jump(lay.offsets[k], "record offset");
    out.push_back(get_record(in));
  }
  return out;
}

DiskRecord read_record_at(const std::string& path, std::uint64_t offset) {
  const std::vector<std::uint8_t> file = load(path);
  wire::Source in(file, "RTS1 record at " + std::to_string(offset) + " of " + path);
  in.jump(offset, "record offset");
  return get_record(in);
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
