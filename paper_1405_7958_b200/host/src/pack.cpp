// RTP1 template packs (rt/pack.hpp; field table in DESIGN.md §8).
//
// Decoding is two-phase: parse() turns the bytes into a flat description
// whose payloads are views into the caller's buffer (every length and enum is
// checked here, nothing is allocated for payloads), then assemble() builds the
// RegionTemplate and checks what only the assembled object can tell (dense
// payload lengths, the materialised flag, the declared box).  The byte layout
// is the reference's (pack.cpp:33-132); the code structure is not.
#include "rt/pack.hpp"

#include <string>

#include "wire_codec.hpp"

namespace rt {
namespace {

constexpr std::uint8_t kFlagPayloads = 0x01;

struct ChunkView {
  std::uint64_t id;
  BoundingBox box;
  std::span<const std::uint8_t> bytes;
};

struct RegionView {
  wire::Identity ident;
  IoMode io = IoMode::kInput;
  bool lazy = false, materialized = false;
  BoundingBox box, roi;
  std::string binding;
  std::vector<ChunkView> chunks;
};

struct TemplateView {
  std::string name;
  BoundingBox declared;
  std::vector<RegionView> regions;
};

TemplateView parse(std::span<const std::uint8_t> bytes) {
  wire::Source in(bytes, "RTP1 header");
  const auto magic = in.get<std::uint32_t>("magic");
  if (magic != kPackMagic) in.fail("not an RTP1 pack (magic " + std::to_string(magic) + ")");
  const auto flags = in.get<std::uint8_t>("flags");
  if (flags & ~kFlagPayloads) in.fail("undefined flag bits " + std::to_string(flags));

  TemplateView t;
  t.name = in.get_text("template name");
  t.declared = in.get_extent("template box");
  const auto count = in.get<std::uint32_t>("region count");
  // a region record takes at least 43 bytes: four empty texts, two i64, five
  // u8, two rank-0 extents and a chunk count
  if (std::uint64_t(count) * 43 > in.left())
    in.fail("region count " + std::to_string(count) + " cannot fit in " +
            std::to_string(in.left()) + " bytes");
  t.regions.resize(count);
  for (std::uint32_t k = 0; k < count; ++k) {
    in.relabel("RTP1 region " + std::to_string(k));
    RegionView& r = t.regions[k];
    r.ident = wire::get_identity(in);
    r.io = in.get_enum("io mode", IoMode::kInputOutput);
    r.lazy = in.get<std::uint8_t>("lazy") != 0;
    r.materialized = in.get<std::uint8_t>("materialized") != 0;
    r.box = in.get_extent("box");
    r.roi = in.get_extent("roi");
    r.binding = in.get_text("storage binding");
    const auto nchunks = in.get<std::uint32_t>("chunk count");
    for (std::uint32_t c = 0; c < nchunks; ++c) {
      ChunkView v;
      v.id = in.get<std::uint64_t>("chunk id");
      v.box = in.get_extent("chunk box");
      v.bytes = in.get_blob(in.get<std::uint64_t>("payload length"), "payload");
      r.chunks.push_back(v);
    }
  }
  if (in.left() != 0) in.fail(std::to_string(in.left()) + " bytes follow the last region");
  return t;
}

RegionTemplate assemble(const TemplateView& v) {
  RegionTemplate t(v.name);
  for (const RegionView& rv : v.regions) {
    DataRegion r(rv.ident.id, rv.ident.kind, rv.ident.element, rv.box);
    r.set_roi(rv.roi);
    r.set_io_mode(rv.io);
    r.set_lazy(rv.lazy);
    r.set_storage_binding(rv.binding);
    for (const ChunkView& c : rv.chunks)
      r.put_chunk(c.box, Bytes(c.bytes.begin(), c.bytes.end())).chunk_id = c.id;
    if (r.materialized() != rv.materialized)
      throw DecodeError("RTP1 region " + rv.ident.id.to_string() + " says materialized=" +
                        std::to_string(int(rv.materialized)) + " but carries " +
                        std::to_string(rv.chunks.size()) + " chunks");
    t.insert_data_region(std::move(r));
  }
  if (t.bbox() != v.declared)
    throw DecodeError("RTP1 template box " + v.declared.to_string() +
                      " differs from its regions' union " + t.bbox().to_string());
  return t;
}

}  // namespace

std::vector<std::uint8_t> pack_template(const RegionTemplate& t, bool include_payload) {
  wire::Sink out;
  out.put(kPackMagic);
  out.put(std::uint8_t(include_payload ? kFlagPayloads : 0));
  out.put_text(t.name());
  out.put_extent(t.bbox());
  out.put(std::uint32_t(t.regions().size()));
  for (const auto& [id, r] : t.regions()) {
    const bool ship = include_payload && r.materialized();
    wire::put_identity(out, id, r.kind(), r.element_kind());
    out.put(r.io_mode());
    out.put(std::uint8_t(r.lazy()));
    out.put(std::uint8_t(ship));
    out.put_extent(r.bbox());
    out.put_extent(r.roi());
    out.put_text(r.storage_binding());
    // metadata-only packs send no chunks even for materialised regions
    out.put(std::uint32_t(include_payload ? r.chunks().size() : 0));
    if (!include_payload) continue;
    for (const auto& [box, c] : r.chunks()) {
      out.put(c.chunk_id);
      out.put_extent(box);
      out.put(std::uint64_t(c.payload.size()));
      out.put_blob(c.payload.data(), c.payload.size());
    }
  }
  return std::move(out.bytes());
}

RegionTemplate unpack_template(std::span<const std::uint8_t> bytes) {
  try {
    return assemble(parse(bytes));
  } catch (const DecodeError&) {
    throw;
  } catch (const Error& e) {
    // the bytes describe an object the containers reject (inverted box,
    // bad dense length, duplicate id, rank mix): that is a corrupt pack
    throw DecodeError(std::string("RTP1 pack describes an invalid template: ") + e.what());
  }
}

}  // namespace rt
