// Write-session files "RTS1" (the reference's disk_store.hpp / .cpp:150-217):
// how staged regions — e.g. a stage's Mask / Labels / Features outputs — land
// on disk, byte-compatible with the reference's DiskStore sessions.
//
//   file   := magic u32 ("RTS1") | session_seq u64 | count u32 | record*
//             | offset u64 * count | footer_offset u64 | end_magic u32 ("RTSE")
//   record := ns str | key str | type_tag str | timestamp i64 | version i64
//             | kind u8 | element_kind u8 | box | seq u64 | payload_len u64
//             | payload                  (integers little-endian, str/box as RTP1)
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "rt/region.hpp"

namespace rt {

struct DiskRecord {
  DataRegionId id;
  RegionKind kind = RegionKind::kDense2D;
  ElementKind element_kind = ElementKind::kU8;
  BoundingBox box;
  std::uint64_t seq = 0;
  Bytes payload;
};

inline constexpr std::uint32_t kSessionMagic = 0x31535452u;     // "RTS1"
inline constexpr std::uint32_t kSessionEndMagic = 0x45535452u;  // "RTSE"

// Writes one session file; returns each record's byte offset.  IoError when
// the file cannot be written.
std::vector<std::uint64_t> write_session_file(const std::string& path, std::uint64_t session_seq,
                                              const std::vector<DiskRecord>& records);
// IoError when the file cannot be opened, DecodeError on corruption.
std::vector<DiskRecord> read_session_file(const std::string& path);
DiskRecord read_record_at(const std::string& path, std::uint64_t offset);

// Every chunk of the template's materialised regions as a record (the
// records a DiskStore write session would flush for them), seq = seq0, ...
std::vector<DiskRecord> template_records(const RegionTemplate& t, std::uint64_t seq0);

}  // namespace rt
