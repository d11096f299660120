// host_format.h — host side of the PcRecord format: header, index, page
// headers, writer.  Mirrors format.hpp / metadata.hpp of the reference
// (proj/core/include/pcpipe/) with B200-pipeline-oriented types.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "pcp_internal.h"

namespace pcp {

// Internal exception; converted to an int status at the C ABI.
struct Fail : std::runtime_error {
  int32_t code;
  Fail(int32_t c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int32_t code, const std::string& msg) { throw Fail(code, msg); }
const char* errc_name(int32_t status);  // errors.cpp:5-50 names

struct FieldSpec {
  std::string name;
  int32_t kind = kBytes;
  std::vector<uint32_t> shape;
  uint32_t elems() const {
    uint32_t n = 1;
    for (auto d : shape) n *= d;
    return n;
  }
};

struct Group {  // GroupDesc (format.hpp:110-125)
  uint32_t group_id = 0, slice = 0;
  uint64_t first_sample = 0;
  uint32_t sample_count = 0;
  uint64_t scalar_off = 0, scalar_len = 0, block_off = 0, block_len = 0;
  std::vector<std::array<uint64_t, 2>> blob_ranges;
  std::vector<std::vector<uint64_t>> blob_lens;
};

struct Header {  // FileHeader (format.hpp:127-146)
  uint16_t version = 1;
  uint64_t total_size_bytes = 0;
  uint32_t scalar_page_size_bytes = 0, block_page_size_bytes = 0;
  std::vector<FieldSpec> schema;
  std::vector<std::string> slice_paths;
  std::vector<Group> groups;
  uint64_t header_bytes = 0;  // magic+version+len+json of the primary slice
};

// MetadataEntry (metadata.hpp:13-24) reduced to what the device path needs.
struct Entry {
  uint32_t shard_id = 0;  // slice
  uint32_t group_id = 0;
  uint32_t group_index = 0;  // index into Header::groups
  uint32_t row = 0;
  uint64_t blob_start = 0, blob_end = 0;
};

struct PageHead {  // the 21-byte EncodedPage prefix (format.cpp:276-299)
  uint8_t flags = 0;
  uint64_t raw_len = 0, pay_len = 0;
  uint32_t crc = 0;
};

// read_header (format.cpp:612-653): magic, version, JSON, invariants, slice
// sizes.  Throws Fail with the reference's Errc.
Header read_header(const std::string& primary);
// The same from header bytes in memory (e.g. a streamed meta index), no
// slice-size checks (the slices are not local yet).
Header parse_header_bytes(const uint8_t* p, size_t n);
// build_index (metadata.cpp:20-52) for one header.
std::vector<Entry> build_index(const Header& h);
// Reads one slice's data area (whole file; primary minus its header).
std::vector<uint8_t> read_slice_data(const Header& h, const std::string& dir, uint32_t slice);

PageHead parse_page_head(const uint8_t* p, uint64_t avail);

// Host CRC-32 (zlib-compatible) and the reference's greedy LZ4 block
// compressor (lz4_block.cpp:33-103), used by the writer only.
uint32_t crc32_host(const uint8_t* p, size_t n);
std::vector<uint8_t> lz4_compress_host(const uint8_t* src, size_t n);

// write_dataset (format.cpp:499-610), byte-identical, groups encoded on
// n_threads host threads.
struct SampleIn {
  // per schema field: raw bytes of the value (bytes blob / packed numbers /
  // string characters)
  std::vector<std::vector<uint8_t>> values;
};
// device >= 0: the pages are encoded on that GPU (page_encode.cu), same bytes.
Header write_dataset(const std::vector<FieldSpec>& schema, const std::vector<SampleIn>& samples,
                     uint32_t slice_count, uint32_t group_size, const std::string& out_dir,
                     const std::string& stem, uint32_t n_threads, int device = -1);

std::vector<FieldSpec> schema_from_json(const std::string& json_text);

}  // namespace pcp
