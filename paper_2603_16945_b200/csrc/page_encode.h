// page_encode.h — batched PcRecord page encoder on the device (page_encode.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace pcp {

struct EncPage {
  uint64_t raw_off, raw_len;  // raw page bytes in the batch buffer
  uint64_t hash_off;          // first hash slot (positions < raw_len - 12)
  uint64_t vis_off;           // first visited-bitmap word
  uint64_t seq_off;           // first sequence slot
  uint64_t comp_off;          // compressed output offset
};
struct EncColumn {  // XOR-delta column (width 4) of a page: [off, off + len)
  uint64_t off, len;
  uint32_t page, pad;
};
struct EncSeq {  // one LZ4 sequence: literals [lit_start, +lit_len), then a match
  uint32_t lit_start, lit_len, match_len, offset;
};

struct EncArgs {
  uint32_t n_pages, n_cols;
  uint64_t raw_total, hash_total;
  const uint8_t* raw;      // raw pages
  uint8_t* work;           // post-delta pages (the stored-raw payload)
  const EncPage* pages;
  const EncColumn* cols;
  uint32_t *keys, *keys_alt, *vals, *vals_alt;  // [hash_total]
  const int* hash_begin;   // [n_pages] segment bounds for the sort
  const int* hash_end;
  uint32_t* prev;          // [hash_total]
  uint32_t* visited;       // [n_pages][65536] parse hash tables (position + 1)
  uint64_t visited_bytes;
  EncSeq* seqs;
  uint32_t* n_seqs;        // [n_pages]
  uint8_t* comp;           // compressed pages
  uint64_t* comp_len;      // [n_pages]
  uint32_t* crc;           // [n_pages] payload CRC
  const uint32_t* shift_tab;
  void* cub;
  size_t cub_bytes;
};

struct EncScratchSizes {
  uint64_t keys, vals, prev, visited, seqs, comp, cub;
};
EncScratchSizes enc_scratch_sizes(uint64_t raw_total, uint64_t hash_total, uint32_t n_pages);
cudaError_t launch_encode_pages(const EncArgs& e, cudaStream_t st);

}  // namespace pcp
