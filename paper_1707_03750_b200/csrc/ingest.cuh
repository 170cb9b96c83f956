// ingest.cuh — device side of the GPU CSV ingest (ingest.cu) shared with the host driver (capi.cu).
#pragma once
#include <string>
#include <vector>

#include "common.cuh"

namespace itt {

// columns of interest, in the order the reference resolves them (ingest.hpp:205-222)
enum { kColStart = 0, kColDuration, kColSize, kColThroughput, kColDevice, kColStream, kColName, kIngestCols };
enum : uint8_t { kLineIgnore = 0, kLineRecord = 1, kLineSkip = 2 };
// skip reasons in the reference's check order (ingest.hpp:318-371)
enum : uint8_t { kSkipNone = 0, kSkipName, kSkipStart, kSkipDuration, kSkipStream, kSkipSize, kSkipThroughput };

struct LineOut {
  uint8_t status, reason, flags, pad_;
  uint32_t stream;
  int64_t start, dur, size;
  uint64_t name_b, name_e;  // raw field span of Name
  uint64_t dev_b, dev_e;    // raw field span of Device
  uint32_t name_first, name_len;  // trimmed, unescaped extent within the field
  uint32_t dev_first, dev_len;    // dev_len 0: "unknown"
  uint64_t dev_hash;
};

struct IngestArgs {
  const uint8_t* text;
  uint64_t len;
  const uint64_t* nl;  // newline positions
  uint64_t n_nl;
  uint64_t n_lines;
  uint64_t first_line;  // first line that may be a data row (after the header and units row)
  int col[kIngestCols];  // field index or -1
  int64_t start_factor, duration_factor, size_factor;
  LineOut* out;  // [n_lines - first_line]
};

// Parsed trace: columns in cudaMalloc'd device memory owned by the object (they outlive the
// call), records in source line order; host-side report.
struct ParsedCsv {
  uint64_t n = 0;
  int col[kIngestCols];
  int64_t* start = nullptr;
  int64_t* dur = nullptr;
  int64_t* size = nullptr;
  uint8_t* flags = nullptr;
  uint32_t* stream = nullptr;
  uint16_t* device = nullptr;
  uint64_t* name_off = nullptr;
  uint8_t* name_bytes = nullptr;
  std::vector<uint64_t> line;  // 1-based source line of each record (TraceRecord::row)
  std::vector<std::string> device_labels, warnings, skip_reason;
  std::vector<uint64_t> skip_line;
  uint64_t rows_total = 0, rows_parsed = 0, rows_skipped = 0;
  void alloc_columns(uint64_t cap) {
    ITT_CUDA(cudaMalloc(&start, cap * 8));
    ITT_CUDA(cudaMalloc(&dur, cap * 8));
    ITT_CUDA(cudaMalloc(&size, cap * 8));
    ITT_CUDA(cudaMalloc(&flags, cap));
    ITT_CUDA(cudaMalloc(&stream, cap * 4));
    ITT_CUDA(cudaMalloc(&device, cap * 2));
    ITT_CUDA(cudaMalloc(&name_off, (cap + 1) * 8));
  }
  void alloc_names(uint64_t bytes) { ITT_CUDA(cudaMalloc(&name_bytes, bytes + 16)); }
  void release() {
    for (void* p : {static_cast<void*>(start), static_cast<void*>(dur), static_cast<void*>(size),
                    static_cast<void*>(flags), static_cast<void*>(stream), static_cast<void*>(device),
                    static_cast<void*>(name_off), static_cast<void*>(name_bytes)})
      if (p) cudaFree(p);
    start = dur = size = nullptr;
    flags = nullptr, stream = nullptr, device = nullptr, name_off = nullptr, name_bytes = nullptr;
  }
};

// parse_trace_text (ingest.hpp:154-402) on the GPU; throws Error like the reference
void parse_csv(Ctx* c, const char* text, uint64_t len, const std::string& label, ParsedCsv& out);

__global__ void k_parse_lines(IngestArgs a);
__global__ void k_copy_names(const uint8_t* __restrict__ text, const LineOut* __restrict__ lines,
                             const uint32_t* __restrict__ rec_line, uint64_t n_rec, const uint64_t* __restrict__ name_off,
                             uint8_t* __restrict__ names);

}  // namespace itt
