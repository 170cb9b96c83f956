// pipeline.cuh — device-side state of one trace flowing through the hot path, and the
// stage entry points implemented across intern.cu / sa.cu / mine.cu / match.cu / metrics.cu.
#pragma once
#include <vector>

#include "common.cuh"
#include "radix.cuh"
#include "scan.cuh"

namespace itt {

constexpr uint32_t kNone = 0xFFFFFFFFu;

// ------------------------------------------------------------------ records (intern.cu)
struct DevRecords {
  uint64_t n = 0;
  const int64_t* start = nullptr;
  const int64_t* dur = nullptr;
  const int64_t* size = nullptr;
  const uint8_t* flags = nullptr;
  const uint32_t* stream = nullptr;
  const uint16_t* device = nullptr;  // may be null
  const uint64_t* name_off = nullptr;
  const uint8_t* name_bytes = nullptr;  // null when the names are streamed from host memory
  const uint8_t* host_names = nullptr;  // streamed names (ITT_MEM_*_NAMES modes)
  int64_t name_total = -1;               // name_off[n] when known on the host (host columns)
  uint64_t stream_chunk = 0;             // streamed-name chunk bytes (0: default 1 GiB)
  cudaEvent_t cols_ready = nullptr;      // host columns copied on the copy stream (auto-streamed names)
  // late durations (analyze of large pinned host traces): the duration column crosses PCIe after
  // the names, while the suffix array is built; the census's stream ends and the token / HtoD ends
  // are filled in by finish_late_durations before anything reads them
  const int64_t* dur_host = nullptr;     // pinned source of the late copy (null: no late copy)
  cudaEvent_t dur_ready = nullptr;       // recorded on the copy stream after the late copy
  bool census_ends_late = false;         // the census ran without durations: last_end pending
  bool compact_ends_late = false;        // the compaction ran without durations: tok_end / htod_end pending
  ~DevRecords() {
    if (cols_ready) cudaEventDestroy(cols_ready);
    if (dur_ready) {  // a late copy still in flight (an error path) must land before o_dur is released
      cudaEventSynchronize(dur_ready);
      cudaEventDestroy(dur_ready);
    }
  }
  int order = ITT_ORDER_UNKNOWN;
  // owned copies when the caller passed host memory
  DBuf<int64_t> o_start, o_dur, o_size;
  DBuf<uint8_t> o_flags, o_names;
  DBuf<uint32_t> o_stream;
  DBuf<uint16_t> o_device;
  DBuf<uint64_t> o_off;
};

// Records flowing through intern: (start,row) order, the name dictionary, the census.
struct TraceState {
  Ctx* c = nullptr;
  DevRecords rec;
  // ordering (K1)
  bool sorted = true;
  DBuf<uint32_t> perm;  // sorted position -> source row (only when !sorted)
  DBuf<unsigned long long> order_stats;
  bool order_pending = false;  // order_launch ran; order_finish has not read the verdict yet
  bool perm_local = false;  // perm only moves rows inside their 256-row block (the block-sort fast path)
  // name dictionary (K2)
  uint32_t table_bits = 0;
  DBuf<uint64_t> tkey;     // 64-bit name hash per slot (0 = empty)
  DBuf<uint32_t> trep;     // smallest source row carrying the slot's name
  DBuf<uint32_t> tfirst;   // first main-stream token index with this name
  DBuf<uint8_t> tflags;    // classify bits of the slot's name
  DBuf<uint32_t> used;     // claimed slots
  uint32_t n_used = 0;
  DBuf<uint32_t> slot;     // per source row
  DBuf<uint8_t> kind;      // per source row (ITT_KIND_*)
  // device census
  std::vector<uint64_t> dev_counts;
  uint32_t n_devices = 1;
  uint16_t majority = 0;
  bool filtering = false;  // more than one device: drop non-majority records
  uint64_t kept = 0;
  // stream census
  std::vector<itt_stream_summary> streams;
  // compaction outputs (K3)
  uint64_t n_tok = 0, n_htod = 0;
  DBuf<uint32_t> tok_slot;
  DBuf<int32_t> tokens;
  DBuf<int64_t> tok_start, tok_end;
  DBuf<uint8_t> tok_kind;     // ITT_KIND_* per token (a12)
  DBuf<uint64_t> tok_record;  // sorted-order record index (only for build_token_sequence)
  DBuf<int64_t> htod_start, htod_end, htod_size;
  DBuf<unsigned long long> htod_range;  // [min, max] HtoD end, sign bit flipped (set by compact_main)
  uint32_t n_names = 0;
  std::vector<uint64_t> name_row;  // token id -> source row
  DBuf<uint64_t> compact_tiles;    // the reduce-then-scan tile offsets, kept for the late ends pass
  uint32_t main_stream = 0;
  ScanScratch scan;
  radix::Scratch rs;
};

void upload_records(Ctx* c, const itt_records* r, DevRecords& d, bool allow_late_dur = false);
void order_records(TraceState& t);
void order_launch(TraceState& t);  // order_records in two halves: launches + deferred verdict copy
void order_finish(TraceState& t);  // reads the verdict (after a later sync), radix fallback if needed
void build_dictionary(TraceState& t);          // hash + verify + classify + device census
void stream_census(TraceState& t);             // summaries over the kept records (classified)
void compact_main(TraceState& t, uint32_t main_stream, bool want_record_index);
void renumber_tokens(TraceState& t);           // first-appearance ids + token map
int64_t count_overlaps(TraceState& t);         // count_interval_overlaps on the compacted main stream
void release_rows(TraceState& t);              // free per-record arrays (and owned column copies) after tokens
void release_rows_but_late(TraceState& t);     // the same, keeping the columns the late ends pass reads
void issue_late_durations(TraceState& t);      // the late duration copy on the copy stream (once)
void finish_late_durations(TraceState& t);     // wait for it; stream ends, token / HtoD ends

// ------------------------------------------------------------------ suffix array (sa.cu)
struct SuffixState {
  uint64_t n = 0;   // tokens
  uint64_t np = 0;  // n + 1 suffixes
  DBuf<int32_t> text;         // tokens + [terminator] (codes)
  DBuf<uint32_t> sa;          // [np]
  DBuf<uint32_t> lcp;         // [np]
  std::vector<DBuf<uint32_t>> levels;  // rank (group head) after each doubling round
  std::vector<uintptr_t> level_tags;   // their addresses, bit 0 set for a u16 level
  std::vector<uint32_t> level_h;       // prefix length each level separates (ascending; see lift_ratio in sa.cu)
  uint32_t h0 = 1;            // prefix length of levels[0]
  int32_t lo = 0;             // text code = token - lo
  int rounds = 0;
  uint32_t h_final = 0;       // prefix length the last level separates
  uint32_t cap = 0xFFFFFFFFu; // LCP values are min(lcp, cap); SA exact up to ties of h_final-prefixes
  bool keep_levels = true;    // false: only the newest two levels stay allocated (SA without LCP at 1B+)
};
// tokens: device int32[n]; term: unique terminator.  cap: only the first `cap` symbols matter
// (mining with max length L_max needs cap = L_max + 1); 0xFFFFFFFF = full suffix array.
// known_alphabet: the caller guarantees tokens in [0, term) (interned ids, term = V), which
// skips the range/terminator scan and the init sort's trivial-pass readback (two host syncs).
void build_suffix_array(Ctx* c, const int32_t* tokens, uint64_t n, int32_t term, SuffixState& s, bool want_lcp,
                        radix::Scratch& rs, ScanScratch& scan, uint32_t cap = 0xFFFFFFFFu, bool known_alphabet = false);

// Many traces' suffix arrays in one doubling sequence (batched analyze, C4): tokens device
// int32[n] with ids < vmax; sa / lcp device [n + 1] outputs; LCP capped at cap (>= every L_max+1).
struct BatchSAItem {
  const int32_t* tokens;
  uint64_t n;
  uint32_t* sa;
  uint32_t* lcp;
};
void build_batched_sa(Ctx* c, const std::vector<BatchSAItem>& items, int32_t vmax, uint32_t cap, radix::Scratch& rs,
                      ScanScratch& scan);

// ------------------------------------------------------------------ mining (mine.cu)
struct IntervalState {
  DBuf<uint32_t> cnt;  // count of the interval represented at k (0 = not a representative)
  DBuf<uint32_t> par;  // parent depth
  DBuf<uint32_t> lb;   // left boundary
  DBuf<uint4> list;    // list mode: (LCP, count, parent depth, left boundary) of the candidate intervals
  DBuf<unsigned int> n_list;
};
// list_max_len > 0: list mode for mining with repeats cut at list_max_len (the largest L_max of the
// loops); 0: the dense per-position arrays (enumerate_repeats)
void lcp_intervals(Ctx* c, const SuffixState& s, IntervalState& iv, uint32_t list_max_len = 0);

struct MinedPattern {
  int status = 0;
  std::string error;
  std::vector<int32_t> tokens;
  int64_t count = 0, first_token = 0, epsilon_used = 0;
};
// mine_pattern_impl (mine.hpp:75-111) over shared SA/LCP/intervals
MinedPattern mine_one(Ctx* c, const SuffixState& s, const IntervalState& iv, const itt_mining_cfg& cfg,
                      const std::string& label);
std::vector<MinedPattern> mine_loops(Ctx* c, const SuffixState& s, const IntervalState& iv,
                                     const std::vector<itt_mining_cfg>& loops, bool multi);

// ------------------------------------------------------------------ matching (match.cu)
struct SpanState {
  uint64_t n = 0;
  DBuf<uint32_t> start, end, extra;
};
// `head` = pattern[0] (the caller holds the pattern on the host).
void approx_match_dev(Ctx* c, const int32_t* tokens, uint64_t n, const int32_t* pattern_dev, int32_t head, uint64_t m,
                      int64_t k0, SpanState& out, ScanScratch& scan);

// ------------------------------------------------------------------ aggregates (metrics.cu)
void iteration_aggregates(Ctx* c, const int64_t* tok_start, const int64_t* tok_end, uint64_t n_tok,
                          const int64_t* htod_start, const int64_t* htod_end, const int64_t* htod_size, uint64_t n_htod,
                          const unsigned long long* htod_range, const SpanState& spans,
                          itt_iter_row* rows /* host, spans.n */, itt_clamps& clamps,
                          ScanScratch& scan);

// ------------------------------------------------------------------ a12 per-op profile (profile.cu)
// a12 over device token columns and spans.  op_totals [n_ops] / iter_totals [spans.n]: host
// buffers (either may be null).  With want_cells the (iteration, op) grid comes back in a pinned
// block from c->out_alloc.  method: ITT_OP_PROFILE_*.
struct OpProfile {
  itt_op_cell* cells = nullptr;
  uint64_t n = 0;
};
OpProfile op_profile(Ctx* c, const int32_t* tokens, const int64_t* tok_start, const int64_t* tok_end,
                     const uint8_t* tok_kind, uint64_t n_tok, uint32_t n_ops, const SpanState& spans, int method,
                     bool want_cells, itt_op_total* op_totals, itt_iter_op_total* iter_totals, ScanScratch& scan,
                     radix::Scratch& rs);

// ------------------------------------------------------------------ distributed SA steps (dist.cu)
namespace dsa {
void keys(Ctx* c, const int32_t* text, uint64_t np, uint64_t lo, uint64_t cnt, int bits, int k, const uint32_t* rank,
          const uint32_t* rank2, uint64_t n2, int b, uint64_t* a, uint32_t* v);
void partition(Ctx* c, const uint64_t* a, const uint32_t* b, uint64_t cnt, int mode, const uint64_t* spl_a,
               const uint32_t* spl_b, uint32_t nspl, const uint64_t* bounds, uint32_t P, uint64_t* oa, uint32_t* ob,
               uint64_t* counts_host);
void sort(Ctx* c, uint64_t* a, uint32_t* b, uint64_t cnt, int bits);
uint64_t ids(Ctx* c, const uint64_t* a, const uint32_t* b, uint64_t cnt, bool has_prev, uint64_t prev, uint32_t offset,
             uint64_t* out);
void scatter_hi(Ctx* c, const uint64_t* p, uint64_t cnt, uint64_t lo, uint32_t* dst);
void lcp_requests(Ctx* c, const uint64_t* packed, uint64_t cnt, uint64_t kbase, bool has_prev, uint64_t prev, uint64_t* a,
                  uint32_t* b);
void kasai(Ctx* c, const int32_t* text, uint64_t np, uint64_t lo, uint64_t cnt, const uint64_t* req_a, const uint32_t* req_b,
           uint32_t cap, uint64_t* out);
void sample(Ctx* c, const uint64_t* a, const uint32_t* b, uint64_t cnt, uint32_t s, uint64_t* oa, uint32_t* ob);
}  // namespace dsa

}  // namespace itt

// the C-ABI's opaque context (capi.cu, dist_driver.cu)
struct itt_ctx {
  itt::Ctx c;
};
