/*
 * ref_api.h — C entry points of oracle/_ref/libitertrace_ref.so.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the UNMODIFIED reference (header-only
 * C++20 at /root/reference/proj/include/itertrace) compiled by oracle/Makefile from
 * the sources where they lie, behind a thin C wrapper (oracle/ref_wrapper.cpp).  It is
 * used (a) by tests/ as the parity oracle and to pin oracle/itt_oracle.c, and
 * (b) by bench.py's cpu_baseline / --impl reference legs as the CPU reference.
 * The product path (libitertrace_cuda.so) never links or loads it.
 */
#ifndef ITT_REF_API_H
#define ITT_REF_API_H
#include <stdint.h>
#include "itertrace_cuda.h"
#ifdef __cplusplus
extern "C" {
#endif

typedef struct ref_iter {
  int64_t index, start_token, end_token, extra, t_start, t_end;
  int64_t interval_ns, htod_bytes;
  int32_t has_interval, has_overlap;
  double overlap_ratio, op_gap_mean_ns;
} ref_iter;

typedef struct ref_loop {
  int64_t iterations_declared, pattern_length, pattern_count, epsilon_used, first_token, k0_used;
  int32_t* pattern_tokens;
  uint64_t n_iterations;
  ref_iter* iters;
  double avg_interval_ns, avg_overlap, avg_operation_ns, avg_size_bytes;
  int64_t max_interval_ns;
  int32_t insufficient_intervals, diagnosis; /* DiagnosisCode, report.hpp:24 */
} ref_loop;

typedef struct ref_stage_times { /* steady_clock milliseconds per stage */
  double order_ms, filter_census_ms, intern_ms, mine_ms, match_ms, metrics_ms, total_ms;
  double analyze_ms; /* the analyze_trace (or staged) call alone: no AoS marshalling, no rendering */
} ref_stage_times;

typedef struct ref_analysis {
  int32_t status;         /* 0 or 1 + ErrorKind */
  char* error;            /* malloc'd message or NULL */
  uint32_t n_streams;
  itt_stream_summary* streams;
  uint32_t main_stream;
  uint64_t n_tokens;
  uint32_t n_names;
  uint32_t n_loops;
  ref_loop* loops;
  char* warnings;         /* '\n'-joined Report.warnings */
  char* summary_json;     /* summary_to_json(report).dump(2) + "\n" (report.hpp:304) */
  char* details_csv;      /* details_to_csv of loop 1 */
  ref_stage_times times;
} ref_analysis;

/* parse-free analyze: columns -> NormalizedTrace (stable sort by (start,row), ingest.hpp:396-400)
 * -> analyze_trace (pipeline.hpp:34-134).  staged != 0 runs the same stage calls one by one
 * with steady_clock timers instead of analyze_trace (for the CPU baseline); results agree. */
int ref_analyze(const itt_records* recs, const itt_analyze_opts* opts, int staged, ref_analysis* out);
void ref_free_analysis(ref_analysis* a);

/* SA/LCP from the reference suffix tree: DFS in child-key order (suffix_tree.hpp:33), leaf ->
 * suffix (n+1) - depth; LCP by Kasai over that SA. */
int ref_suffix_array(const int32_t* tokens, uint64_t n, int32_t term, uint32_t* sa, uint32_t* lcp);
/* enumerate_repeats (mine.hpp:46-60) on SuffixTree(tokens, term) */
int ref_enumerate_repeats(const int32_t* tokens, uint64_t n, int32_t term, int64_t min_count, int64_t max_len,
                          itt_repeat** out, uint64_t* n_out);
/* mine_pattern / mine_patterns_multi (mine.hpp:119-165) with a TokenSequence whose names are
 * n_names placeholders (terminator == n_names). */
int ref_mine_patterns(const int32_t* tokens, uint64_t n, uint32_t n_names, const itt_mining_cfg* loops, uint32_t n_loops,
                      int multi, itt_pattern* out, char* err, uint64_t err_cap);
/* approx_match (match.hpp:41-85) */
int ref_approx_match(const int32_t* tokens, uint64_t n, const int32_t* pattern, uint64_t m, int64_t k0, itt_span** out,
                     uint64_t* n_out);
/* build_token_sequence (streams.hpp:147-169) on the (start,row)-sorted records */
int ref_build_token_sequence(const itt_records* recs, uint32_t main_stream, int32_t* tokens, uint64_t* record_index,
                             uint64_t* n_out, uint32_t* n_names, uint64_t* name_row);
/* compute_iteration_metrics (metrics.hpp:109-164) + clamps, on the sorted records */
int ref_iteration_metrics(const itt_records* recs, uint32_t main_stream, const itt_span* spans, uint64_t n_spans,
                          ref_iter* rows, itt_clamps* clamps);
/* summarize_streams + classify_streams (streams.hpp:60-103) after the optional device filter */
int ref_summarize_streams(const itt_records* recs, int filter_device, itt_stream_summary* out, uint32_t cap,
                          uint32_t* n_out, uint64_t* dropped);
void ref_free(void* p);

/* ---- CSV ingest (ingest.hpp:154-402) */
typedef struct ref_parsed {
  int32_t status;        /* 0 or 1 + ErrorKind */
  char* error;
  uint64_t n;            /* records, in the reference's output order (stable-sorted by (start, row)) */
  int64_t* start_ns;
  int64_t* duration_ns;
  int64_t* size_bytes;   /* 0 when absent */
  uint8_t* flags;        /* ITT_REC_HAS_SIZE | ITT_REC_HAS_THROUGHPUT */
  uint32_t* stream;
  uint64_t* row;
  uint64_t* name_off;    /* [n+1] */
  uint8_t* name_bytes;
  uint64_t* device_off;  /* [n+1] device label bytes per record */
  uint8_t* device_bytes;
  uint64_t rows_total, rows_parsed, rows_skipped;
  uint64_t n_skips;
  uint64_t* skip_line;
  char* skip_reasons;    /* '\n'-joined */
  int32_t column[7];     /* Start, Duration, Size, Throughput, Device, Stream, Name; -1 absent */
  char* warnings;        /* '\n'-joined NormalizedTrace::warnings */
} ref_parsed;
int ref_parse_csv(const char* text, uint64_t len, const char* label, ref_parsed* out);
void ref_free_parsed(ref_parsed* p);
/* the reference generator's CSV (synth.hpp:187): malloc'd text */
char* ref_synth_csv(uint64_t seed, int64_t pattern_len, int64_t iterations, int64_t vocab_size, double insert_prob,
                    int64_t max_inserts, int32_t inside_pattern, int32_t pathology, uint64_t* len);
/* parse_trace_text + analyze_trace end to end (summary JSON / details CSV as the CLI writes them) */
int ref_analyze_csv(const char* text, uint64_t len, const char* label, const itt_analyze_opts* opts, ref_analysis* out);

/* nlohmann::json(v).dump() — pins paper_1707_03750_b200/jsonfloat.py */
int ref_json_double(double v, char* out, int cap);

#ifdef __cplusplus
}
#endif
#endif
