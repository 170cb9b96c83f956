/*
 * itt_oracle.h — CPU restatement of the reference hot path in plain C (oracle/itt_oracle.c).
 *
 * TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the checker; the product (libitertrace_cuda.so) never links it.
 * Each function cites the reference file:line it restates (paths under
 * /root/reference/proj/include/itertrace/).  The restatement is pinned against the
 * reference itself (oracle/_ref, built from the reference headers) and the reference's
 * known-answer tests by tests/test_oracle_pinning.py.
 */
#ifndef ITT_ORACLE_H
#define ITT_ORACLE_H
#include <stdint.h>
#include "itertrace_cuda.h"
#include "ref_api.h"
#ifdef __cplusplus
extern "C" {
#endif

/* stable order by (start, row): ingest.hpp:396-400.  perm[k] = source row of the k-th record */
void orc_sort_records(uint64_t n, const int64_t* start, uint64_t* perm);
/* classify_op_kind: trace.hpp:103-113 */
int orc_classify(const uint8_t* name, uint64_t len, int has_throughput);
/* summarize_streams + classify_streams (streams.hpp:60-103) after filter_majority_device
 * (streams.hpp:179-207) when filter_device != 0 */
int orc_summarize_streams(const itt_records* r, int filter_device, itt_stream_summary* out, uint32_t cap,
                          uint32_t* n_out, uint64_t* dropped);
/* select_main_stream: streams.hpp:113-145 (returns ITT_E_NO_MAIN_STREAM when none) */
int orc_select_main_stream(const itt_stream_summary* s, uint32_t n, uint32_t* main_stream, uint32_t* n_main);
/* build_token_sequence: streams.hpp:147-169 over the (start,row)-sorted records */
int orc_build_token_sequence(const itt_records* r, uint32_t main_stream, int32_t* tokens, uint64_t* record_index,
                             uint64_t* n_out, uint32_t* n_names, uint64_t* name_row);
/* suffix array of tokens+[term] by plain prefix doubling (qsort), LCP by Kasai */
int orc_suffix_array(const int32_t* tokens, uint64_t n, int32_t term, uint32_t* sa, uint32_t* lcp);
/* enumerate_repeats: mine.hpp:46-60, through LCP intervals */
int orc_enumerate_repeats(const int32_t* tokens, uint64_t n, int32_t term, int64_t min_count, int64_t max_len,
                          itt_repeat** out, uint64_t* n_out);
/* mine_pattern / mine_patterns_multi: mine.hpp:64-165 */
int orc_mine_patterns(const int32_t* tokens, uint64_t n, uint32_t n_names, const itt_mining_cfg* loops,
                      uint32_t n_loops, int multi, itt_pattern* out, char* err, uint64_t err_cap);
/* approx_match: match.hpp:41-85 */
int orc_approx_match(const int32_t* tokens, uint64_t n, const int32_t* pattern, uint64_t m, int64_t k0, itt_span** out,
                     uint64_t* n_out);
/* partition_iterations + collect_htod_records + compute_iteration_metrics: metrics.hpp:44-164 */
int orc_iteration_metrics(const itt_records* r, uint32_t main_stream, const itt_span* spans, uint64_t n_spans,
                          ref_iter* rows, itt_clamps* clamps);
/* a12 per-op profile — no reference function; restates include/itertrace_cuda.h itt_op_cell
 * (parity unpinned by the reference) */
int orc_op_profile(const int32_t* tokens, const int64_t* tok_start, const int64_t* tok_end, const uint8_t* tok_kind,
                   uint64_t n, uint32_t n_ops, const itt_span* spans, uint64_t I, itt_op_cell** out, uint64_t* n_out);
void orc_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
