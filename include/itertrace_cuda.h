/*
 * itertrace_cuda.h — C-ABI of libitertrace_cuda.so, the B200 (sm_100a) hot path of
 * DeepProf-style trace mining: intern -> suffix array -> LCP -> repeat/period ->
 * iteration boundaries -> per-iteration aggregates.
 *
 * Every entry point replaces one function of the reference's header-only C++ API
 * (paths relative to /root/reference/proj/include/itertrace/); the replaced function
 * is cited beside each declaration.  The reference has no FFI of its own:
 * this header is the contract a maintainer binds from the reference's C++ headers
 * (see INTEGRATION.md).
 *
 * Conventions
 *  - All entry points return 0 on success, otherwise an itt_status.  1..12 are
 *    1 + (int)itertrace::ErrorKind (errors.hpp:8-21) so the C++ shim can rethrow
 *    itertrace::Error with the same kind; the stage-prefixed message ("pattern-mining: ...")
 *    is available from itt_last_error(ctx) until the next call on that context.
 *  - Inputs are borrowed for the duration of the call.  Fixed-size outputs are
 *    caller-allocated; variable-size outputs are allocated by the library and
 *    released with itt_free().
 *  - One context per host thread and device; it owns one cudaStream_t.  Calls are
 *    synchronous with respect to the host (the reference API returns by value).
 *  - There is no CPU fallback: without a usable sm_100 device itt_ctx_create fails
 *    with ITT_E_CUDA.
 */
#ifndef ITERTRACE_CUDA_H
#define ITERTRACE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ITT_ABI_VERSION 2

typedef enum itt_status {
  ITT_OK = 0,
  /* 1 + itertrace::ErrorKind, errors.hpp:8-21 */
  ITT_E_UNREADABLE_FILE = 1,
  ITT_E_MISSING_COLUMN = 2,
  ITT_E_TOO_MANY_BAD_ROWS = 3,
  ITT_E_EMPTY_TRACE = 4,
  ITT_E_NO_MAIN_STREAM = 5,
  ITT_E_EMPTY_MAIN_STREAM = 6,
  ITT_E_INVALID_ITERATION_COUNT = 7,
  ITT_E_NO_PATTERN_FOUND = 8,
  ITT_E_AMBIGUOUS_LOOPS = 9,
  ITT_E_NO_ITERATIONS = 10,
  ITT_E_INVALID_CONFIG = 11,
  ITT_E_IO_ERROR = 12,
  /* device / library failures: not an ErrorKind; the shim throws std::runtime_error (exit 1) */
  ITT_E_CUDA = 100,
  ITT_E_NCCL = 101,
  ITT_E_INVALID_ARGUMENT = 102,
} itt_status;

/* OpKind, trace.hpp:17-24 */
enum { ITT_KIND_KERNEL = 0, ITT_KIND_HTOD, ITT_KIND_DTOH, ITT_KIND_DTOD, ITT_KIND_MEMSET, ITT_KIND_OTHER };
/* StreamClass, streams.hpp:34 */
enum { ITT_CLASS_MAIN = 0, ITT_CLASS_COPY_HTOD, ITT_CLASS_COPY_DTOH, ITT_CLASS_COPY_MIXED, ITT_CLASS_ASSIST };

/* itt_records.flags bits: presence of TraceRecord::size_bytes / throughput_bps (trace.hpp:46-47) */
#define ITT_REC_HAS_SIZE 0x1u
#define ITT_REC_HAS_THROUGHPUT 0x2u

#define ITT_MEM_HOST 0
#define ITT_MEM_DEVICE 1
/* Names that do not fit in HBM next to the pipeline (C5: 80 GB): name_bytes stays in host memory
 * (pinned — cudaHostRegister'd or cudaMallocHost — for overlapped DMA) and is streamed through
 * two bounded device windows (1 GiB, ITT_STREAM_CHUNK overrides), chunk by chunk, into the hash
 * pass; the distinct names' bytes are kept in a small device arena.  The other columns are host
 * memory (ITT_MEM_HOST_STREAM_NAMES) or device memory (ITT_MEM_DEVICE_HOST_NAMES). */
#define ITT_MEM_HOST_STREAM_NAMES 2
#define ITT_MEM_DEVICE_HOST_NAMES 3

#define ITT_ORDER_UNKNOWN 0 /* rows in source order; the library stable-sorts by (start, row) */
#define ITT_ORDER_SORTED 1  /* rows already in NormalizedTrace order (ingest.hpp:396-400) */

/*
 * Columnar trace records: the NormalizedTrace/TraceRecord AoS (trace.hpp:43-66) as
 * structure-of-arrays.  Row i is record i in source order (its TraceRecord::row).
 * Device labels are interned by the caller in byte-lexicographic order, so the
 * reference's "ties to the lexicographically smallest label" (streams.hpp:187-194)
 * becomes "ties to the smallest id".
 */
typedef struct itt_records {
  uint64_t n;                 /* number of records */
  const int64_t* start_ns;    /* [n] */
  const int64_t* duration_ns; /* [n] */
  const int64_t* size_bytes;  /* [n]; read only where flags & ITT_REC_HAS_SIZE */
  const uint8_t* flags;       /* [n] */
  const uint32_t* stream;     /* [n] */
  const uint16_t* device;     /* [n] device-label rank; NULL = single device 0 */
  const uint64_t* name_off;   /* [n+1]; name of row i = name_bytes[name_off[i] .. name_off[i+1]) */
  const uint8_t* name_bytes;  /* [name_off[n]] */
  int32_t mem;                /* ITT_MEM_HOST / ITT_MEM_DEVICE (all pointers alike), or a *_NAMES mode */
  int32_t order;              /* ITT_ORDER_UNKNOWN or ITT_ORDER_SORTED */
} itt_records;

typedef struct itt_ctx itt_ctx;

/* ---------------------------------------------------------------- context */
int itt_abi_version(void);
int itt_ctx_create(int device, itt_ctx** out);
int itt_ctx_destroy(itt_ctx* ctx);
const char* itt_last_error(itt_ctx* ctx);
int itt_free(itt_ctx* ctx, void* p);

/* profiling: per-kernel CUDA-event timing on the context stream (off by default) */
typedef struct itt_kernel_stat {
  char name[48];
  uint64_t launches;
  double total_ms;  /* sum of per-launch event durations */
  double bytes;     /* sum of algorithmic bytes declared per launch */
} itt_kernel_stat;
int itt_ctx_set_profiling(itt_ctx* ctx, int enabled);
int itt_ctx_reset_stats(itt_ctx* ctx);
int itt_ctx_kernel_stats(itt_ctx* ctx, itt_kernel_stat* out, uint32_t cap, uint32_t* n_out);
/* total kernel launches issued by the library on this context since creation */
int itt_ctx_launch_count(itt_ctx* ctx, uint64_t* out);
/* device memory of the context's stream-ordered pool: bytes in use now and the high-water mark
 * since creation or the last reset (reset != 0 restarts the high-water mark) */
int itt_ctx_mem_stats(itt_ctx* ctx, uint64_t* used, uint64_t* used_high, int reset);
/* device memory helpers for callers that keep inputs resident in HBM */
int itt_device_alloc(itt_ctx* ctx, uint64_t bytes, void** out);
int itt_device_free(itt_ctx* ctx, void* p);
int itt_memcpy_h2d(itt_ctx* ctx, void* dst, const void* src, uint64_t bytes);
int itt_memcpy_d2h(itt_ctx* ctx, void* dst, const void* src, uint64_t bytes);
/* any direction (unified addressing), synchronous like the others */
int itt_memcpy(itt_ctx* ctx, void* dst, const void* src, uint64_t bytes);
int itt_host_register(itt_ctx* ctx, void* p, uint64_t bytes);
int itt_host_unregister(itt_ctx* ctx, void* p);
int itt_ctx_synchronize(itt_ctx* ctx);
/* the context's cudaStream_t (for callers that time with CUDA events on it) */
int itt_ctx_stream(itt_ctx* ctx, void** stream);

/* ------------------------------------------------------- L2 streams (a1, a2) */
typedef struct itt_stream_summary { /* StreamSummary, streams.hpp:16-32 */
  uint32_t stream;
  int32_t cls;        /* ITT_CLASS_* from classify_streams (streams.hpp:85-103) */
  int64_t counts[6];  /* indexed by ITT_KIND_* */
  int64_t first_start;
  int64_t last_end;
} itt_stream_summary;

typedef struct itt_census {
  uint32_t n_streams;
  itt_stream_summary* streams; /* sorted by stream id (std::map order, streams.hpp:64) */
  uint32_t n_devices;          /* distinct device ids seen */
  uint16_t majority_device;    /* filter_majority_device choice (streams.hpp:179-207) */
  uint64_t dropped_records;    /* records of other devices */
  uint64_t n_records;
} itt_census;

/* summarize_streams (streams.hpp:60-81) + classify_streams (:85-103) after
 * filter_majority_device (:179-207) when filter_device != 0.  Frees with itt_free(census->streams). */
int itt_summarize_streams(itt_ctx* ctx, const itt_records* recs, int filter_device, itt_census* out);

/* select_main_stream (streams.hpp:113-145) over a census */
int itt_select_main_stream(itt_ctx* ctx, const itt_census* census, uint32_t* main_stream, uint32_t* n_main_streams);

typedef struct itt_tokens { /* TokenSequence, streams.hpp:49-58 */
  uint64_t n;
  int32_t* tokens;        /* [n] token ids, first-appearance order */
  uint64_t* record_index; /* [n] position of the token's record in (start,row) order */
  uint32_t n_names;       /* V; terminator() == V */
  uint64_t* name_row;     /* [V] source row (itt_records index) of one record carrying name id v */
} itt_tokens;

/* build_token_sequence (streams.hpp:147-169).  Records are taken in (start,row)
 * order; no device filter is applied (the reference applies it in analyze_trace). */
int itt_build_token_sequence(itt_ctx* ctx, const itt_records* recs, uint32_t main_stream, itt_tokens** out);

/* count_interval_overlaps (streams.hpp:212-221) */
int itt_count_interval_overlaps(itt_ctx* ctx, const itt_records* recs, uint32_t stream, int64_t* out);

/* ------------------------------------------------------- primitives */
/* Stable LSD onesweep radix sort of (u32 key, u32 value) pairs on key bits [begin_bit, end_bit),
 * in place.  mem selects host (copied in and out) or device pointers.  The sort behind the
 * suffix array (K4/K5) and the (start,row) ingest order (K1, ingest.hpp:396-400). */
int itt_radix_sort_pairs_u32(itt_ctx* ctx, uint32_t* keys, uint32_t* vals, uint64_t n, int begin_bit, int end_bit,
                             int mem);

/* ------------------------------------------------------- L3 mining (a3-a6) */
/* Suffix array + LCP of tokens[0..n) followed by a unique terminator `term`:
 * sa[k] = start of the k-th smallest suffix of tokens+[term] (n+1 entries), lcp[0] = 0,
 * lcp[k] = lcp(sa[k-1], sa[k]).  Equals the leaf order of SuffixTree (suffix_tree.hpp:21-190)
 * in ascending child-key order.  lcp may be NULL (then only two rank levels stay resident, so
 * the SA of ~1B tokens fits one B200).  Buffers of n+1 entries, each in host OR device memory
 * (told apart through CUDA unified addressing).  n+1 < 2^32 - 1. */
int itt_suffix_array(itt_ctx* ctx, const int32_t* tokens, uint64_t n, int32_t term, uint32_t* sa, uint32_t* lcp);
/* The capped suffix array the mining path builds (mine.hpp:64-67 never looks past L_max; DESIGN
 * §3.1): suffixes ordered by their first h >= cap symbols (ties of equal cap-prefixes in an
 * unspecified but deterministic order), lcp[k] = min(lcp(sa[k-1], sa[k]), cap).  cap = 0xFFFFFFFF
 * is the full suffix array.  Host or device buffers. */
int itt_suffix_array_capped(itt_ctx* ctx, const int32_t* tokens, uint64_t n, int32_t term, uint32_t cap, uint32_t* sa,
                            uint32_t* lcp);

typedef struct itt_repeat { /* RepeatCandidate, mine.hpp:31-35 */
  int32_t start;
  int32_t length;
  int64_t count;
} itt_repeat;
/* enumerate_repeats (mine.hpp:46-60) over the suffix tree of tokens+[term] (any order). */
int itt_enumerate_repeats(itt_ctx* ctx, const int32_t* tokens, uint64_t n, int32_t term, int64_t min_count,
                          int64_t max_len, itt_repeat** out, uint64_t* n_out);

typedef struct itt_mining_cfg { /* MiningConfig, mine.hpp:18-22 */
  int64_t iterations;
  int64_t epsilon0;
  int64_t epsilon_cap; /* <= 0 means "defaults to iterations" (std::nullopt) */
} itt_mining_cfg;

typedef struct itt_pattern { /* PatternCandidate, mine.hpp:24-29 */
  int64_t length;
  int32_t* tokens; /* [length], library-allocated (freed with the itt_pattern array via itt_free_patterns) */
  int64_t count;
  int64_t first_token;
  int64_t epsilon_used;
} itt_pattern;

/* mine_pattern (mine.hpp:119-122) when multi == 0 and n_loops == 1;
 * mine_patterns_multi (mine.hpp:132-165) when multi != 0. */
int itt_mine_patterns(itt_ctx* ctx, const int32_t* tokens, uint64_t n, int32_t term, const itt_mining_cfg* loops,
                      uint32_t n_loops, int multi, itt_pattern** out);
int itt_free_patterns(itt_ctx* ctx, itt_pattern* p, uint32_t n_loops);

/* mine_pattern / mine_patterns_multi over a suffix array built elsewhere (the distributed
 * prefix doubling below, gathered to one device).  All pointers are DEVICE memory: tokens[n] in
 * [0, term), sa[n+1], lcp[n+1] with lcp values min(lcp, cap) for a cap >= max L_max + 1
 * (mine.hpp:64-67) — what itt_dsa_* produce.  Same results and errors as itt_mine_patterns. */
int itt_mine_patterns_sa(itt_ctx* ctx, const int32_t* tokens, uint64_t n, int32_t term, const uint32_t* sa,
                         const uint32_t* lcp, const itt_mining_cfg* loops, uint32_t n_loops, int multi, itt_pattern** out);

/* ------------------------------------------------------- distributed suffix array (C5)
 * Per-rank device steps of prefix doubling with a sample-sort all-to-all over G ranks; the
 * exchanges are the host driver's (paper_1707_03750_b200/dist_sa.py).  Every pointer is DEVICE
 * memory unless marked host.  Suffix positions are block-partitioned: a rank owns [lo, lo+cnt).
 * Records are (u64 a, u32 b) pairs.  Replaces, for traces beyond one device, the same suffix
 * order and node depths as itt_suffix_array (SuffixTree, suffix_tree.hpp:21-190); n+1 < 2^31. */
/* keys of own positions: rank == NULL: a = first k symbols of text[i..] (sym_bits each, text =
 * tokens + [term], np entries, replicated); else a = rank[j] << b | (j < n2 ? rank2[j] + 1 : 0)
 * with rank2 = ranks of positions lo+h.. ; v = i. */
int itt_dsa_keys(itt_ctx* ctx, const int32_t* text, uint64_t np, uint64_t lo, uint64_t cnt, int sym_bits, int k,
                 const uint32_t* rank, const uint32_t* rank2, uint64_t n2, int b, uint64_t* a, uint32_t* v);
/* stable partition by destination rank: mode 0 = number of splitters (spl_a, spl_b)[nspl] <= (a, b);
 * mode 1 = owner of position (uint32)a under bounds[P+1].  counts: host[P]. */
int itt_dsa_partition(itt_ctx* ctx, const uint64_t* a, const uint32_t* b, uint64_t cnt, int mode, const uint64_t* spl_a,
                      const uint32_t* spl_b, uint32_t nspl, const uint64_t* bounds, uint32_t P, uint64_t* out_a,
                      uint32_t* out_b, uint64_t* counts);
/* stable sort of (a, b) by the low `bits` bits of a, in place */
int itt_dsa_sort(itt_ctx* ctx, uint64_t* a, uint32_t* b, uint64_t cnt, int bits);
/* dense group ids over this rank's slice of the sorted records: flag_j = a_j != a_{j-1} (a_{-1} =
 * prev when has_prev); out_j = (offset + #flags<=j - 1) << 32 | b_j; n_groups: host, #flags. */
int itt_dsa_ids(itt_ctx* ctx, const uint64_t* a, const uint32_t* b, uint64_t cnt, int has_prev, uint64_t prev,
                uint32_t offset, uint64_t* out, uint64_t* n_groups);
/* dst[(uint32)p_j - lo] = p_j >> 32 */
int itt_dsa_scatter(itt_ctx* ctx, const uint64_t* p, uint64_t cnt, uint64_t lo, uint32_t* dst);
/* LCP requests from the sorted slice (packed (id << 32) | SA, global positions kbase..):
 * a = k << 32 | SA_k, b = SA_{k-1} | 1 << 31 when in the same final group (0x7FFFFFFF at k = 0) */
int itt_dsa_lcp_requests(itt_ctx* ctx, const uint64_t* packed, uint64_t cnt, uint64_t kbase, int has_prev, uint64_t prev,
                         uint64_t* a, uint32_t* b);
/* capped Kasai over own positions from the requests routed to their owner: out_j = plcp << 32 | k
 * (in text order of [lo, lo+cnt)) */
int itt_dsa_kasai(itt_ctx* ctx, const int32_t* text, uint64_t np, uint64_t lo, uint64_t cnt, const uint64_t* req_a,
                  const uint32_t* req_b, uint32_t cap, uint64_t* out);
/* s evenly spaced records (splitter candidates) */
int itt_dsa_sample(itt_ctx* ctx, const uint64_t* a, const uint32_t* b, uint64_t cnt, uint32_t s, uint64_t* out_a,
                   uint32_t* out_b);

/* The same doubling driven natively (csrc/dist_driver.cu; dist_sa.py is its Python restatement):
 * the exchanges go through a communicator — NCCL between GPUs (grouped ncclSend/ncclRecv
 * all-to-alls, ncclAllGather, ncclBroadcast on the context's stream; libnccl is loaded on first
 * use), or virtual ranks (threads of one process sharing one device: device-to-device copies
 * behind a barrier, for tests).  One context and one communicator per rank and host thread. */
typedef struct itt_comm itt_comm;
int itt_comm_nccl_unique_id(uint8_t* id /* [128] */);
int itt_comm_create_nccl(itt_ctx* ctx, int nranks, int rank, const uint8_t* id /* [128] */, itt_comm** out);
int itt_comm_create_local(int nranks, itt_comm** comms /* [nranks] */);
int itt_comm_abort(itt_comm* comm); /* virtual ranks: release the others after one failed */
int itt_comm_destroy(itt_comm* comm);
typedef struct itt_dsa_info {
  int32_t rounds;      /* doubling rounds after the first sort */
  int32_t pad_;
  uint64_t groups;     /* groups of the last level (n+1: a full suffix array) */
  uint32_t h_final;    /* prefix length the last level separates */
  uint32_t cap;        /* LCP values are min(lcp, cap); 0xFFFFFFFF when the SA is full */
} itt_dsa_info;
/* SPMD over the communicator's ranks: text = tokens + [term] (n+1 int32, DEVICE, replicated,
 * tokens in [0, term)).  This rank's slice of the suffix array (sorted positions
 * [kbase, kbase + count)) and, when want_lcp, of the LCP capped at cap (0xFFFFFFFF: full) come back
 * as device allocations released with itt_device_free.  Same suffix order and node depths as
 * itt_suffix_array / SuffixTree (suffix_tree.hpp:21-190); n+1 < 2^31 - 1. */
int itt_dsa_build(itt_ctx* ctx, itt_comm* comm, const int32_t* text, uint64_t n, int32_t term, uint32_t cap, int want_lcp,
                  uint32_t** sa, uint32_t** lcp, uint64_t* kbase, uint64_t* count, itt_dsa_info* info);
/* itt_analyze over G ranks: on the root, set itt_analyze_opts.sa_provider = itt_dsa_provide and
 * sa_user = a provider; the tokens are broadcast, every rank builds its slice, the slices are
 * gathered into the analyze's buffers.  The other ranks call itt_dsa_serve (returns after the
 * root's itt_dsa_stop).  ctx: this rank's context for the distributed steps (on the root, not the
 * one running itt_analyze). */
typedef struct itt_dsa_provider itt_dsa_provider;
int itt_dsa_provider_create(itt_ctx* ctx, itt_comm* comm, int root, itt_dsa_provider** out);
int itt_dsa_provider_destroy(itt_dsa_provider* p);
int itt_dsa_provide(void* user, const int32_t* tokens, uint64_t n, int32_t term, uint32_t cap, uint32_t* sa, uint32_t* lcp);
int itt_dsa_serve(itt_dsa_provider* p);
int itt_dsa_stop(itt_dsa_provider* p);
int itt_dsa_last_info(itt_dsa_provider* p, itt_dsa_info* info);

/* ------------------------------------------------------- L4 matching (a7) */
typedef struct itt_span { /* MatchSpan, match.hpp:28-34 */
  int64_t start_token;
  int64_t end_token;
  int64_t extra;
} itt_span;
/* approx_match (match.hpp:41-85) */
int itt_approx_match(itt_ctx* ctx, const int32_t* tokens, uint64_t n, const int32_t* pattern, uint64_t m, int64_t k0,
                     itt_span** out, uint64_t* n_out);

/* ------------------------------------------------------- L5 aggregates (a8-a11) */
typedef struct itt_iter_row { /* integer core of IterationMetrics, metrics.hpp:21-31 */
  int64_t start_token, end_token, extra;
  int64_t t_start, t_end;     /* partition_iterations (metrics.hpp:44-55) */
  int64_t interval_ns;        /* valid when has_interval (k > 0), clamped at 0 (metrics.hpp:124-130) */
  int64_t copy_ns;            /* clipped HtoD union in the gap; meaningful when interval_ns > 0 (:131-135, :76-100) */
  int64_t htod_bytes;         /* (:138-143) */
  int64_t gap_sum, gap_count; /* op_gap_mean = gap_sum / gap_count, 0 when gap_count == 0 (:145-160) */
  int32_t has_interval;
  int32_t pad_;
} itt_iter_row;

typedef struct itt_clamps {
  int64_t negative_gap_clamps;      /* IterationAnalysis, metrics.hpp:68-72 */
  int64_t negative_interval_clamps;
} itt_clamps;

/* partition_iterations + collect_htod_records + compute_iteration_metrics
 * (metrics.hpp:44-164).  record_index indexes records in (start,row) order; HtoD records are
 * all MemcpyHtoD records of `recs` (all streams).  rows: library-allocated [n_spans]. */
int itt_iteration_metrics(itt_ctx* ctx, const itt_records* recs, const uint64_t* record_index, uint64_t n_tokens,
                          const itt_span* spans, uint64_t n_spans, itt_iter_row** rows, itt_clamps* clamps);

/* ------------------------------------------------------- a12: second-level per-op profile
 * The north star's per-iteration segmented reduction "per op and per iteration" (SURVEY §8a
 * row a12).  The reference has NO such function; the definition below is this library's, built
 * on the reference's own windows (approx_match spans, match.hpp:41-85) and its op-gap rule
 * (metrics.hpp:145-157).  For every span k = [s_k, e_k] (main-stream tokens, inclusive) and every
 * op id v occurring in it, one cell:
 *   count     = #{ j in [s_k, e_k] : tokens[j] = v }
 *   kernel_ns = sum of (end_j - start_j) over those j whose record kind is ITT_KIND_KERNEL
 *   memcpy_ns = sum of (end_j - start_j) over those j of any other kind (copies, memsets, other)
 *   idle_ns   = sum of max(0, start_j - end_{j-1}) over those j with j > s_k: the idle gap in
 *               front of op j inside the iteration, so that sum_v idle_ns(k, v) equals the
 *               reference's clamped op-gap sum of iteration k (metrics.hpp:145-157)
 * Cells are ordered by (iteration, op).  The two reductions of the cell grid: */
/* ------------------------------------------------------- host finish at scale (§8f row 4)
 * The reference's host-side finish over the integer rows, natively: I reaches 500K at C5, where
 * an interpreted finish costs seconds.  Both are pure host functions (ctx only carries errors). */
typedef struct itt_summary { /* SummaryMetrics, metrics.hpp:33-42 */
  double avg_interval_ns;
  int64_t max_interval_ns;
  double avg_overlap;
  double avg_operation_ns;
  double avg_size_bytes;
  int64_t iterations_found;
  int64_t iterations_declared;
  int32_t insufficient_intervals;
  int32_t pad_;
} itt_summary;
/* compute_summary (metrics.hpp:166-202): same operations in the same order (bit-identical
 * doubles); 1 + NoIterations with the reference's message when n == 0. */
int itt_compute_summary(itt_ctx* ctx, const itt_iter_row* rows, uint64_t n, int64_t iterations_declared, itt_summary* out);
/* details_to_csv (report.hpp:191-220) of rows[n], byte for byte, formatted by host threads in
 * row blocks; *out is NUL-terminated, released with itt_free. */
int itt_render_details_csv(itt_ctx* ctx, const itt_iter_row* rows, uint64_t n, char** out, uint64_t* len);

typedef struct itt_op_cell {
  uint32_t iteration;
  int32_t op;
  uint32_t count;
  uint32_t pad_;
  int64_t kernel_ns;
  int64_t memcpy_ns;
  int64_t idle_ns;
} itt_op_cell;

typedef struct itt_op_total { /* per op id, summed over iterations */
  int64_t iterations; /* iterations in which the op occurs (cells of the op) */
  int64_t count;
  int64_t kernel_ns;
  int64_t memcpy_ns;
  int64_t idle_ns;
} itt_op_total;

typedef struct itt_iter_op_total { /* per iteration, summed over ops */
  int64_t distinct_ops; /* cells of the iteration */
  int64_t kernel_ns;
  int64_t memcpy_ns;
  int64_t idle_ns;      /* == the reference's clamped op-gap sum of the iteration */
} itt_iter_op_total;

enum { ITT_OP_PROFILE_AUTO = 0, ITT_OP_PROFILE_SMEM = 1, ITT_OP_PROFILE_SORT = 2 };

/* Token-level entry: tokens/start/end/kind are per main-stream token (host or device memory),
 * op ids in [0, n_ops), spans disjoint and increasing.  method: AUTO picks the shared-memory
 * table when n_ops fits, else the sort-based segmented reduction.  op_totals [n_ops] and
 * iter_totals [n_spans] are caller-allocated (either may be NULL).  cells: NULL to skip the cell
 * grid, else *cells is library-allocated [*n_cells] and released by itt_free. */
int itt_op_profile(itt_ctx* ctx, const int32_t* tokens, const int64_t* tok_start, const int64_t* tok_end,
                   const uint8_t* tok_kind, uint64_t n, uint32_t n_ops, const itt_span* spans, uint64_t n_spans,
                   int method, itt_op_total* op_totals, itt_iter_op_total* iter_totals, itt_op_cell** cells,
                   uint64_t* n_cells);

/* ------------------------------------------------------- CSV ingest
 * parse_trace_text (ingest.hpp:154-402) on the GPU: the header / units rows are read on the host,
 * every data line is parsed by one device thread with the reference's exact rules (quoted fields,
 * inline units, exact decimal scaling, strtod acceptance of Throughput), skipped rows and their
 * reasons, the 10% TooManyBadRows rule and the unit warnings.  The records stay in HBM in source
 * line order (itt_analyze sorts them by (start, row) like ingest.hpp:396-400); device labels are
 * interned to ranks in byte-lexicographic order. */
typedef struct itt_parsed_trace {
  itt_records records;               /* ITT_MEM_DEVICE columns owned by this object, ITT_ORDER_UNKNOWN */
  const uint64_t* line;              /* [records.n] 1-based source line (TraceRecord::row) */
  uint32_t n_device_labels;
  const char* const* device_labels;  /* records.device indexes this, byte-lexicographic */
  uint64_t rows_total, rows_parsed, rows_skipped;   /* IngestReport (ingest.hpp:21-28) */
  uint64_t n_skips;
  const uint64_t* skip_line;         /* [n_skips] */
  const char* const* skip_reason;    /* [n_skips], the reference's reason text */
  int32_t column[7];                 /* field index of Start, Duration, Size, Throughput, Device, Stream, Name; -1 absent */
  uint32_t n_warnings;
  const char* const* warnings;       /* NormalizedTrace::warnings (unit row) */
} itt_parsed_trace;
int itt_parse_csv(itt_ctx* ctx, const char* text, uint64_t len, const char* origin_label, itt_parsed_trace** out);
int itt_free_parsed(itt_ctx* ctx, itt_parsed_trace* p);

/* ------------------------------------------------------- L7 orchestration */
/* itt_analyze_opts.flags: OP_PROFILE fills op_totals / iter_op_totals of every loop result;
 * OP_CELLS also returns the (iteration, op) cell grid (size ~ tokens: large) */
enum { ITT_ANALYZE_OP_PROFILE = 1u, ITT_ANALYZE_OP_CELLS = 2u,
       /* itt_batch_analyze only: the suffix arrays of the traces in flight are built together,
        * one doubling sequence over their concatenation, instead of one per trace */
       ITT_ANALYZE_BATCHED_SA = 4u };

typedef struct itt_analyze_opts { /* AnalyzeOptions, pipeline.hpp:18-25 */
  const int64_t* loops;
  uint32_t n_loops;
  int64_t epsilon0;
  int64_t k0;           /* < 0: default_k0(pattern length) (match.hpp:19-21) */
  int64_t main_stream;  /* < 0: select_main_stream */
  uint32_t flags;       /* ITT_ANALYZE_* (0 = the reference's outputs only) */
  /* Suffix array provider (NULL: the single-device capped doubling, sa.cu).  Called once per
   * analyze on the calling thread, after the token sequence exists and the library's stream is
   * idle, with DEVICE pointers: tokens[n] (ids in [0, term)), and sa / lcp [n+1] to fill with the
   * suffix array of tokens+[term] and its LCP capped at `cap` (= max L_max + 1, mine.hpp:64-67).
   * The distributed suffix array (dist_sa.py, itt_dsa_*) plugs in here; 0 = success. */
  int (*sa_provider)(void* user, const int32_t* tokens, uint64_t n, int32_t term, uint32_t cap, uint32_t* sa,
                     uint32_t* lcp);
  void* sa_user;
} itt_analyze_opts;

typedef struct itt_loop_result { /* LoopReport (report.hpp:92-103) integer fields + details rows */
  int64_t iterations_declared;
  int64_t pattern_length;
  int32_t* pattern_tokens; /* [pattern_length] token ids (names via itt_analysis.name_row) */
  int64_t pattern_count;
  int64_t epsilon_used;
  int64_t first_token;
  int64_t k0_used;
  uint64_t n_iterations;
  itt_iter_row* rows;      /* [n_iterations] */
  itt_clamps clamps;
  itt_op_total* op_totals;           /* a12 (ITT_ANALYZE_OP_PROFILE): [itt_analysis.n_names], else NULL */
  itt_iter_op_total* iter_op_totals; /* a12: [n_iterations], else NULL */
  uint64_t n_op_cells;               /* a12 (ITT_ANALYZE_OP_CELLS), else 0 */
  itt_op_cell* op_cells;             /* [n_op_cells], (iteration, op) order */
} itt_loop_result;

typedef struct itt_analysis {
  itt_census census;          /* after the majority-device filter */
  uint32_t main_stream;
  uint32_t n_main_streams;    /* kernel-bearing streams (MultipleMainStreams warning when > 1) */
  int32_t main_stream_override_non_main; /* MainStreamOverride warning (pipeline.hpp:62-67) */
  int32_t pad_;
  uint64_t n_tokens;
  uint32_t n_names;
  uint64_t* name_row;         /* [n_names] source row carrying each token id's name */
  int64_t overlapping_kernels; /* count_interval_overlaps on the main stream */
  uint32_t n_loops;
  itt_loop_result* loops;
  itt_ctx* owner;             /* the context whose pinned blocks hold the rows (itt_free_analysis) */
} itt_analysis;

/* analyze_trace (pipeline.hpp:34-134) up to the per-loop integer aggregates; the
 * host finishes compute_summary / diagnose / warnings in reference order. */
int itt_analyze(itt_ctx* ctx, const itt_records* recs, const itt_analyze_opts* opts, itt_analysis** out);
int itt_free_analysis(itt_ctx* ctx, itt_analysis* a); /* ctx may be NULL: a->owner is used */

/* ------------------------------------------------------- batches of independent traces (C4)
 * A native executor: `workers` host threads, each with its own context (CUDA
 * stream + memory pool) on `device`, pull traces from a shared counter and run itt_analyze, so
 * the small, latency-bound traces overlap on the GPU with no interpreter in the loop.  Multi-GPU
 * sharding of a batch is the caller's (one executor per GPU, contiguous shards; no collective). */
typedef struct itt_batch itt_batch;
int itt_batch_create(int device, uint32_t workers, itt_batch** out);
int itt_batch_destroy(itt_batch* b);
/* out[i] and status[i] for trace i (status = itt_analyze's return code; on failure out[i] = NULL
 * and itt_batch_error(b, i) holds the message until the next call).  opts: one shared options
 * struct, or n structs when opts_per_trace != 0.  Returns ITT_OK when every trace ran (per-trace
 * failures are reported in status), else a context-creation error. */
int itt_batch_analyze(itt_batch* b, const itt_records* traces, uint64_t n, const itt_analyze_opts* opts,
                      int opts_per_trace, itt_analysis** out, int* status);
const char* itt_batch_error(itt_batch* b, uint64_t i);
/* kernels launched by the executor's worker contexts since creation */
int itt_batch_launch_count(itt_batch* b, uint64_t* out);
/* frees every non-NULL analysis (not concurrently with a running itt_batch_analyze) */
int itt_batch_free(itt_batch* b, itt_analysis** out, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif /* ITERTRACE_CUDA_H */
