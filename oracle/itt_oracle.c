/*
 * itt_oracle.c — CPU restatement of the reference hot path (see itt_oracle.h).
 * TEST INFRASTRUCTURE ONLY; never linked into the product.  Plain C11, single-threaded,
 * written for clarity over speed: it is the checker, not the thing measured.
 */
#include "itt_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_ERR(code, ...)                        \
  do {                                            \
    if (err && err_cap) snprintf(err, err_cap, __VA_ARGS__); \
    return (code);                                \
  } while (0)

void orc_free(void* p) { free(p); }

/* ------------------------------------------------ ingest ordering, ingest.hpp:396-400 */
static const int64_t* g_sort_start;
static int cmp_row_by_start(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  if (g_sort_start[x] != g_sort_start[y]) return g_sort_start[x] < g_sort_start[y] ? -1 : 1;
  return x < y ? -1 : (x > y); /* row tie-break == stability */
}
void orc_sort_records(uint64_t n, const int64_t* start, uint64_t* perm) {
  for (uint64_t i = 0; i < n; ++i) perm[i] = i;
  g_sort_start = start;
  qsort(perm, n, sizeof(uint64_t), cmp_row_by_start);
}

/* ------------------------------------------------ classify_op_kind, trace.hpp:81-113 */
static int lower(int c) { return (c >= 'A' && c <= 'Z') ? c + 32 : c; }
static int contains_ci(const uint8_t* h, uint64_t hl, const char* needle) {
  const uint64_t nl = strlen(needle);
  if (nl == 0) return 1;
  if (hl < nl) return 0;
  for (uint64_t i = 0; i + nl <= hl; ++i) {
    uint64_t j = 0;
    while (j < nl && lower(h[i + j]) == needle[j]) ++j;
    if (j == nl) return 1;
  }
  return 0;
}
int orc_classify(const uint8_t* name, uint64_t len, int has_tp) {
  if (contains_ci(name, len, "memcpy")) {
    if (contains_ci(name, len, "htod")) return ITT_KIND_HTOD;
    if (contains_ci(name, len, "dtoh")) return ITT_KIND_DTOH;
    if (contains_ci(name, len, "dtod")) return ITT_KIND_DTOD;
  }
  if (contains_ci(name, len, "memset")) return ITT_KIND_MEMSET;
  return has_tp ? ITT_KIND_OTHER : ITT_KIND_KERNEL;
}
static int kind_of(const itt_records* r, uint64_t i) {
  return orc_classify(r->name_bytes + r->name_off[i], r->name_off[i + 1] - r->name_off[i],
                      (r->flags[i] & ITT_REC_HAS_THROUGHPUT) != 0);
}
static uint16_t dev_of(const itt_records* r, uint64_t i) { return r->device ? r->device[i] : 0; }

/* ------------------------------------------------ filter_majority_device, streams.hpp:179-207 */
static int majority_device(const itt_records* r, uint16_t* maj, uint64_t* dropped) {
  uint64_t* cnt = calloc(65536, sizeof(uint64_t));
  uint32_t distinct = 0;
  for (uint64_t i = 0; i < r->n; ++i) distinct += cnt[dev_of(r, i)]++ == 0;
  uint64_t best = 0;
  *maj = 0;
  for (uint32_t d = 0; d < 65536; ++d) /* ascending label order; strict > keeps the smallest on ties */
    if (cnt[d] > best) best = cnt[d], *maj = (uint16_t)d;
  *dropped = distinct <= 1 ? 0 : r->n - best;
  free(cnt);
  return distinct > 1;
}

/* ------------------------------------------------ summarize + classify, streams.hpp:60-103 */
int orc_summarize_streams(const itt_records* r, int filter_device, itt_stream_summary* out, uint32_t cap,
                          uint32_t* n_out, uint64_t* dropped) {
  uint16_t maj = 0;
  int filtering = 0;
  *dropped = 0;
  if (filter_device) filtering = majority_device(r, &maj, dropped);
  uint32_t ns = 0;
  for (uint64_t i = 0; i < r->n; ++i) {
    if (filtering && dev_of(r, i) != maj) continue;
    uint32_t k = 0;
    while (k < ns && out[k].stream != r->stream[i]) ++k;
    const int64_t s = r->start_ns[i], e = s + r->duration_ns[i];
    if (k == ns) {
      if (ns == cap) return ITT_E_INVALID_ARGUMENT;
      memset(&out[ns], 0, sizeof(out[ns]));
      out[ns].stream = r->stream[i];
      out[ns].first_start = s;
      out[ns].last_end = e;
      ++ns;
    }
    out[k].counts[kind_of(r, i)] += 1;
    if (s < out[k].first_start) out[k].first_start = s;
    if (e > out[k].last_end) out[k].last_end = e;
  }
  if (ns == 0) return ITT_E_EMPTY_TRACE;
  /* std::map order: ascending stream id */
  for (uint32_t a = 1; a < ns; ++a)
    for (uint32_t b = a; b > 0 && out[b - 1].stream > out[b].stream; --b) {
      itt_stream_summary t = out[b];
      out[b] = out[b - 1];
      out[b - 1] = t;
    }
  for (uint32_t k = 0; k < ns; ++k) {
    const int64_t* c = out[k].counts;
    const int64_t total = c[0] + c[1] + c[2] + c[3] + c[4] + c[5];
    const int64_t mem = c[ITT_KIND_HTOD] + c[ITT_KIND_DTOH] + c[ITT_KIND_DTOD];
    int cls = ITT_CLASS_ASSIST;
    if (c[ITT_KIND_KERNEL] > 0) cls = ITT_CLASS_MAIN;
    else if (total > 0 && mem == total) {
      const int h = c[ITT_KIND_HTOD] > 0, d = c[ITT_KIND_DTOH] > 0, dd = c[ITT_KIND_DTOD] > 0;
      if (h && !d && !dd) cls = ITT_CLASS_COPY_HTOD;
      else if (d && !h && !dd) cls = ITT_CLASS_COPY_DTOH;
      else cls = ITT_CLASS_COPY_MIXED;
    }
    out[k].cls = cls;
  }
  *n_out = ns;
  return 0;
}

/* ------------------------------------------------ select_main_stream, streams.hpp:113-145 */
int orc_select_main_stream(const itt_stream_summary* s, uint32_t n, uint32_t* main_stream, uint32_t* n_main) {
  int found = 0;
  uint32_t best = 0;
  *n_main = 0;
  for (uint32_t k = 0; k < n; ++k) {
    if (s[k].cls != ITT_CLASS_MAIN) continue;
    ++*n_main;
    if (!found || s[k].counts[0] > s[best].counts[0] ||
        (s[k].counts[0] == s[best].counts[0] && s[k].stream < s[best].stream))
      best = k, found = 1;
  }
  if (!found) return ITT_E_NO_MAIN_STREAM;
  *main_stream = s[best].stream;
  return 0;
}

/* ------------------------------------------------ build_token_sequence, streams.hpp:147-169 */
typedef struct {
  uint64_t cap;
  uint64_t* row;  /* representative source row + 1 (0 = empty) */
  int32_t* id;
} name_map;
static uint64_t fnv(const uint8_t* p, uint64_t n) {
  uint64_t h = 1469598103934665603ull;
  for (uint64_t i = 0; i < n; ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}
int orc_build_token_sequence(const itt_records* r, uint32_t main_stream, int32_t* tokens, uint64_t* record_index,
                             uint64_t* n_out, uint32_t* n_names, uint64_t* name_row) {
  uint64_t* perm = malloc((r->n + 1) * sizeof(uint64_t));
  orc_sort_records(r->n, r->start_ns, perm);
  name_map m;
  m.cap = 1024;
  while (m.cap < 2 * r->n + 16) m.cap <<= 1;
  m.row = calloc(m.cap, sizeof(uint64_t));
  m.id = calloc(m.cap, sizeof(int32_t));
  uint64_t n = 0;
  uint32_t v = 0;
  for (uint64_t k = 0; k < r->n; ++k) {
    const uint64_t i = perm[k];
    if (r->stream[i] != main_stream) continue;
    const uint8_t* p = r->name_bytes + r->name_off[i];
    const uint64_t len = r->name_off[i + 1] - r->name_off[i];
    uint64_t s = fnv(p, len) & (m.cap - 1);
    for (;;) {
      if (m.row[s] == 0) { /* first appearance: next id (streams.hpp:152-157) */
        m.row[s] = i + 1;
        m.id[s] = (int32_t)v;
        if (name_row) name_row[v] = i;
        ++v;
        break;
      }
      const uint64_t j = m.row[s] - 1;
      const uint64_t lj = r->name_off[j + 1] - r->name_off[j];
      if (lj == len && memcmp(r->name_bytes + r->name_off[j], p, len) == 0) break;
      s = (s + 1) & (m.cap - 1);
    }
    tokens[n] = m.id[s];
    record_index[n] = k;
    ++n;
  }
  free(perm);
  free(m.row);
  free(m.id);
  if (n == 0) return ITT_E_EMPTY_MAIN_STREAM;
  *n_out = n;
  *n_names = v;
  return 0;
}

/* ------------------------------------------------ suffix array by prefix doubling */
typedef struct {
  int64_t a, b;
  uint32_t i;
} sa_item;
static int cmp_sa_item(const void* x, const void* y) {
  const sa_item* p = x;
  const sa_item* q = y;
  if (p->a != q->a) return p->a < q->a ? -1 : 1;
  if (p->b != q->b) return p->b < q->b ? -1 : 1;
  return 0;
}
int orc_suffix_array(const int32_t* tokens, uint64_t n, int32_t term, uint32_t* sa, uint32_t* lcp) {
  const uint64_t np = n + 1;
  int32_t* text = malloc(np * sizeof(int32_t));
  memcpy(text, tokens, n * sizeof(int32_t));
  text[n] = term;
  int64_t* rank = malloc(np * sizeof(int64_t));
  int64_t* tmp = malloc(np * sizeof(int64_t));
  sa_item* it = malloc(np * sizeof(sa_item));
  for (uint64_t i = 0; i < np; ++i) rank[i] = text[i];
  for (uint64_t h = 1;; h <<= 1) {
    for (uint64_t i = 0; i < np; ++i) {
      it[i].a = rank[i];
      it[i].b = i + h < np ? rank[i + h] : INT64_MIN; /* unique terminator: never decisive */
      it[i].i = (uint32_t)i;
    }
    qsort(it, np, sizeof(sa_item), cmp_sa_item);
    int64_t r = 0;
    for (uint64_t k = 0; k < np; ++k) {
      if (k > 0 && cmp_sa_item(&it[k - 1], &it[k]) != 0) ++r;
      tmp[it[k].i] = r;
    }
    memcpy(rank, tmp, np * sizeof(int64_t));
    if ((uint64_t)r == np - 1) break;
  }
  for (uint64_t k = 0; k < np; ++k) sa[k] = it[k].i;
  if (lcp) { /* Kasai */
    int64_t h = 0;
    for (uint64_t k = 0; k < np; ++k) tmp[sa[k]] = (int64_t)k;
    lcp[0] = 0;
    for (uint64_t i = 0; i < np; ++i) {
      const int64_t k = tmp[i];
      if (k > 0) {
        const uint64_t j = sa[k - 1];
        while (i + h < np && j + h < np && text[i + h] == text[j + h]) ++h;
        lcp[k] = (uint32_t)h;
        if (h > 0) --h;
      } else {
        h = 0;
      }
    }
  }
  free(text);
  free(rank);
  free(tmp);
  free(it);
  return 0;
}

/* ------------------------------------------------ enumerate_repeats, mine.hpp:46-60 */
/* Internal node <=> LCP interval [lb, rb] with depth l > 0 (leaf_count = rb-lb+1,
 * first_leaf = min SA[lb..rb], parent depth = the enclosing interval's depth).  One
 * bottom-up stack pass over the LCP array visits every internal node once. */
typedef struct {
  int64_t lcp, lb;
  uint32_t mn;
} stk_entry;
typedef void (*node_visit)(void* user, int64_t depth, int64_t lb, int64_t rb, uint32_t first_leaf, int64_t parent_depth);
static void for_each_internal_node(const uint32_t* sa, const uint32_t* lcp, uint64_t np, node_visit f, void* user) {
  stk_entry* st = malloc((np + 2) * sizeof(stk_entry));
  int64_t top = 0;
  st[0].lcp = 0;
  st[0].lb = 0;
  st[0].mn = sa[0];
  for (uint64_t i = 1; i <= np; ++i) {
    const int64_t l = i < np ? (int64_t)lcp[i] : 0;
    int64_t lb = (int64_t)i - 1;
    uint32_t carry = UINT32_MAX;
    int popped = 0;
    while (l < st[top].lcp) {
      stk_entry e = st[top--];
      const uint32_t full = e.mn < carry ? e.mn : carry;
      const int64_t parent = st[top].lcp > l ? st[top].lcp : l;
      f(user, e.lcp, e.lb, (int64_t)i - 1, full, parent);
      carry = full;
      lb = e.lb;
      popped = 1;
    }
    if (i == np) break;
    if (l > st[top].lcp) {
      ++top;
      st[top].lcp = l;
      st[top].lb = lb;
      st[top].mn = popped ? carry : sa[i - 1];
      if (!popped && sa[i - 1] < st[top].mn) st[top].mn = sa[i - 1];
    } else if (popped && carry < st[top].mn) {
      st[top].mn = carry;
    }
    if (sa[i] < st[top].mn) st[top].mn = sa[i];
  }
  free(st);
}

typedef struct {
  itt_repeat* v;
  uint64_t n, cap;
  int64_t min_count, max_len;
} rep_list;
static void collect_repeat(void* user, int64_t depth, int64_t lb, int64_t rb, uint32_t first_leaf, int64_t parent) {
  rep_list* L = user;
  const int64_t count = rb - lb + 1;
  if (count < L->min_count) return;
  const int64_t len = depth < L->max_len ? depth : L->max_len;
  if (len <= parent) return; /* mid-edge truncation must stay below the node (mine.hpp:53-54) */
  if (L->n == L->cap) {
    L->cap = L->cap ? 2 * L->cap : 64;
    L->v = realloc(L->v, L->cap * sizeof(itt_repeat));
  }
  L->v[L->n].start = (int32_t)first_leaf;
  L->v[L->n].length = (int32_t)len;
  L->v[L->n].count = count;
  ++L->n;
}
static int repeats_from_sa(const uint32_t* sa, const uint32_t* lcp, uint64_t np, int64_t min_count, int64_t max_len,
                           rep_list* L) {
  memset(L, 0, sizeof(*L));
  L->min_count = min_count;
  L->max_len = max_len;
  if (max_len < 1) return 0; /* mine.hpp:50 */
  for_each_internal_node(sa, lcp, np, collect_repeat, L);
  return 0;
}
int orc_enumerate_repeats(const int32_t* tokens, uint64_t n, int32_t term, int64_t min_count, int64_t max_len,
                          itt_repeat** out, uint64_t* n_out) {
  uint32_t* sa = malloc((n + 1) * sizeof(uint32_t));
  uint32_t* lcp = malloc((n + 1) * sizeof(uint32_t));
  orc_suffix_array(tokens, n, term, sa, lcp);
  rep_list L;
  repeats_from_sa(sa, lcp, n + 1, min_count, max_len, &L);
  free(sa);
  free(lcp);
  *out = L.v ? L.v : malloc(sizeof(itt_repeat));
  *n_out = L.n;
  return 0;
}

/* ------------------------------------------------ mine_pattern(s), mine.hpp:64-165 */
static int preferred(const itt_repeat* a, const itt_repeat* b) { /* candidate_preferred, mine.hpp:69-73 */
  if (a->length != b->length) return a->length > b->length;
  if (a->count != b->count) return a->count > b->count;
  return a->start < b->start;
}
static int mine_one(const int32_t* text, const uint32_t* sa, const uint32_t* lcp, uint64_t n, const itt_mining_cfg* cfg,
                    const char* label, itt_pattern* out, char* err, uint64_t err_cap) {
  const int64_t iters = cfg->iterations;
  if (iters < 2 || cfg->epsilon0 < 1 || cfg->epsilon0 >= iters)
    ORC_ERR(ITT_E_INVALID_ITERATION_COUNT,
            "pattern-mining%s: need iterations >= 2 and 1 <= epsilon0 < iterations (got iterations=%lld, epsilon0=%lld)",
            label, (long long)iters, (long long)cfg->epsilon0);
  if ((int64_t)n < iters)
    ORC_ERR(ITT_E_INVALID_ITERATION_COUNT, "pattern-mining%s: sequence of %lld operations cannot contain %lld iterations",
            label, (long long)n, (long long)iters);
  const int64_t cap = cfg->epsilon_cap > 0 ? cfg->epsilon_cap : iters;
  const int64_t max_len = ((int64_t)n - 1) / iters; /* mine.hpp:64-67 */
  for (int64_t eps = cfg->epsilon0; eps < cap; eps *= 2) {
    rep_list L;
    repeats_from_sa(sa, lcp, n + 1, iters - eps + 1, max_len, &L);
    const itt_repeat* best = NULL;
    for (uint64_t k = 0; k < L.n; ++k) {
      if (L.v[k].count > iters) continue;
      if (!best || preferred(&L.v[k], best)) best = &L.v[k];
    }
    if (best) {
      out->length = best->length;
      out->tokens = malloc((size_t)best->length * sizeof(int32_t) + 4);
      memcpy(out->tokens, text + best->start, (size_t)best->length * sizeof(int32_t));
      out->count = best->count;
      out->first_token = best->start;
      out->epsilon_used = eps;
      free(L.v);
      return 0;
    }
    free(L.v);
  }
  ORC_ERR(ITT_E_NO_PATTERN_FOUND,
          "pattern-mining%s: no repeated substring satisfies the repetition and length criteria for iterations=%lld "
          "(epsilon exhausted at cap %lld); the trace may not be iterative at the declared count",
          label, (long long)iters, (long long)cap);
}

int orc_mine_patterns(const int32_t* tokens, uint64_t n, uint32_t n_names, const itt_mining_cfg* loops,
                      uint32_t n_loops, int multi, itt_pattern* out, char* err, uint64_t err_cap) {
  if (multi) {
    if (n_loops == 0) ORC_ERR(ITT_E_INVALID_CONFIG, "pattern-mining: no loop specs given");
    for (uint32_t a = 0; a < n_loops; ++a)
      for (uint32_t b = 0; b < a; ++b)
        if (loops[a].iterations == loops[b].iterations)
          ORC_ERR(ITT_E_INVALID_CONFIG, "pattern-mining: loop iteration counts must be pairwise distinct (duplicate %lld)",
                  (long long)loops[a].iterations);
  }
  uint32_t* sa = malloc((n + 1) * sizeof(uint32_t));
  uint32_t* lcp = malloc((n + 1) * sizeof(uint32_t));
  orc_suffix_array(tokens, n, (int32_t)n_names, sa, lcp); /* terminator = names.size(), mine.hpp:38-40 */
  int rc = 0;
  uint32_t done = 0;
  for (uint32_t k = 0; k < (multi ? n_loops : 1u); ++k) {
    char label[32] = "";
    if (multi) snprintf(label, sizeof(label), " (loop %u)", k + 1);
    rc = mine_one(tokens, sa, lcp, n, &loops[k], label, &out[k], err, err_cap);
    if (rc) break;
    ++done;
  }
  if (!rc && multi)
    for (uint32_t a = 0; a < n_loops && !rc; ++a)
      for (uint32_t b = a + 1; b < n_loops && !rc; ++b)
        if (out[a].length == out[b].length &&
            memcmp(out[a].tokens, out[b].tokens, (size_t)out[a].length * sizeof(int32_t)) == 0) {
          if (err && err_cap)
            snprintf(err, err_cap,
                     "pattern-mining: loops %u and %u mined the same pattern; the loop specs are ambiguous", a + 1, b + 1);
          rc = ITT_E_AMBIGUOUS_LOOPS;
        }
  if (rc)
    for (uint32_t k = 0; k < done; ++k) free(out[k].tokens), out[k].tokens = NULL;
  free(sa);
  free(lcp);
  return rc;
}

/* ------------------------------------------------ approx_match, match.hpp:41-85 */
int orc_approx_match(const int32_t* s, uint64_t n_, const int32_t* p, uint64_t m_, int64_t k0, itt_span** out,
                     uint64_t* n_out) {
  const int64_t n = (int64_t)n_, m = (int64_t)m_;
  uint64_t cap = 64, cnt = 0;
  itt_span* v = malloc(cap * sizeof(itt_span));
  if (m > 0 && n >= m) {
    int64_t anchor = 0;
    while (anchor < n) {
      if (s[anchor] != p[0]) {
        ++anchor;
        continue;
      }
      int64_t pos = anchor, matched = 0, extra = 0, last = anchor;
      int complete = 1;
      while (matched < m) {
        if (pos == n) {
          complete = 0;
          break;
        }
        if (s[pos] == p[matched]) {
          last = pos;
          ++matched;
          ++pos;
        } else {
          if (++extra > k0) {
            complete = 0;
            break;
          }
          ++pos;
        }
      }
      if (complete) {
        if (cnt == cap) v = realloc(v, (cap *= 2) * sizeof(itt_span));
        v[cnt].start_token = anchor;
        v[cnt].end_token = last;
        v[cnt].extra = extra;
        ++cnt;
        anchor = last + 1;
      } else {
        ++anchor;
      }
    }
  }
  *out = v;
  *n_out = cnt;
  return 0;
}

/* ------------------------------------------------ iteration metrics, metrics.hpp:44-164 */
typedef struct {
  int64_t a, b;
} seg;
static int cmp_seg(const void* x, const void* y) {
  const seg* p = x;
  const seg* q = y;
  if (p->a != q->a) return p->a < q->a ? -1 : 1;
  return p->b < q->b ? -1 : (p->b > q->b);
}
int orc_iteration_metrics(const itt_records* r, uint32_t main_stream, const itt_span* spans, uint64_t I, ref_iter* rows,
                          itt_clamps* clamps) {
  uint64_t* perm = malloc((r->n + 1) * sizeof(uint64_t));
  orc_sort_records(r->n, r->start_ns, perm);
  /* record_index of main-stream tokens (streams.hpp:147-169) and HtoD records (metrics.hpp:57-63) */
  uint64_t* tok = malloc((r->n + 1) * sizeof(uint64_t));
  uint64_t* htod = malloc((r->n + 1) * sizeof(uint64_t));
  uint64_t nt = 0, H = 0;
  for (uint64_t k = 0; k < r->n; ++k) {
    const uint64_t i = perm[k];
    if (r->stream[i] == main_stream) tok[nt++] = i;
    if (kind_of(r, i) == ITT_KIND_HTOD) htod[H++] = i;
  }
  seg* segs = malloc((H + 1) * sizeof(seg));
  memset(clamps, 0, sizeof(*clamps));
  int64_t prev_end = 0;
  for (uint64_t k = 0; k < I; ++k) {
    const uint64_t f = tok[spans[k].start_token], l = tok[spans[k].end_token];
    const int64_t t_start = r->start_ns[f], t_end = r->start_ns[l] + r->duration_ns[l];
    ref_iter* o = &rows[k];
    memset(o, 0, sizeof(*o));
    o->index = (int64_t)k + 1;
    o->start_token = spans[k].start_token;
    o->end_token = spans[k].end_token;
    o->extra = spans[k].extra;
    o->t_start = t_start;
    o->t_end = t_end;
    if (k > 0) {
      int64_t interval = t_start - prev_end;
      if (interval < 0) {
        interval = 0;
        ++clamps->negative_interval_clamps;
      }
      o->has_interval = 1;
      o->interval_ns = interval;
      if (interval > 0) { /* clipped_union_length, metrics.hpp:76-100 */
        const int64_t lo = prev_end, hi = t_start;
        uint64_t ns = 0;
        for (uint64_t h = 0; h < H; ++h) {
          const uint64_t i = htod[h];
          const int64_t a = r->start_ns[i] > lo ? r->start_ns[i] : lo;
          const int64_t e = r->start_ns[i] + r->duration_ns[i];
          const int64_t b = e < hi ? e : hi;
          if (b > a) segs[ns].a = a, segs[ns].b = b, ++ns;
        }
        qsort(segs, ns, sizeof(seg), cmp_seg);
        int64_t total = 0, cl = 0, ch = 0;
        int open = 0;
        for (uint64_t q = 0; q < ns; ++q) {
          if (!open || segs[q].a > ch) {
            if (open) total += ch - cl;
            cl = segs[q].a;
            ch = segs[q].b;
            open = 1;
          } else if (segs[q].b > ch) {
            ch = segs[q].b;
          }
        }
        if (open) total += ch - cl;
        o->has_overlap = 1;
        o->overlap_ratio = (double)total / (double)interval;
      }
    }
    const int64_t lo_b = k > 0 ? prev_end : -1; /* metrics.hpp:138-143 */
    for (uint64_t h = 0; h < H; ++h) {
      const uint64_t i = htod[h];
      if (r->start_ns[i] > lo_b && r->start_ns[i] <= t_end)
        o->htod_bytes += (r->flags[i] & ITT_REC_HAS_SIZE) ? r->size_bytes[i] : 0;
    }
    int64_t gap_sum = 0, gap_count = 0; /* metrics.hpp:145-160 */
    for (int64_t t = spans[k].start_token; t < spans[k].end_token; ++t) {
      const uint64_t c = tok[t], x = tok[t + 1];
      int64_t gap = r->start_ns[x] - (r->start_ns[c] + r->duration_ns[c]);
      if (gap < 0) {
        gap = 0;
        ++clamps->negative_gap_clamps;
      }
      gap_sum += gap;
      ++gap_count;
    }
    o->op_gap_mean_ns = gap_count > 0 ? (double)gap_sum / (double)gap_count : 0.0;
    prev_end = t_end;
  }
  free(perm);
  free(tok);
  free(htod);
  free(segs);
  return 0;
}

/* ---- a12 per-op profile.  No reference function exists: this restates the
 * definition in include/itertrace_cuda.h (itt_op_cell) with plain loops — the reference's own
 * pieces it builds on are the spans (match.hpp:41-85) and the clamped op gap
 * (metrics.hpp:145-157: max(0, start[j+1] - end[j]) for j in [s, e)). */
static int cmp_u32(const void* x, const void* y) {
  const uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
  return a < b ? -1 : a > b;
}

int orc_op_profile(const int32_t* tokens, const int64_t* tok_start, const int64_t* tok_end, const uint8_t* tok_kind,
                   uint64_t n, uint32_t n_ops, const itt_span* spans, uint64_t I, itt_op_cell** out, uint64_t* n_out) {
  *out = NULL;
  *n_out = 0;
  for (uint64_t j = 0; j < n; ++j)
    if (tokens[j] < 0 || (uint32_t)tokens[j] >= n_ops) return ITT_E_INVALID_ARGUMENT;
  uint32_t* cnt = calloc(n_ops + 1, sizeof(uint32_t));
  int64_t* kern = calloc(n_ops + 1, sizeof(int64_t));
  int64_t* mem = calloc(n_ops + 1, sizeof(int64_t));
  int64_t* idle = calloc(n_ops + 1, sizeof(int64_t));
  uint32_t* touched = malloc((n_ops + 1) * sizeof(uint32_t));
  uint64_t cap = 16, m = 0;
  itt_op_cell* cells = malloc(cap * sizeof(itt_op_cell));
  for (uint64_t k = 0; k < I; ++k) {
    const uint64_t s = (uint64_t)spans[k].start_token, e = (uint64_t)spans[k].end_token;
    uint32_t nt = 0;
    for (uint64_t j = s; j <= e; ++j) {
      const uint32_t v = (uint32_t)tokens[j];
      if (cnt[v]++ == 0) touched[nt++] = v;
      const int64_t d = tok_end[j] - tok_start[j];
      if (tok_kind[j] == ITT_KIND_KERNEL) kern[v] += d;
      else mem[v] += d;
      if (j > s) { /* the gap in front of op j inside the iteration */
        const int64_t g = tok_start[j] - tok_end[j - 1];
        if (g > 0) idle[v] += g;
      }
    }
    qsort(touched, nt, sizeof(uint32_t), cmp_u32);
    for (uint32_t q = 0; q < nt; ++q) {
      const uint32_t v = touched[q];
      if (m == cap) {
        cap *= 2;
        cells = realloc(cells, cap * sizeof(itt_op_cell));
      }
      itt_op_cell* c = &cells[m++];
      c->iteration = (uint32_t)k;
      c->op = (int32_t)v;
      c->count = cnt[v];
      c->pad_ = 0;
      c->kernel_ns = kern[v];
      c->memcpy_ns = mem[v];
      c->idle_ns = idle[v];
      cnt[v] = 0, kern[v] = 0, mem[v] = 0, idle[v] = 0;
    }
  }
  free(cnt), free(kern), free(mem), free(idle), free(touched);
  *out = cells;
  *n_out = m;
  return 0;
}
