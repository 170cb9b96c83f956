// ingest.cu — profiler CSV text -> columnar records on the GPU, sm_100a.
//
// parse_trace_text (ingest.hpp:154-402): the header row, the optional units row and comment /
// blank lines before them are a handful of lines and are read by the host (capi.cu); every data
// line is parsed here, one thread per line, with the reference's exact rules:
//   * fields split RFC-style: commas inside quotes, doubled quotes (split_csv, ingest.hpp:104-131),
//     cells trimmed of ' ' and '\t' (trim, :133-137);
//   * an inline unit suffix overrides the column unit (split_inline_unit, :140-149);
//   * times and sizes: parse_scaled_decimal (:66-100) — at most 18 digits, round-half-up of
//     digits * factor / 10^frac in 128-bit integers;
//   * Stream: decimal digits <= UINT32_MAX (:330-343); Throughput: only its presence reaches the
//     analysis, but std::stod's acceptance decides whether the row is skipped (:263-277), so the
//     strtod grammar (decimal and hex forms, nan/inf) and its ERANGE boundaries (results that
//     overflow, or decimal results below DBL_MIN) are decided exactly with integer arithmetic;
//   * skip order: empty Name, Start, Duration, Stream, Size, Throughput (:318-371).
// Lines are found with one newline-count scan; the records are compacted in line order (the
// pipeline's order stage sorts by (start, row) like ingest.hpp:396-400).
#include <algorithm>
#include <cstring>

#include "pipeline.cuh"
#include "ingest.cuh"

namespace itt {

namespace {

// exact thresholds of strtod's ERANGE: value >= 2^1024 - 2^970 overflows; a nonzero decimal value
// below 2^-1022 - 2^-1075 rounds to a subnormal.  Significant digits of 0.D x 10^E.
__device__ const char kTmaxDigits[] =
    "17976931348623158079372897140530341507993413271003782693617377898044496829276475094664901797758720709633028641"
    "66928879109465555478519404026306574886715058206819089020007083836762738548458177115317644757302700698555713669"
    "59622842914819860834936475292719074168444365510704342711559699508093042880177904174497792";
constexpr int kTmaxExp = 309;
__device__ const char kTminDigits[] =
    "22250738585072011360574097967091319759348195463516456480234261097248222220210769455165295239081350879141491589"
    "13039621106870086438694594645527657207407820621743379988141063267329253552286881372149012981122451451889849057"
    "22230728525513315575501591439747639798341180199932396254828901710708185069063066665599493827577257201576306269"
    "06633326475653000092458883164330377797918696120494973903778297049050510806099407302629371289589500035837999672"
    "07254304360284078895771796150945516748243471030702609144621572289880258182545180325707018860872113128079512233"
    "42628836862232150377566662250398253433597456888442390026549819838548794829220689472168983109969836584681402285"
    "424333066033985088644580400103493397042756718644338377048603786162277173854562306587467901408672332763671875";
constexpr int kTminExp = -307;

// unescaped characters of one field (split_csv semantics; a field starts unquoted)
struct CellIter {
  const uint8_t* t;
  uint64_t i, e;
  bool quoted;
  __device__ CellIter(const uint8_t* text, uint64_t b, uint64_t end) : t(text), i(b), e(end), quoted(false) {}
  __device__ __forceinline__ bool next(uint8_t& c) {
    while (i < e) {
      const uint8_t x = t[i++];
      if (quoted) {
        if (x == '"') {
          if (i < e && t[i] == '"') {
            ++i;
            c = '"';
            return true;
          }
          quoted = false;
          continue;
        }
        c = x;
        return true;
      }
      if (x == '"') {
        quoted = true;
        continue;
      }
      c = x;
      return true;
    }
    return false;
  }
};

__device__ __forceinline__ bool is_ws(uint8_t c) { return c == ' ' || c == '\t'; }
__device__ __forceinline__ bool is_unit_char(uint8_t c) {
  return (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || c == '/';
}

// one pass over a cell: trimmed extent [first, last] (unescaped indices; first > last when the
// cell is empty after trim), the trailing unit run (last_num = last index of the number part),
// and the unit's characters (at most 8 kept)
struct CellShape {
  int64_t len = 0, first = -1, last = -2, last_num = -2;
  uint8_t unit[8];
  int unit_len = 0;
  bool unit_long = false;
};
__device__ CellShape cell_shape(CellIter it) {
  CellShape s;
  uint8_t c;
  int64_t k = 0;
  // unit run tracking: the run resets on every non-unit char that is not (yet) known trailing ws
  int run_len = 0;
  bool run_long = false;
  int64_t last_nonunit = -1;  // last index of a non-unit char before the pending ws
  int64_t pending_ws = -1;    // start of a trailing whitespace stretch (-1: none)
  uint8_t run[8];
  for (; it.next(c); ++k) {
    if (is_ws(c)) {
      if (s.first < 0) continue;  // leading
      if (pending_ws < 0) pending_ws = k;
      continue;
    }
    if (s.first < 0) s.first = k;
    if (pending_ws >= 0) {  // internal whitespace: part of the cell, not a unit char
      last_nonunit = k - 1;
      run_len = 0, run_long = false;
      pending_ws = -1;
    }
    s.last = k;
    if (is_unit_char(c)) {
      if (run_len < 8) run[run_len++] = c;
      else run_long = true;
    } else {
      last_nonunit = k;
      run_len = 0, run_long = false;
    }
  }
  s.len = k;
  if (s.first < 0) return s;  // empty after trim
  s.last_num = last_nonunit;  // number part: [first, last_num]
  s.unit_len = run_len;
  s.unit_long = run_long;
  for (int q = 0; q < run_len; ++q) s.unit[q] = run[q];
  return s;
}

__device__ bool unit_is(const CellShape& s, const char* u) {
  int n = 0;
  while (u[n]) ++n;
  if (s.unit_long || s.unit_len != n) return false;
  for (int q = 0; q < n; ++q)
    if (s.unit[q] != static_cast<uint8_t>(u[q])) return false;
  return true;
}
__device__ int64_t time_factor(const CellShape& s) {  // 0: not a time unit (ingest.hpp:35-41)
  if (unit_is(s, "s")) return 1000000000;
  if (unit_is(s, "ms")) return 1000000;
  if (unit_is(s, "us")) return 1000;
  if (unit_is(s, "ns")) return 1;
  return 0;
}
__device__ int64_t size_factor(const CellShape& s) {  // ingest.hpp:43-49
  if (unit_is(s, "B")) return 1;
  if (unit_is(s, "KB")) return 1024;
  if (unit_is(s, "MB")) return 1024 * 1024;
  if (unit_is(s, "GB")) return 1024LL * 1024 * 1024;
  return 0;
}
__device__ bool tp_unit_ok(const CellShape& s) {  // ingest.hpp:51-57
  return unit_is(s, "B/s") || unit_is(s, "KB/s") || unit_is(s, "MB/s") || unit_is(s, "GB/s");
}

// the unescaped characters [a, b] of a cell (a <= b), re-walked from the field start
struct SubIter {
  CellIter it;
  int64_t k = 0, a, b;
  __device__ SubIter(CellIter c, int64_t a_, int64_t b_) : it(c), a(a_), b(b_) {
    uint8_t x;
    while (k < a && it.next(x)) ++k;
  }
  __device__ __forceinline__ bool next(uint8_t& c) {
    if (k > b) return false;
    if (!it.next(c)) return false;
    ++k;
    return true;
  }
};

// parse_scaled_decimal (ingest.hpp:66-100) over the number part
__device__ bool scaled_decimal(SubIter s, int64_t factor, int64_t& out) {
  uint8_t c;
  bool have = s.next(c);
  bool negative = false;
  if (have && (c == '+' || c == '-')) {
    negative = c == '-';
    have = s.next(c);
  }
  unsigned __int128 digits = 0;
  int n_digits = 0, n_frac = 0;
  bool seen_point = false, seen_digit = false;
  for (; have; have = s.next(c)) {
    if (c == '.') {
      if (seen_point) return false;
      seen_point = true;
      continue;
    }
    if (c < '0' || c > '9') return false;
    seen_digit = true;
    if (++n_digits > 18) return false;
    digits = digits * 10 + static_cast<unsigned>(c - '0');
    if (seen_point) ++n_frac;
  }
  if (!seen_digit) return false;
  unsigned __int128 scale = 1;
  for (int k = 0; k < n_frac; ++k) scale *= 10;
  const unsigned __int128 scaled = digits * static_cast<unsigned __int128>(factor);
  const unsigned __int128 rounded = (scaled + scale / 2) / scale;
  if (rounded > static_cast<unsigned __int128>(INT64_MAX)) return false;
  const int64_t mag = static_cast<int64_t>(rounded);
  out = negative ? -mag : mag;
  return true;
}

// parse_time_cell / parse_size_cell: inline unit overrides the column factor
__device__ bool time_cell(const CellIter& it, const CellShape& s, int64_t column_factor, int64_t& out) {
  if (s.first < 0) return false;  // empty
  int64_t f = column_factor;
  if (s.last_num < s.last) {
    f = time_factor(s);
    if (!f) return false;
  }
  if (s.last_num < s.first) return false;  // no number part
  return scaled_decimal(SubIter(it, s.first, s.last_num), f, out);
}
__device__ bool size_cell(const CellIter& it, const CellShape& s, int64_t column_factor, int64_t& out) {
  int64_t f = column_factor;
  if (s.last_num < s.last) {
    f = size_factor(s);
    if (!f) return false;
  }
  if (s.last_num < s.first) return false;
  return scaled_decimal(SubIter(it, s.first, s.last_num), f, out);
}

// compare the significant digits of a cell (streamed: skip sign / point / leading zeros, stop at
// the exponent marker) with a threshold 0.D x 10^e; -1 less, 0 equal, 1 greater
template <typename It>
__device__ int cmp_digits(It s, bool hex_exp_marker, const char* d) {
  uint8_t c;
  bool started = false;
  int i = 0;
  while (s.next(c)) {
    if (c == '+' || c == '-' || c == '.') continue;
    if (c == 'e' || c == 'E' || (hex_exp_marker && (c == 'p' || c == 'P'))) break;
    if (!started && c == '0') continue;
    started = true;
    const char dc = d[i];
    if (!dc) {
      if (c != '0') return 1;  // threshold digits exhausted: any further nonzero digit is more
      continue;
    }
    if (c != static_cast<uint8_t>(dc)) return c > static_cast<uint8_t>(dc) ? 1 : -1;
    ++i;
  }
  return d[i] ? -1 : 0;  // remaining threshold digits are nonzero (digit strings end in a nonzero digit)
}

// std::stod acceptance of the number part, fully consumed, finite and >= 0, no ERANGE
// (ingest.hpp:269-276 with glibc strtod semantics)
__device__ bool stod_ok(const CellIter& it, int64_t a, int64_t b) {
  if (a > b) return false;  // std::stod("") throws invalid_argument
  SubIter s(it, a, b);
  uint8_t c;
  bool have = s.next(c);
  int64_t pos = a;
  // strtod skips leading isspace (the cell was trimmed of ' ' and '\t' only)
  while (have && (c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r')) have = s.next(c), ++pos;
  bool neg = false;
  if (have && (c == '+' || c == '-')) {
    neg = c == '-';
    have = s.next(c);
    ++pos;
  }
  if (!have) return false;
  const int64_t body = pos;  // first char after the sign
  auto lower = [](uint8_t x) -> uint8_t { return (x >= 'A' && x <= 'Z') ? x + 32 : x; };
  const uint8_t l0 = lower(c);
  if (l0 == 'i' || l0 == 'n') return false;  // inf / infinity / nan(...): never finite and >= 0
  // hex form: "0x" followed by at least one hex digit (else strtod stops after the "0")
  if (c == '0') {
    SubIter h(it, body, b);
    uint8_t x0, x1, x2;
    h.next(x0);
    if (h.next(x1) && lower(x1) == 'x') {
      bool hd = h.next(x2);
      auto is_hex = [&](uint8_t x) { return (x >= '0' && x <= '9') || (lower(x) >= 'a' && lower(x) <= 'f'); };
      if (hd && (is_hex(x2) || x2 == '.')) {
        // [hex digits][.hex digits] then optional p[sign]digits; must consume everything
        uint64_t m = 0;        // first 16 significant hex digits
        int sig = 0;           // significant hex digits taken into m
        bool sticky = false;   // nonzero digits beyond them
        int64_t scale4 = 0;    // value = m * 16^scale4 (before the binary exponent)
        bool any = false, point = false;
        uint8_t x = x2;
        bool more = true;
        for (; more; more = h.next(x)) {
          if (x == '.') {
            if (point) return false;
            point = true;
            continue;
          }
          if (!is_hex(x)) break;
          any = true;
          const int v = (x <= '9') ? x - '0' : lower(x) - 'a' + 10;
          if (sig == 0 && v == 0) {
            if (point) --scale4;
            continue;
          }
          if (sig < 16) {
            m = m * 16 + static_cast<uint64_t>(v);
            ++sig;
            if (point) --scale4;
          } else {
            if (v) sticky = true;
            if (!point) ++scale4;
          }
        }
        if (!any) return false;
        int64_t bexp = 0;
        if (more) {  // x is the first char after the mantissa
          if (lower(x) != 'p') return false;
          uint8_t y;
          if (!h.next(y)) return false;  // "p" without digits is not consumed
          bool eneg = false;
          if (y == '+' || y == '-') {
            eneg = y == '-';
            if (!h.next(y)) return false;
          }
          if (y < '0' || y > '9') return false;
          int64_t ev = 0;
          bool emore = true;
          for (; emore; emore = h.next(y)) {
            if (y < '0' || y > '9') return false;
            if (ev < 100000000) ev = ev * 10 + (y - '0');
          }
          bexp = eneg ? -ev : ev;
        }
        if (m == 0) return true;  // zero (signed zero is >= 0)
        if (neg) return false;
        // value = m * 2^(4*scale4 + bexp) (+ sticky below m's last digit)
        const int top = 63 - __clzll(static_cast<long long>(m));  // leading bit of m
        const int64_t B = top + 4 * scale4 + bexp;                 // binary exponent of the value
        if (B >= 1024) return false;
        if (B == 1023) {  // overflow iff the 54 bits from the leading one are all ones
          if (top >= 53) {
            const uint64_t want = (1ull << 54) - 1;
            if (((m >> (top - 53)) & want) == want) return false;
          }
          return true;
        }
        if (B >= -1022) return true;
        // subnormal region: ERANGE unless exact (no bits below 2^-1074) — values rounding up to
        // DBL_MIN (>= 2^-1022 - 2^-1075) are normal results
        if (B == -1023 && top >= 52) {
          const uint64_t want = (1ull << 53) - 1;
          if (((m >> (top - 52)) & want) == want) return true;  // >= the midpoint below DBL_MIN
        }
        const int64_t low = 4 * scale4 + bexp;  // weight exponent of m's lowest bit
        if (sticky) return false;
        if (low >= -1074) return true;
        const int64_t drop = -1074 - low;       // bits of m below 2^-1074
        if (drop >= 64) return false;
        return (m & ((1ull << drop) - 1)) == 0;
      }
      // "0x" with no hex digit: strtod consumes only "0"
      return false;
    }
  }
  // decimal: digits* [. digits*] with at least one digit, [e [sign] digits+]
  int64_t int_digits = 0, frac_digits = 0, lead_zeros = 0, lead_frac_zeros = 0;
  bool any = false, point = false, nonzero = false;
  bool more = true;
  for (; more; more = s.next(c)) {
    if (c == '.') {
      if (point) return false;
      point = true;
      continue;
    }
    if (c < '0' || c > '9') break;
    any = true;
    if (!point) {
      ++int_digits;
      if (!nonzero && c == '0') ++lead_zeros;
    } else {
      ++frac_digits;
      if (!nonzero && c == '0') ++lead_frac_zeros;
    }
    if (c != '0') nonzero = true;
  }
  if (!any) return false;
  int64_t e10 = 0;
  if (more) {
    if (c != 'e' && c != 'E') return false;
    uint8_t y;
    if (!s.next(y)) return false;  // "e" without digits is not consumed
    bool eneg = false;
    if (y == '+' || y == '-') {
      eneg = y == '-';
      if (!s.next(y)) return false;
    }
    if (y < '0' || y > '9') return false;
    int64_t ev = 0;
    bool emore = true;
    for (; emore; emore = s.next(y)) {
      if (y < '0' || y > '9') return false;
      if (ev < 100000000) ev = ev * 10 + (y - '0');
    }
    e10 = eneg ? -ev : ev;
  }
  if (!nonzero) return true;  // zero (a "-0" is >= 0)
  if (neg) return false;
  // value = 0.S x 10^E with S the significant digits
  const int64_t E = (int_digits > lead_zeros) ? (int_digits - lead_zeros) + e10 : -lead_frac_zeros + e10;
  if (E > kTmaxExp) return false;
  if (E == kTmaxExp && cmp_digits(SubIter(it, body, b), false, kTmaxDigits) >= 0) return false;
  if (E < kTminExp) return false;
  if (E == kTminExp && cmp_digits(SubIter(it, body, b), false, kTminDigits) < 0) return false;
  return true;
}

__device__ bool stream_cell(CellIter it, uint32_t& out) {  // ingest.hpp:330-343 on the trimmed cell
  uint8_t c;
  bool started = false, trailing = false;
  uint64_t v = 0;
  while (it.next(c)) {
    if (is_ws(c)) {
      if (started) trailing = true;
      continue;
    }
    if (trailing) return false;  // internal whitespace is part of the trimmed cell
    if (c < '0' || c > '9') return false;
    started = true;
    v = v * 10 + static_cast<unsigned>(c - '0');
    if (v > UINT32_MAX) return false;
  }
  if (!started) return false;
  out = static_cast<uint32_t>(v);
  return true;
}

__device__ __forceinline__ uint64_t fnv_mix(uint64_t h, uint8_t c) { return (h ^ c) * 0x100000001b3ull; }

}  // namespace

// One thread per data line (lines [first_line, n_lines)).
__global__ void k_parse_lines(IngestArgs a) {
  const uint64_t ln = a.first_line + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (ln >= a.n_lines) return;
  const uint64_t k = ln - a.first_line;
  uint64_t b = ln == 0 ? 0 : a.nl[ln - 1] + 1;
  uint64_t e = ln < a.n_nl ? a.nl[ln] : a.len;
  if (e > b && a.text[e - 1] == '\r') --e;
  LineOut o{};
  // blank (after trim) and "==" comment lines are not data rows (ingest.hpp:290-291)
  bool blank = true;
  for (uint64_t i = b; i < e; ++i)
    if (!is_ws(a.text[i])) {
      blank = false;
      break;
    }
  if (blank || (e - b >= 2 && a.text[b] == '=' && a.text[b + 1] == '=')) {
    o.status = kLineIgnore;
    a.out[k] = o;
    return;
  }
  // field spans of the columns of interest (split_csv, ingest.hpp:104-131)
  uint64_t fb[kIngestCols], fe[kIngestCols];
  for (int q = 0; q < kIngestCols; ++q) fb[q] = fe[q] = 0;
  {
    bool quoted = false;
    int f = 0;
    uint64_t start = b;
    for (uint64_t i = b; i <= e; ++i) {
      const bool end = i == e;
      const uint8_t c = end ? ',' : a.text[i];
      if (!end && quoted) {
        if (c == '"') {
          if (i + 1 < e && a.text[i + 1] == '"') ++i;
          else quoted = false;
        }
        continue;
      }
      if (!end && c == '"') {
        quoted = true;
        continue;
      }
      if (c == ',') {
        for (int q = 0; q < kIngestCols; ++q)
          if (a.col[q] == f) fb[q] = start, fe[q] = i;
        ++f;
        start = i + 1;
      }
    }
  }
  auto cell = [&](int q) { return CellIter(a.text, fb[q], fe[q]); };  // absent column: empty span
  // Name (empty -> skip)
  const CellShape sn = cell_shape(cell(kColName));
  if (sn.first < 0) {
    o.status = kLineSkip, o.reason = kSkipName;
    a.out[k] = o;
    return;
  }
  int64_t start, dur;
  const CellShape ss = cell_shape(cell(kColStart));
  if (!time_cell(cell(kColStart), ss, a.start_factor, start) || start < 0) {
    o.status = kLineSkip, o.reason = kSkipStart;
    a.out[k] = o;
    return;
  }
  const CellShape sd = cell_shape(cell(kColDuration));
  if (!time_cell(cell(kColDuration), sd, a.duration_factor, dur) || dur < 0) {
    o.status = kLineSkip, o.reason = kSkipDuration;
    a.out[k] = o;
    return;
  }
  uint32_t stream = 0;
  if (!stream_cell(cell(kColStream), stream)) {
    o.status = kLineSkip, o.reason = kSkipStream;
    a.out[k] = o;
    return;
  }
  uint8_t flags = 0;
  int64_t size = 0;
  const CellShape sz = cell_shape(cell(kColSize));
  if (sz.first >= 0) {
    if (!size_cell(cell(kColSize), sz, a.size_factor, size) || size < 0) {
      o.status = kLineSkip, o.reason = kSkipSize;
      a.out[k] = o;
      return;
    }
    flags |= ITT_REC_HAS_SIZE;
  }
  const CellShape st = cell_shape(cell(kColThroughput));
  if (st.first >= 0) {
    const bool unit_ok = st.last_num == st.last || tp_unit_ok(st);
    if (!unit_ok || !stod_ok(cell(kColThroughput), st.first, st.last_num)) {
      o.status = kLineSkip, o.reason = kSkipThroughput;
      a.out[k] = o;
      return;
    }
    flags |= ITT_REC_HAS_THROUGHPUT;
  }
  // device label: hash of the trimmed cell ("unknown" when absent or empty)
  const CellShape sv = cell_shape(cell(kColDevice));
  uint64_t dh = 0xcbf29ce484222325ull;
  uint32_t dlen = 0;
  if (sv.first >= 0) {
    SubIter d(cell(kColDevice), sv.first, sv.last);
    uint8_t c;
    while (d.next(c)) dh = fnv_mix(dh, c), ++dlen;
  } else {
    for (const char* u = "unknown"; *u; ++u) dh = fnv_mix(dh, static_cast<uint8_t>(*u)), ++dlen;
  }
  o.status = kLineRecord;
  o.flags = flags;
  o.stream = stream;
  o.start = start;
  o.dur = dur;
  o.size = size;
  o.name_b = fb[kColName], o.name_e = fe[kColName];
  o.name_first = static_cast<uint32_t>(sn.first);
  o.name_len = static_cast<uint32_t>(sn.last - sn.first + 1);
  o.dev_b = fb[kColDevice], o.dev_e = fe[kColDevice];
  o.dev_first = sv.first >= 0 ? static_cast<uint32_t>(sv.first) : 0;
  o.dev_len = sv.first >= 0 ? dlen : 0;  // 0: "unknown"
  o.dev_hash = dh;
  a.out[k] = o;
}

// the trimmed, unescaped Name / Device cell bytes of record r
__global__ void k_copy_names(const uint8_t* __restrict__ text, const LineOut* __restrict__ lines,
                             const uint32_t* __restrict__ rec_line, uint64_t n_rec, const uint64_t* __restrict__ name_off,
                             uint8_t* __restrict__ names) {
  const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n_rec) return;
  const LineOut& o = lines[rec_line[r]];
  SubIter it(CellIter(text, o.name_b, o.name_e), o.name_first, o.name_first + o.name_len - 1);
  uint8_t c;
  uint64_t w = name_off[r];
  while (it.next(c)) names[w++] = c;
}

namespace {

// ---- newline positions: 16-byte chunks, one scan
struct NewlineF {
  const uint8_t* text;
  uint64_t len;
  uint64_t* nl;
  __device__ __forceinline__ uint64_t load(uint64_t c) const {
    uint64_t n = 0;
    const uint64_t b = c * 16, e = b + 16 < len ? b + 16 : len;
    for (uint64_t i = b; i < e; ++i) n += text[i] == '\n';
    return n;
  }
  __device__ __forceinline__ void store(uint64_t c, uint64_t excl, uint64_t v) const {
    if (!v) return;
    const uint64_t b = c * 16, e = b + 16 < len ? b + 16 : len;
    for (uint64_t i = b; i < e; ++i)
      if (text[i] == '\n') nl[excl++] = i;
  }
};

// ---- record compaction: columns in line order
struct RecordF {
  const LineOut* lines;
  uint32_t* rec_line;
  int64_t* start;
  int64_t* dur;
  int64_t* size;
  uint8_t* flags;
  uint32_t* stream;
  uint64_t* name_len;
  __device__ __forceinline__ uint64_t load(uint64_t k) const { return lines[k].status == kLineRecord; }
  __device__ __forceinline__ void store(uint64_t k, uint64_t r, uint64_t v) const {
    if (!v) return;
    const LineOut& o = lines[k];
    rec_line[r] = static_cast<uint32_t>(k);
    start[r] = o.start;
    dur[r] = o.dur;
    size[r] = o.size;
    flags[r] = o.flags;
    stream[r] = o.stream;
    name_len[r] = o.name_len;
  }
};
struct SkipF {  // skipped lines, in line order
  const LineOut* lines;
  uint32_t* skip_line;
  __device__ __forceinline__ uint32_t load(uint64_t k) const { return lines[k].status == kLineSkip; }
  __device__ __forceinline__ void store(uint64_t k, uint32_t q, uint32_t v) const {
    if (v) skip_line[q] = static_cast<uint32_t>(k);
  }
};
struct OffF {  // exclusive prefix of name lengths -> name_off
  const uint64_t* len;
  uint64_t* off;
  uint64_t n;
  __device__ __forceinline__ uint64_t load(uint64_t r) const { return len[r]; }
  __device__ __forceinline__ void store(uint64_t r, uint64_t excl, uint64_t v) const {
    off[r] = excl;
    if (r + 1 == n) off[n] = excl + v;
  }
};

// ---- device labels: a small open-addressing table of label hashes (first record = representative)
constexpr uint32_t kDevTable = 1u << 17;
__device__ __forceinline__ bool same_label(const uint8_t* text, const LineOut& x, const LineOut& y) {
  if (x.dev_len != y.dev_len) return false;
  if (x.dev_len == 0) return true;  // both "unknown"
  SubIter a(CellIter(text, x.dev_b, x.dev_e), x.dev_first, x.dev_first + x.dev_len - 1);
  SubIter b(CellIter(text, y.dev_b, y.dev_e), y.dev_first, y.dev_first + y.dev_len - 1);
  uint8_t c, d;
  while (a.next(c)) {
    if (!b.next(d) || c != d) return false;
  }
  return true;
}
__global__ void k_dev_insert(const uint8_t* __restrict__ text, const LineOut* __restrict__ lines,
                             const uint32_t* __restrict__ rec_line, uint64_t n_rec, uint64_t seed,
                             unsigned long long* table /* (hash|1) << 32 | rep record */, uint32_t* slot_of,
                             uint32_t* used, uint32_t* counters /* [0] used, [1] overflow, [2] collision */) {
  const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n_rec) return;
  const LineOut& o = lines[rec_line[r]];
  const uint64_t h = (o.dev_hash ^ seed) * 0x9E3779B97F4A7C15ull;
  const unsigned long long frag = ((h >> 32) | 1ull) << 32;
  uint32_t s = static_cast<uint32_t>(h) & (kDevTable - 1);
  for (uint32_t probe = 0;; ++probe) {
    if (probe >= kDevTable) {
      atomicOr(&counters[1], 1u);
      return;
    }
    // a plain read first: nearly every record finds its (few) labels already inserted, and a CAS
    // per record on one hot slot would serialize
    unsigned long long k = __ldcg(&table[s]);
    if (k == 0) k = atomicCAS(&table[s], 0ull, frag | r);
    if (k == 0) {
      used[atomicAdd(&counters[0], 1u)] = s;
      break;
    }
    if ((k & 0xFFFFFFFF00000000ull) == frag) {
      const uint32_t rep = static_cast<uint32_t>(k);
      if (!same_label(text, o, lines[rec_line[rep]])) atomicOr(&counters[2], 1u);
      break;
    }
    s = (s + 1) & (kDevTable - 1);
  }
  slot_of[r] = s;
}
// [begin, end) byte span of data lines (k relative to first_line)
__device__ __forceinline__ void line_span(const uint64_t* nl, uint64_t n_nl, uint64_t len, uint64_t ln, uint64_t& b,
                                          uint64_t& e) {
  b = ln == 0 ? 0 : nl[ln - 1] + 1;
  e = ln < n_nl ? nl[ln] : len;
}
__global__ void k_line_spans(const uint32_t* __restrict__ ks, uint32_t n, const uint64_t* __restrict__ nl, uint64_t n_nl,
                             uint64_t len, uint64_t first_line, uint64_t* __restrict__ span) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) line_span(nl, n_nl, len, first_line + ks[q], span[2 * q], span[2 * q + 1]);
}
__global__ void k_skip_info(const LineOut* __restrict__ lines, const uint32_t* __restrict__ ks, uint64_t n,
                            const uint64_t* __restrict__ nl, uint64_t n_nl, uint64_t len, uint64_t first_line,
                            uint64_t* __restrict__ span, uint8_t* __restrict__ why) {
  const uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  line_span(nl, n_nl, len, first_line + ks[q], span[2 * q], span[2 * q + 1]);
  why[q] = lines[ks[q]].reason;
}
__global__ void k_dev_rank(const uint32_t* __restrict__ slot_of, uint64_t n_rec, const uint16_t* __restrict__ rank_of_slot,
                           uint16_t* __restrict__ device) {
  const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < n_rec) device[r] = rank_of_slot[slot_of[r]];
}

// ---- host side: the reference's header / units / cell rules for the few lines read on the host
std::vector<std::string> host_split(const char* p, size_t n) {  // split_csv (ingest.hpp:104-131)
  std::vector<std::string> f;
  std::string cur;
  bool quoted = false;
  for (size_t i = 0; i < n; ++i) {
    const char c = p[i];
    if (quoted) {
      if (c == '"') {
        if (i + 1 < n && p[i + 1] == '"') {
          cur.push_back('"');
          ++i;
        } else {
          quoted = false;
        }
      } else {
        cur.push_back(c);
      }
    } else if (c == '"') {
      quoted = true;
    } else if (c == ',') {
      f.push_back(cur);
      cur.clear();
    } else {
      cur.push_back(c);
    }
  }
  f.push_back(cur);
  return f;
}
std::string host_trim(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && (s[a] == ' ' || s[a] == '\t')) ++a;
  while (b > a && (s[b - 1] == ' ' || s[b - 1] == '\t')) --b;
  return s.substr(a, b - a);
}
int64_t host_time_factor(const std::string& u) {
  if (u == "s") return 1000000000;
  if (u == "ms") return 1000000;
  if (u == "us") return 1000;
  if (u == "ns") return 1;
  return 0;
}
int64_t host_size_factor(const std::string& u) {
  if (u == "B") return 1;
  if (u == "KB") return 1024;
  if (u == "MB") return 1024 * 1024;
  if (u == "GB") return 1024LL * 1024 * 1024;
  return 0;
}
bool host_tp_unit(const std::string& u) { return u == "B/s" || u == "KB/s" || u == "MB/s" || u == "GB/s"; }
bool host_unit_token(const std::string& t) { return host_time_factor(t) || host_size_factor(t) || host_tp_unit(t); }

struct HostLines {  // line cursor over host text (next_line, ingest.hpp:180-190)
  const char* t;
  uint64_t n, pos = 0, idx = 0;  // idx: 0-based index of the next line
  bool next(const char*& p, size_t& len, uint64_t& line_idx) {
    if (pos >= n) return false;
    const char* nlp = static_cast<const char*>(std::memchr(t + pos, '\n', n - pos));
    const uint64_t e = nlp ? static_cast<uint64_t>(nlp - t) : n;
    p = t + pos;
    len = e - pos;
    if (len && p[len - 1] == '\r') --len;
    pos = nlp ? e + 1 : n;
    line_idx = idx++;
    return true;
  }
};
bool host_content(const char* p, size_t len) {  // not blank, not a "==" comment
  const std::string l(p, len);
  if (host_trim(l).empty()) return false;
  return !(len >= 2 && p[0] == '=' && p[1] == '=');
}

}  // namespace

void parse_csv(Ctx* c, const char* text, uint64_t len, const std::string& label, ParsedCsv& out) {
  // ---- header and units row on the host (ingest.hpp:196-252, 287-316)
  HostLines hl{text, len};
  const char* p = nullptr;
  size_t plen = 0;
  uint64_t li = 0;
  bool header = false;
  for (int q = 0; q < kIngestCols; ++q) out.col[q] = -1;
  static const char* kNames[kIngestCols] = {"Start", "Duration", "Size", "Throughput", "Device", "Stream", "Name"};
  while (hl.next(p, plen, li)) {
    if (!host_content(p, plen)) continue;
    const auto f = host_split(p, plen);
    for (size_t i = 0; i < f.size(); ++i) {
      const std::string nm = host_trim(f[i]);
      for (int q = 0; q < kIngestCols; ++q)
        if (nm == kNames[q]) out.col[q] = static_cast<int>(i);  // the last occurrence wins
    }
    for (int q : {kColStart, kColDuration, kColStream, kColName})
      if (out.col[q] < 0)
        fail(ITT_E_MISSING_COLUMN, std::string("ingest: required column '") + kNames[q] + "' missing from header of '" +
                                       label + "'");
    header = true;
    break;
  }
  if (!header) fail(ITT_E_MISSING_COLUMN, "ingest: no header row found in '" + label + "'");
  int64_t start_factor = 1000, duration_factor = 1000, size_factor = 1;
  uint64_t first_line = hl.idx;  // the line after the header
  while (hl.next(p, plen, li)) {
    if (!host_content(p, plen)) continue;
    const auto f = host_split(p, plen);
    bool any = false, all_units = true;
    for (const auto& x : f) {
      const std::string tok = host_trim(x);
      if (tok.empty()) continue;
      any = true;
      if (!host_unit_token(tok)) {
        all_units = false;
        break;
      }
    }
    if (any && all_units) {  // apply_units_row (ingest.hpp:224-252)
      auto unit_at = [&](int q) -> std::string {
        return out.col[q] < 0 || static_cast<size_t>(out.col[q]) >= f.size() ? std::string() : host_trim(f[out.col[q]]);
      };
      if (auto u = unit_at(kColStart); !u.empty()) {
        if (int64_t x = host_time_factor(u)) start_factor = x;
        else out.warnings.push_back("ingest: unit '" + u + "' is not a time unit; Start defaults to us");
      }
      if (auto u = unit_at(kColDuration); !u.empty()) {
        if (int64_t x = host_time_factor(u)) duration_factor = x;
        else out.warnings.push_back("ingest: unit '" + u + "' is not a time unit; Duration defaults to us");
      }
      if (auto u = unit_at(kColSize); !u.empty()) {
        if (int64_t x = host_size_factor(u)) size_factor = x;
        else out.warnings.push_back("ingest: unit '" + u + "' is not a size unit; Size defaults to B");
      }
      if (auto u = unit_at(kColThroughput); !u.empty()) {
        if (!host_tp_unit(u)) out.warnings.push_back("ingest: unit '" + u + "' is not a throughput unit; Throughput defaults to B/s");
      }
      first_line = li + 1;
    } else {
      first_line = li;  // the units check happens once; this line is data
    }
    break;
  }
  // ---- device: lines, per-line parse, compaction
  DBuf<uint8_t> dtext(c, len + 16);
  h2d_bulk(c, dtext.p, text, len);
  ScanScratch scan;
  const uint64_t chunks = (len + 15) / 16;
  const uint64_t nl_cap = len + 1;
  DBuf<uint64_t> nl(c, nl_cap);
  uint64_t n_nl = 0;
  if (chunks) {
    device_scan<uint64_t, SumOp<uint64_t>>(c, "ingest_newlines", len * 1.0, NewlineF{dtext.p, len, nl.p}, chunks, scan);
    n_nl = scan.total(c);
  }
  const uint64_t n_lines = n_nl + ((len > 0 && text[len - 1] != '\n') ? 1 : 0);
  const uint64_t n_data = n_lines > first_line ? n_lines - first_line : 0;
  out.n = 0;
  out.rows_total = 0;
  DBuf<LineOut> lines(c, std::max<uint64_t>(1, n_data));
  if (n_data) {
    IngestArgs a{dtext.p, len, nl.p, n_nl, n_lines, first_line, {}, start_factor, duration_factor, size_factor, lines.p};
    for (int q = 0; q < kIngestCols; ++q) a.col[q] = out.col[q];
    launch(c, "ingest_lines", static_cast<double>(len), k_parse_lines, dim3(grid_for(n_data, 128)), dim3(128), 0, a);
  }
  // records
  DBuf<uint32_t> rec_line(c, std::max<uint64_t>(1, n_data));
  DBuf<uint64_t> name_len(c, std::max<uint64_t>(1, n_data));
  out.alloc_columns(std::max<uint64_t>(1, n_data));
  uint64_t n_rec = 0;
  if (n_data) {
    device_scan<uint64_t, SumOp<uint64_t>>(c, "ingest_records", n_data * 64.0,
                                           RecordF{lines.p, rec_line.p, out.start, out.dur, out.size, out.flags, out.stream,
                                                   name_len.p},
                                           n_data, scan);
    n_rec = scan.total(c);
  }
  // skipped lines -> reasons on the host (the messages quote the offending cell, re-split there)
  uint64_t n_skip = 0;
  if (n_data) {
    DBuf<uint32_t> sk(c, n_data);
    device_scan<uint32_t, SumOp<uint32_t>>(c, "ingest_skips", n_data * 4.0, SkipF{lines.p, sk.p}, n_data, scan);
    n_skip = scan.total(c);
    if (n_skip) {
      DBuf<uint64_t> span(c, 2 * n_skip);
      DBuf<uint8_t> why(c, n_skip);
      launch(c, "ingest_skip_info", n_skip * 16.0, k_skip_info, dim3(grid_for(n_skip, 256)), dim3(256), 0, lines.p, sk.p,
             n_skip, nl.p, n_nl, len, first_line, span.p, why.p);
      std::vector<uint64_t> hs(2 * n_skip);
      std::vector<uint8_t> hw(n_skip);
      std::vector<uint32_t> hk(n_skip);
      readback(c, hs.data(), span.p, 2 * n_skip);
      readback(c, hw.data(), why.p, n_skip);
      readback(c, hk.data(), sk.p, n_skip);
      for (uint64_t q = 0; q < n_skip; ++q) {
        uint64_t e = hs[2 * q + 1];
        const uint64_t b = hs[2 * q];
        if (e > b && text[e - 1] == '\r') --e;
        const auto f = host_split(text + b, e - b);
        auto cell = [&](int col) -> std::string {
          return out.col[col] < 0 || static_cast<size_t>(out.col[col]) >= f.size() ? std::string() : host_trim(f[out.col[col]]);
        };
        std::string reason;
        switch (hw[q]) {
          case kSkipName: reason = "empty Name"; break;
          case kSkipStart: reason = "unparseable Start '" + cell(kColStart) + "'"; break;
          case kSkipDuration: reason = "unparseable Duration '" + cell(kColDuration) + "'"; break;
          case kSkipStream: reason = "unparseable Stream '" + cell(kColStream) + "'"; break;
          case kSkipSize: reason = "unparseable Size '" + cell(kColSize) + "'"; break;
          default: reason = "unparseable Throughput '" + cell(kColThroughput) + "'"; break;
        }
        out.skip_line.push_back(first_line + hk[q] + 1);  // 1-based line number (TraceRecord::row)
        out.skip_reason.push_back(reason);
      }
    }
  }
  out.rows_total = n_rec + n_skip;
  out.rows_parsed = n_rec;
  out.rows_skipped = n_skip;
  if (n_skip * 10 > out.rows_total)
    fail(ITT_E_TOO_MANY_BAD_ROWS, "ingest: " + std::to_string(n_skip) + " of " + std::to_string(out.rows_total) +
                                      " data rows unparseable in '" + label + "'; this looks like a format mismatch");
  out.n = n_rec;
  // names
  if (n_rec) {
    device_scan<uint64_t, SumOp<uint64_t>>(c, "ingest_name_off", n_rec * 16.0, OffF{name_len.p, out.name_off, n_rec}, n_rec,
                                           scan);
    uint64_t nb = 0;
    readback(c, &nb, out.name_off + n_rec, 1);
    out.alloc_names(nb);
    launch(c, "ingest_names", static_cast<double>(nb) * 2.0, k_copy_names, dim3(grid_for(n_rec, 128)), dim3(128), 0,
           dtext.p, lines.p, rec_line.p, n_rec, out.name_off, out.name_bytes);
  } else {
    out.alloc_names(0);
    ITT_CUDA(cudaMemsetAsync(out.name_off, 0, 8, c->stream));
  }
  // device labels -> ranks in byte-lexicographic order (ties of filter_majority_device)
  if (n_rec) {
    DBuf<unsigned long long> table(c, kDevTable);
    DBuf<uint32_t> slot_of(c, n_rec), used(c, kDevTable), counters(c, 4);
    uint64_t seed = 0;
    uint32_t cnt[4];
    for (int attempt = 0;; ++attempt) {
      table.zero();
      counters.zero();
      launch(c, "ingest_devices", n_rec * 12.0, k_dev_insert, dim3(grid_for(n_rec, 256)), dim3(256), 0, dtext.p, lines.p,
             rec_line.p, n_rec, seed, table.p, slot_of.p, used.p, counters.p);
      readback(c, cnt, counters.p, 4);
      if (cnt[1] || cnt[0] > 65536) fail(ITT_E_INVALID_ARGUMENT, "ingest: more than 65536 distinct device labels");
      if (!cnt[2]) break;
      if (attempt >= 3) fail(ITT_E_INVALID_ARGUMENT, "ingest: unresolvable device label hash collision");
      seed = seed * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
    }
    const uint32_t nd = cnt[0];
    std::vector<uint32_t> slots(nd);
    readback(c, slots.data(), used.p, nd);
    std::vector<unsigned long long> tab(kDevTable);
    readback(c, tab.data(), table.p, kDevTable);
    std::vector<uint32_t> rl(n_rec);
    readback(c, rl.data(), rec_line.p, n_rec);
    // label text of each representative, re-split from the host copy of its line
    std::vector<uint32_t> rep_k(nd);
    for (uint32_t q = 0; q < nd; ++q) rep_k[q] = rl[static_cast<uint32_t>(tab[slots[q]])];
    DBuf<uint32_t> dk(c, nd);
    h2d(c, dk.p, rep_k.data(), nd);
    DBuf<uint64_t> span(c, 2 * static_cast<uint64_t>(nd));
    launch(c, "ingest_rep_spans", nd * 16.0, k_line_spans, dim3(grid_for(nd, 256)), dim3(256), 0, dk.p, nd, nl.p, n_nl, len,
           first_line, span.p);
    std::vector<uint64_t> hs(2 * static_cast<uint64_t>(nd));
    readback(c, hs.data(), span.p, hs.size());
    std::vector<std::pair<std::string, uint32_t>> labels;  // (label, slot)
    for (uint32_t q = 0; q < nd; ++q) {
      uint64_t e = hs[2 * q + 1];
      const uint64_t b = hs[2 * q];
      if (e > b && text[e - 1] == '\r') --e;
      std::string lab = "unknown";
      if (out.col[kColDevice] >= 0) {
        const auto f = host_split(text + b, e - b);
        if (static_cast<size_t>(out.col[kColDevice]) < f.size()) {
          const std::string x = host_trim(f[out.col[kColDevice]]);
          if (!x.empty()) lab = x;
        }
      }
      labels.emplace_back(lab, slots[q]);
    }
    std::sort(labels.begin(), labels.end());
    std::vector<uint16_t> rank(kDevTable, 0);
    out.device_labels.clear();
    for (size_t q = 0; q < labels.size(); ++q) {
      rank[labels[q].second] = static_cast<uint16_t>(q);
      out.device_labels.push_back(labels[q].first);
    }
    DBuf<uint16_t> drank(c, kDevTable);
    h2d(c, drank.p, rank.data(), kDevTable);
    launch(c, "ingest_device_rank", n_rec * 6.0, k_dev_rank, dim3(grid_for(n_rec, 256)), dim3(256), 0, slot_of.p, n_rec,
           drank.p, out.device);
    out.line.resize(n_rec);
    for (uint64_t r = 0; r < n_rec; ++r) out.line[r] = first_line + rl[r] + 1;
  }
  c->sync();
}

}  // namespace itt
