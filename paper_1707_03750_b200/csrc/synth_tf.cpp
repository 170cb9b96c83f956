// Deterministic TF-like trace generator (see include/itt_synth.h).  Host-only test and
// bench infrastructure; the GPU path never calls it.
#include "itt_synth.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

namespace {

// mt19937_64 with explicit modulo reductions so identical seeds give identical
// streams everywhere (the reference's SynthRng idea, synth.hpp:86-110).
struct Rng {
  std::mt19937_64 g;
  explicit Rng(uint64_t s) : g(s) {}
  int64_t uniform(int64_t lo, int64_t hi) {  // inclusive
    if (hi <= lo) return lo;
    return lo + static_cast<int64_t>(g() % static_cast<uint64_t>(hi - lo + 1));
  }
  int64_t range(int64_t lo, int64_t hi) { return uniform(lo, hi - 1); }  // [lo, hi)
  bool coin(double p) {
    if (p <= 0.0) return false;
    if (p >= 1.0) return true;
    return static_cast<double>(g() >> 11) * 0x1.0p-53 < p;
  }
};

// Kernel names look like mangled TF/Eigen/cuDNN symbols.  The random alphabet has no
// 'e'/'E', so neither "memcpy" nor "memset" can appear and every name classifies as a
// kernel (trace.hpp:103-113).
const char* kPrefixes[] = {
    "void tensorflow::functor::ColumnReduceKernel<",
    "volta_sgemm_128x64_nn_",
    "void cudnn::winograd_nonfused::winogradForwardData4x4<",
    "void Eigen::internal::EigenMetaKernel<Eigen::TensorAssignOp<",
    "void tensorflow::BiasNHWCKernel<float>_",
    "ampere_fp16_s1688gemm_fp16_256x128_ldg8_f2f_",
    "void cub::DeviceReduceSingleTileKernel<",
    "void tensorflow::functor::SwapDimension1And2InTensor3UsingTiles<",
    "sm80_xmma_fprop_implicit_gemm_indexed_f16f16_",
    "void splitKreduce_kernel<32, 16, int, float>_",
};
const char kAlpha[] = "abcdfghijklnopqrstuvwxyzABCDFGHIJKLNOPQRSTUVWXYZ0123456789_:<>,";

std::string make_name(Rng& rng, int64_t id, int64_t lmin, int64_t lmax) {
  const size_t np = sizeof(kPrefixes) / sizeof(kPrefixes[0]);
  std::string s = kPrefixes[rng.range(0, static_cast<int64_t>(np))];
  char tag[32];
  std::snprintf(tag, sizeof(tag), "#%06lld", static_cast<long long>(id));
  const int64_t target = rng.uniform(lmin, lmax);
  const int64_t fill = target - static_cast<int64_t>(s.size()) - static_cast<int64_t>(std::strlen(tag));
  for (int64_t i = 0; i < fill; ++i) s.push_back(kAlpha[rng.range(0, static_cast<int64_t>(sizeof(kAlpha) - 1))]);
  s += tag;  // makes names unique
  if (static_cast<int64_t>(s.size()) > lmax && lmax > static_cast<int64_t>(std::strlen(tag))) {
    s = s.substr(s.size() - static_cast<size_t>(lmax));
  }
  return s;
}

struct Rec {  // 48 bytes: a 1B-event trace keeps its records in ~48 GB of host RAM
  int64_t start, dur, size;
  uint64_t seq;
  uint32_t stream;
  int32_t name;  // index into names table
  uint16_t device;
  uint8_t flags;
};

}  // namespace

extern "C" void itt_synth_default(itt_synth_cfg* c) {
  std::memset(c, 0, sizeof(*c));
  c->seed = 1;
  c->iterations = 100;
  c->body_len = 200;
  c->vocab = 150;
  c->init_ops = 16;
  c->noise_frac = 0.0;
  c->shuffle_window = 0;
  c->minority_frac = 0.0;
  c->name_min = 40;
  c->name_max = 120;
  c->kdur_lo = 2000;
  c->kdur_hi = 4000;
  c->intra_lo = 500;
  c->intra_hi = 1500;
  c->inter_lo = 4000;
  c->inter_hi = 12000;
  c->htod_lo = 1024;
  c->htod_hi = 9216;
  c->body_inserts = 0;
  c->insert_prob = 0.0;
  c->extra_stream_frac = 0.0;
}

extern "C" int itt_synth_generate(const itt_synth_cfg* cfg, itt_synth_trace* out) {
  if (!cfg || !out || cfg->iterations < 1 || cfg->body_len < 1 || cfg->vocab < 1 || cfg->init_ops < 0) return 1;
  std::memset(out, 0, sizeof(*out));
  Rng rng(cfg->seed);

  // name table: [0, V) body names, [V, V+init) init names, then fixed copy-engine names.
  std::vector<std::string> names;
  const int64_t V = cfg->vocab;
  names.reserve(static_cast<size_t>(V + cfg->init_ops + cfg->body_inserts + 8));
  for (int64_t v = 0; v < V + cfg->init_ops; ++v) names.push_back(make_name(rng, v, cfg->name_min, cfg->name_max));
  const int64_t n_foreign = cfg->body_inserts > 0 ? 8 : 0;
  const int32_t foreign0 = static_cast<int32_t>(names.size());
  for (int64_t v = 0; v < n_foreign; ++v) names.push_back(make_name(rng, V + cfg->init_ops + v, cfg->name_min, cfg->name_max));
  const int32_t kMemset = static_cast<int32_t>(names.size());
  names.push_back("[CUDA memset]");
  const int32_t kHtoD = static_cast<int32_t>(names.size());
  names.push_back("[CUDA memcpy HtoD]");
  const int32_t kDtoH = static_cast<int32_t>(names.size());
  names.push_back("[CUDA memcpy DtoH]");

  // body: every name at least once when L >= V, then shuffled
  std::vector<int32_t> body(static_cast<size_t>(cfg->body_len));
  {
    std::vector<int32_t> perm(static_cast<size_t>(V));
    for (int64_t v = 0; v < V; ++v) perm[static_cast<size_t>(v)] = static_cast<int32_t>(v);
    for (int64_t i = V - 1; i > 0; --i) std::swap(perm[static_cast<size_t>(i)], perm[static_cast<size_t>(rng.uniform(0, i))]);
    for (int64_t j = 0; j < cfg->body_len; ++j) {
      body[static_cast<size_t>(j)] = j < V ? perm[static_cast<size_t>(j)] : static_cast<int32_t>(rng.range(0, V));
    }
    for (int64_t i = cfg->body_len - 1; i > 0; --i) std::swap(body[static_cast<size_t>(i)], body[static_cast<size_t>(rng.uniform(0, i))]);
  }

  const uint32_t kMain = 13, kHtoDStream = 14, kDtoHStream = 15, kAssist = 7;
  const int64_t bw = 10;  // bytes per ns (10 GB/s): duration = ceil(bytes / 10)
  auto copy_dur = [&](int64_t bytes) { return (bytes + bw - 1) / bw; };

  std::vector<Rec> recs;
  const double est = static_cast<double>(cfg->iterations) * static_cast<double>(cfg->body_len) * (1.0 + cfg->noise_frac + cfg->minority_frac) +
                     3.0 * static_cast<double>(cfg->iterations) + static_cast<double>(cfg->init_ops) + 16.0;
  recs.reserve(static_cast<size_t>(est * 1.02));
  uint64_t seq = 0;
  auto push = [&](int64_t start, int64_t dur, int64_t size, uint8_t flags, uint32_t stream, int32_t name) {
    Rec r;
    r.start = start, r.dur = dur, r.size = size, r.seq = seq++;
    r.stream = stream, r.name = name, r.device = 0, r.flags = flags;
    recs.push_back(r);
  };
  const uint8_t SZ = 0x1, TP = 0x2;

  // assist stream: memset + HtoD at time ~0 (synth.hpp:230-234)
  push(0, 1000, 1024, SZ, kAssist, kMemset);
  push(1200, copy_dur(1024), 1024, SZ | TP, kAssist, kHtoD);
  int64_t cursor = 1200 + copy_dur(1024) + rng.range(cfg->intra_lo, cfg->intra_hi);
  int64_t prev_end = cursor;
  auto emit_kernel = [&](int32_t name) {
    const int64_t dur = rng.range(cfg->kdur_lo, cfg->kdur_hi);
    push(cursor, dur, 0, 0, kMain, name);
    if (cfg->noise_frac > 0.0 && rng.coin(cfg->noise_frac)) {
      const bool htod = rng.coin(0.5);
      const int64_t bytes = rng.uniform(256, 65536);
      push(cursor + rng.range(0, dur), copy_dur(bytes), bytes, SZ | TP, htod ? kHtoDStream : kDtoHStream, htod ? kHtoD : kDtoH);
    }
    prev_end = cursor + dur;
    cursor = prev_end + rng.range(cfg->intra_lo, cfg->intra_hi);
  };
  for (int64_t j = 0; j < cfg->init_ops; ++j) emit_kernel(static_cast<int32_t>(V + j));
  for (int64_t k = 1; k <= cfg->iterations; ++k) {
    const int64_t gap = rng.range(cfg->inter_lo, cfg->inter_hi);
    const int64_t block_start = prev_end + gap;
    if (k >= 2) {
      const int64_t bytes = rng.uniform(cfg->htod_lo, cfg->htod_hi);
      const int64_t d = copy_dur(bytes);
      push(prev_end + std::max<int64_t>(1, (gap - d) / 2), d, bytes, SZ | TP, kHtoDStream, kHtoD);
    }
    cursor = block_start;
    int64_t n_ins = 0, ins_at = -1;
    if (cfg->body_inserts > 0 && rng.coin(cfg->insert_prob)) {
      n_ins = rng.uniform(1, cfg->body_inserts);
      ins_at = rng.range(0, std::max<int64_t>(1, cfg->body_len - 1));
    }
    for (int64_t j = 0; j < cfg->body_len; ++j) {
      emit_kernel(body[static_cast<size_t>(j)]);
      if (j == ins_at)
        for (int64_t x = 0; x < n_ins; ++x) emit_kernel(foreign0 + static_cast<int32_t>(rng.range(0, n_foreign)));
    }
    push(prev_end + 200, copy_dur(512), 512, SZ | TP, kDtoHStream, kDtoH);  // result drain
  }
  // a second kernel-bearing stream (exercise select_main_stream's MultipleMainStreams warning)
  if (cfg->extra_stream_frac > 0.0) {
    const size_t base = recs.size();
    for (size_t i = 0; i < base; ++i) {
      if (recs[i].stream != kMain || !rng.coin(cfg->extra_stream_frac)) continue;
      Rec r = recs[i];
      r.stream = 21;
      r.start += 7;
      r.seq = seq++;
      recs.push_back(r);
    }
  }
  // minority device records (exercise filter_majority_device): copies of random main records
  if (cfg->minority_frac > 0.0) {
    const size_t base = recs.size();
    for (size_t i = 0; i < base; ++i) {
      if (!rng.coin(cfg->minority_frac)) continue;
      Rec r = recs[i];
      r.device = 1;
      r.seq = seq++;
      recs.push_back(r);
    }
  }
  // (start, seq) is unique, so any sort gives the stable order.  Without appended copies the
  // records are emitted nearly sorted (an HtoD copy may precede the previous drain), and an
  // in-place insertion sort is O(n) with no temporary buffer.
  auto before = [](const Rec& a, const Rec& b) { return a.start != b.start ? a.start < b.start : a.seq < b.seq; };
  if (cfg->extra_stream_frac > 0.0 || cfg->minority_frac > 0.0) {
    std::sort(recs.begin(), recs.end(), before);
  } else {
    for (size_t i = 1; i < recs.size(); ++i) {
      if (!before(recs[i], recs[i - 1])) continue;
      Rec x = recs[i];
      size_t j = i;
      while (j > 0 && before(x, recs[j - 1])) {
        recs[j] = recs[j - 1];
        --j;
      }
      recs[j] = x;
    }
  }
  if (cfg->shuffle_window > 1) {
    const size_t w = static_cast<size_t>(cfg->shuffle_window);
    for (size_t b = 0; b < recs.size(); b += w) {
      const size_t e = std::min(recs.size(), b + w);
      for (size_t i = e - 1; i > b; --i) std::swap(recs[i], recs[b + static_cast<size_t>(rng.uniform(0, static_cast<int64_t>(i - b)))]);
    }
  }

  // Two phases keep the peak near max(records + numeric columns, numeric columns + names):
  // the record vector is released before the name bytes are materialised.
  const uint64_t n = recs.size();
  uint64_t nb = 0;
  for (const auto& r : recs) nb += names[static_cast<size_t>(r.name)].size();
  out->n = n;
  out->start_ns = static_cast<int64_t*>(std::malloc(n * 8));
  out->duration_ns = static_cast<int64_t*>(std::malloc(n * 8));
  out->size_bytes = static_cast<int64_t*>(std::malloc(n * 8));
  out->flags = static_cast<uint8_t*>(std::malloc(n ? n : 1));
  out->stream = static_cast<uint32_t*>(std::malloc(n * 4));
  out->device = static_cast<uint16_t*>(std::malloc(n * 2));
  out->name_off = static_cast<uint64_t*>(std::malloc((n + 1) * 8));
  int32_t* name_id = static_cast<int32_t*>(std::malloc(n * 4 + 4));
  if (!out->start_ns || !out->duration_ns || !out->size_bytes || !out->flags || !out->stream || !out->device ||
      !out->name_off || !name_id) {
    std::free(name_id);
    itt_synth_free(out);
    return 2;
  }
  uint64_t off = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const Rec& r = recs[i];
    out->start_ns[i] = r.start;
    out->duration_ns[i] = r.dur;
    out->size_bytes[i] = r.size;
    out->flags[i] = r.flags;
    out->stream[i] = r.stream;
    out->device[i] = r.device;
    out->name_off[i] = off;
    name_id[i] = r.name;
    off += names[static_cast<size_t>(r.name)].size();
    if (r.stream == kMain && r.device == 0) ++out->n_main;
    if (r.name == kHtoD && r.device == 0) ++out->n_htod;
  }
  out->name_off[n] = off;
  std::vector<Rec>().swap(recs);
  // 16 bytes of slack: the device reads names in 16-byte chunks (also in place, ITT_MEM_HOST_MAPPED_NAMES)
  out->name_bytes = static_cast<uint8_t*>(std::calloc(nb + 16, 1));
  out->name_bytes_len = nb;
  if (!out->name_bytes) {
    std::free(name_id);
    itt_synth_free(out);
    return 2;
  }
  for (uint64_t i = 0; i < n; ++i) {
    const std::string& s = names[static_cast<size_t>(name_id[i])];
    std::memcpy(out->name_bytes + out->name_off[i], s.data(), s.size());
  }
  std::free(name_id);
  return 0;
}

extern "C" void itt_synth_free(itt_synth_trace* t) {
  if (!t) return;
  std::free(t->start_ns);
  std::free(t->duration_ns);
  std::free(t->size_bytes);
  std::free(t->flags);
  std::free(t->stream);
  std::free(t->device);
  std::free(t->name_off);
  std::free(t->name_bytes);
  std::memset(t, 0, sizeof(*t));
}

extern "C" int itt_synth_to_csv(const itt_synth_trace* t, char** text, uint64_t* len) {
  if (!t || !text || !len) return 1;
  std::string out;
  out.reserve(static_cast<size_t>(t->n) * 48 + t->name_bytes_len + 128);
  out += "Start,Duration,Size,Throughput,Device,Stream,Name\nns,ns,B,B/s,,,\n";
  char buf[128];
  for (uint64_t i = 0; i < t->n; ++i) {
    int k = std::snprintf(buf, sizeof(buf), "%lld,%lld,", static_cast<long long>(t->start_ns[i]),
                          static_cast<long long>(t->duration_ns[i]));
    out.append(buf, static_cast<size_t>(k));
    if (t->flags[i] & 0x1) out += std::to_string(t->size_bytes[i]);
    out += ',';
    if (t->flags[i] & 0x2) out += "1e9";
    k = std::snprintf(buf, sizeof(buf), ",gpu%u,%u,\"", static_cast<unsigned>(t->device[i]), t->stream[i]);
    out.append(buf, static_cast<size_t>(k));
    for (uint64_t b = t->name_off[i]; b < t->name_off[i + 1]; ++b) {
      const char c = static_cast<char>(t->name_bytes[b]);
      if (c == '"') out += '"';
      out += c;
    }
    out += "\"\n";
  }
  *text = static_cast<char*>(std::malloc(out.size() + 1));
  if (!*text) return 2;
  std::memcpy(*text, out.data(), out.size());
  (*text)[out.size()] = 0;
  *len = out.size();
  return 0;
}
