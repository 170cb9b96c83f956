/*
 * itt_synth.h — deterministic TensorFlow-like trace generator (host only, libitt_synth.so).
 *
 * Test/bench infrastructure, not part of the hot path.  The reference's own
 * generator (synth.hpp:187-372) draws distinct names inside the pattern
 * (synth.hpp:157-161), so it cannot produce the BASELINE shapes (200 ops over 150
 * names); this one follows SURVEY §8(d): same stream shape (main 13, HtoD 14,
 * DtoH 15, assist 7 with memset + HtoD at t~0, synth.hpp:197-234), same
 * mt19937_64 + modulo reductions (synth.hpp:86-110), TF-like names of 40-120 bytes,
 * a fixed random body over V names with repeats, optional memcpy noise and a
 * local row shuffle so that source order != start order.
 */
#ifndef ITT_SYNTH_H
#define ITT_SYNTH_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct itt_synth_cfg {
  uint64_t seed;
  int64_t iterations;     /* I */
  int64_t body_len;       /* ops per iteration */
  int64_t vocab;          /* distinct body names V */
  int64_t init_ops;       /* distinct init-prefix names (16) */
  double noise_frac;      /* per main op: probability of an extra memcpy record on stream 14/15 */
  int64_t shuffle_window; /* rows shuffled inside consecutive windows of this size (<=1: none) */
  double minority_frac;   /* fraction of extra records on a second device label (0: none) */
  int64_t name_min, name_max;          /* name length range in bytes (40, 120) */
  int64_t kdur_lo, kdur_hi;            /* kernel duration [lo, hi) ns (2000, 4000) */
  int64_t intra_lo, intra_hi;          /* intra-iteration gap [lo, hi) (500, 1500) */
  int64_t inter_lo, inter_hi;          /* inter-iteration gap [lo, hi) (4000, 12000) */
  int64_t htod_lo, htod_hi;            /* HtoD bytes per gap [lo, hi] (1024, 9216) */
  int64_t body_inserts;   /* >0: per iteration, with prob insert_prob, insert 1..body_inserts foreign kernels inside the body */
  double insert_prob;
  double extra_stream_frac; /* fraction of main kernels duplicated onto kernel stream 21 */
} itt_synth_cfg;

typedef struct itt_synth_trace {
  uint64_t n;
  int64_t* start_ns;
  int64_t* duration_ns;
  int64_t* size_bytes;
  uint8_t* flags;
  uint32_t* stream;
  uint16_t* device;
  uint64_t* name_off;   /* [n+1] */
  uint8_t* name_bytes;
  uint64_t name_bytes_len;
  uint64_t n_main;      /* main-stream records (tokens) */
  uint64_t n_htod;
} itt_synth_trace;

void itt_synth_default(itt_synth_cfg* cfg);
/* returns 0 on success; free with itt_synth_free */
int itt_synth_generate(const itt_synth_cfg* cfg, itt_synth_trace* out);
void itt_synth_free(itt_synth_trace* t);
/* the trace as profiler CSV text in the reference's format (header + "ns,ns,B,B/s,,," units row,
 * rows in source order, names quoted); *text is malloc'd, release with free() */
int itt_synth_to_csv(const itt_synth_trace* t, char** text, uint64_t* len);

#ifdef __cplusplus
}
#endif
#endif
