// dist_driver.cu — the distributed suffix array of one trace over G ranks, driven natively.
//
// the reference builds one suffix tree on one core
// (suffix_tree.hpp:21-190 via mine.hpp:38-40); here the text positions are block-partitioned
// across G GPUs and every prefix-doubling round is a global sample sort of (rank_i, rank_{i+h})
// keys with an all-to-all, followed by dense ids and a route-back of (id, i) to the owner of i.
// The per-element steps are the dist.cu kernels (itt_dsa_*); this file is the host side that
// paper_1707_03750_b200/dist_sa.py restates in Python (the numpy / gloo tests cover it on CPU):
//   * Transport — the exchanges: NcclTransport (ncclSend/ncclRecv grouped all-to-all,
//     ncclAllGather, ncclBroadcast on the context's stream; libnccl is loaded on first use) and
//     LocalTransport (virtual ranks = threads of one process on one device, device-to-device
//     copies after a barrier; no kernel ever waits on another rank's kernel);
//   * dsa_build — one rank's share of the SA + capped LCP (same steps as suffix_array_dist);
//   * Provider — itt_analyze's sa_provider on the root: the tokens are broadcast, every rank
//     builds its slice, the slices are gathered back into the analyze's buffers; the other ranks
//     sit in itt_dsa_serve until the root calls itt_dsa_stop.
#include <dlfcn.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <vector>

#include "pipeline.cuh"

namespace itt {
namespace dsa {

// ------------------------------------------------------------------ NCCL, loaded on first use
// (a process that never builds a distributed SA does not need libnccl; torch's bundled NCCL is
// the one found when torch already loaded it, the system one otherwise)
namespace nccl {
typedef struct ncclComm* Comm;
struct UniqueId {
  char internal[128];
};
enum Result { kSuccess = 0 };
enum DataType { kUint8 = 1, kUint64 = 5 };
enum RedOp { kMax = 2 };
struct Api {
  int (*GetUniqueId)(UniqueId*);
  int (*CommInitRank)(Comm*, int, UniqueId, int);
  int (*CommDestroy)(Comm);
  int (*Send)(const void*, size_t, int, int, Comm, cudaStream_t);
  int (*Recv)(void*, size_t, int, int, Comm, cudaStream_t);
  int (*GroupStart)();
  int (*GroupEnd)();
  int (*AllGather)(const void*, void*, size_t, int, Comm, cudaStream_t);
  int (*Broadcast)(const void*, void*, size_t, int, int, Comm, cudaStream_t);
  const char* (*GetErrorString)(int);
};
const Api& api() {
  static Api a = [] {
    Api x{};
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return x;
    x.GetUniqueId = reinterpret_cast<int (*)(UniqueId*)>(dlsym(h, "ncclGetUniqueId"));
    x.CommInitRank = reinterpret_cast<int (*)(Comm*, int, UniqueId, int)>(dlsym(h, "ncclCommInitRank"));
    x.CommDestroy = reinterpret_cast<int (*)(Comm)>(dlsym(h, "ncclCommDestroy"));
    x.Send = reinterpret_cast<int (*)(const void*, size_t, int, int, Comm, cudaStream_t)>(dlsym(h, "ncclSend"));
    x.Recv = reinterpret_cast<int (*)(void*, size_t, int, int, Comm, cudaStream_t)>(dlsym(h, "ncclRecv"));
    x.GroupStart = reinterpret_cast<int (*)()>(dlsym(h, "ncclGroupStart"));
    x.GroupEnd = reinterpret_cast<int (*)()>(dlsym(h, "ncclGroupEnd"));
    x.AllGather = reinterpret_cast<int (*)(const void*, void*, size_t, int, Comm, cudaStream_t)>(dlsym(h, "ncclAllGather"));
    x.Broadcast =
        reinterpret_cast<int (*)(const void*, void*, size_t, int, int, Comm, cudaStream_t)>(dlsym(h, "ncclBroadcast"));
    x.GetErrorString = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
    return x;
  }();
  if (!a.CommInitRank) fail(ITT_E_NCCL, "dist: libnccl.so.2 not found");
  return a;
}
inline void check(int rc, const char* what) {
  if (rc != kSuccess) fail(ITT_E_NCCL, std::string("dist: ") + what + ": " + (api().GetErrorString ? api().GetErrorString(rc) : "NCCL error"));
}
}  // namespace nccl

// ------------------------------------------------------------------ transports
struct Transport {
  int P = 1, r = 0;
  virtual ~Transport() = default;
  // all-to-all of variable-size blocks: send holds scounts[q] elements for rank q, back to back;
  // recv gets rcounts[q] elements from rank q, back to back (counts known on every side)
  virtual void alltoallv(Ctx* c, const void* send, const uint64_t* scounts, void* recv, const uint64_t* rcounts,
                         size_t elem) = 0;
  // host values: k per rank -> all[P * k]
  virtual void allgather_host(Ctx* c, const uint64_t* mine, int k, uint64_t* all) = 0;
  // device bytes from root to everyone
  virtual void bcast_dev(Ctx* c, void* buf, size_t bytes, int root) = 0;
  // counts[q] I send to q -> recv[q] q sends to me
  void exchange_counts(Ctx* c, const uint64_t* scounts, uint64_t* rcounts) {
    std::vector<uint64_t> all(static_cast<size_t>(P) * P);
    allgather_host(c, scounts, P, all.data());
    for (int q = 0; q < P; ++q) rcounts[q] = all[static_cast<size_t>(q) * P + r];
  }
  void bcast_host(Ctx* c, uint64_t* vals, int k, int root) {
    std::vector<uint64_t> all(static_cast<size_t>(P) * k);
    allgather_host(c, vals, k, all.data());
    std::copy(all.begin() + static_cast<size_t>(root) * k, all.begin() + static_cast<size_t>(root + 1) * k, vals);
  }
};

struct NcclTransport : Transport {
  nccl::Comm comm = nullptr;
  NcclTransport(Ctx* c, int nranks, int rank, const uint8_t* id) {
    P = nranks;
    r = rank;
    nccl::UniqueId uid;
    std::memcpy(uid.internal, id, sizeof(uid.internal));
    ITT_CUDA(cudaSetDevice(c->device));
    nccl::check(nccl::api().CommInitRank(&comm, nranks, uid, rank), "ncclCommInitRank");
  }
  ~NcclTransport() override {
    if (comm) nccl::api().CommDestroy(comm);
  }
  void alltoallv(Ctx* c, const void* send, const uint64_t* scounts, void* recv, const uint64_t* rcounts,
                 size_t elem) override {
    const auto& a = nccl::api();
    const auto* s = static_cast<const uint8_t*>(send);
    auto* d = static_cast<uint8_t*>(recv);
    nccl::check(a.GroupStart(), "ncclGroupStart");
    uint64_t so = 0, ro = 0;
    for (int q = 0; q < P; ++q) {
      if (scounts[q]) nccl::check(a.Send(s + so * elem, scounts[q] * elem, nccl::kUint8, q, comm, c->stream), "ncclSend");
      if (rcounts[q]) nccl::check(a.Recv(d + ro * elem, rcounts[q] * elem, nccl::kUint8, q, comm, c->stream), "ncclRecv");
      so += scounts[q];
      ro += rcounts[q];
    }
    nccl::check(a.GroupEnd(), "ncclGroupEnd");
  }
  void allgather_host(Ctx* c, const uint64_t* mine, int k, uint64_t* all) override {
    DBuf<uint64_t> in(c, k), out(c, static_cast<size_t>(P) * k);
    h2d(c, in.p, mine, k);
    nccl::check(nccl::api().AllGather(in.p, out.p, static_cast<size_t>(k), nccl::kUint64, comm, c->stream), "ncclAllGather");
    readback(c, all, out.p, static_cast<size_t>(P) * k);
  }
  void bcast_dev(Ctx* c, void* buf, size_t bytes, int root) override {
    nccl::check(nccl::api().Broadcast(buf, buf, bytes, nccl::kUint8, root, comm, c->stream), "ncclBroadcast");
  }
};

// Virtual ranks: threads of one process sharing one device.  A generation barrier orders the
// posting of buffers and the copies out of them; every copy runs on the reader's stream after the
// writer synchronized its own, so no kernel waits on another rank.
struct Board {
  int P;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;
  std::vector<const void*> ptr;
  std::vector<std::vector<uint64_t>> vals;
  explicit Board(int n) : P(n), ptr(n), vals(n) {}
  void wait() {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    cv.wait(lk, [&] { return gen != g || aborted; });
    if (aborted) fail(ITT_E_NCCL, "dist: a virtual rank failed");
  }
  void abort() {
    std::lock_guard<std::mutex> lk(m);
    aborted = true;
    cv.notify_all();
  }
};

struct LocalTransport : Transport {
  std::shared_ptr<Board> b;
  LocalTransport(std::shared_ptr<Board> board, int rank) : b(std::move(board)) {
    P = b->P;
    r = rank;
  }
  void alltoallv(Ctx* c, const void* send, const uint64_t* scounts, void* recv, const uint64_t* rcounts,
                 size_t elem) override {
    ITT_CUDA(cudaStreamSynchronize(c->stream));  // my send buffer is complete
    b->ptr[r] = send;
    b->vals[r].assign(scounts, scounts + P);
    b->wait();
    uint64_t ro = 0;
    for (int q = 0; q < P; ++q) {
      uint64_t so = 0;  // offset of my block inside q's send buffer
      for (int t = 0; t < r; ++t) so += b->vals[q][t];
      if (b->vals[q][r] != rcounts[q]) fail(ITT_E_NCCL, "dist: all-to-all count mismatch");
      if (rcounts[q])
        ITT_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(recv) + ro * elem, static_cast<const uint8_t*>(b->ptr[q]) + so * elem,
                                 rcounts[q] * elem, cudaMemcpyDeviceToDevice, c->stream));
      ro += rcounts[q];
    }
    ITT_CUDA(cudaStreamSynchronize(c->stream));
    b->wait();  // everyone has copied out: the send buffers may be released
  }
  void allgather_host(Ctx*, const uint64_t* mine, int k, uint64_t* all) override {
    b->vals[r].assign(mine, mine + k);
    b->wait();
    for (int q = 0; q < P; ++q) std::copy(b->vals[q].begin(), b->vals[q].begin() + k, all + static_cast<size_t>(q) * k);
    b->wait();
  }
  void bcast_dev(Ctx* c, void* buf, size_t bytes, int root) override {
    ITT_CUDA(cudaStreamSynchronize(c->stream));
    b->ptr[r] = buf;
    b->wait();
    if (r != root && bytes) ITT_CUDA(cudaMemcpyAsync(buf, b->ptr[root], bytes, cudaMemcpyDeviceToDevice, c->stream));
    ITT_CUDA(cudaStreamSynchronize(c->stream));
    b->wait();
  }
};

// ------------------------------------------------------------------ the doubling over G ranks
constexpr uint32_t kSamplesPerRank = 256;

__global__ void k_low32(const uint64_t* __restrict__ p, uint64_t n, uint32_t* __restrict__ out) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = static_cast<uint32_t>(p[i]);
}

struct Slice {
  DBuf<uint32_t> sa, lcp;  // this rank's sorted positions [kbase, kbase + count)
  uint64_t kbase = 0, count = 0;
  uint64_t groups = 0;
  uint32_t h_final = 0, cap = 0;
  int rounds = 0;
};

namespace {

uint64_t last_of(Ctx* c, const uint64_t* a, uint64_t cnt) {
  if (!cnt) return 0;
  uint64_t v = 0;
  readback(c, &v, a + cnt - 1, 1);
  return v;
}

// (has_prev, value): the last element of the nearest non-empty rank before r; table[q] = (count, last)
std::pair<bool, uint64_t> prev_nonempty(const std::vector<uint64_t>& table, int r) {
  for (int q = r - 1; q >= 0; --q)
    if (table[2 * q] > 0) return {true, table[2 * q + 1]};
  return {false, 0};
}

// exchange a partitioned (a[, b]) pair of arrays by the per-destination counts
template <typename A>
void route(Ctx* c, Transport& T, const A* a, const uint32_t* b, const uint64_t* scounts, DBuf<A>& ra, DBuf<uint32_t>* rb,
           uint64_t& rcnt) {
  std::vector<uint64_t> rc(T.P);
  T.exchange_counts(c, scounts, rc.data());
  rcnt = std::accumulate(rc.begin(), rc.end(), uint64_t{0});
  ra.alloc(c, std::max<uint64_t>(1, rcnt));
  T.alltoallv(c, a, scounts, ra.p, rc.data(), sizeof(A));
  if (rb) {
    rb->alloc(c, std::max<uint64_t>(1, rcnt));
    T.alltoallv(c, b, scounts, rb->p, rc.data(), 4);
  }
}

// global sort by (a, position): the splitters are quantiles of pseudo-random samples of every
// rank (evenly spaced samples alias with a periodic trace's period), gathered to every rank
void sample_sort(Ctx* c, Transport& T, DBuf<uint64_t>& a, DBuf<uint32_t>& v, uint64_t& cnt, int key_bits) {
  const int P = T.P;
  if (P == 1) {
    sort(c, a.p, v.p, cnt, key_bits);
    return;
  }
  const uint32_t s = static_cast<uint32_t>(std::min<uint64_t>(kSamplesPerRank, cnt));
  DBuf<uint64_t> sa_(c, kSamplesPerRank);
  DBuf<uint32_t> sb_(c, kSamplesPerRank);
  sample(c, a.p, v.p, cnt, s, sa_.p, sb_.p);
  std::vector<uint64_t> mine(2 * kSamplesPerRank, ~0ull);  // (a, b) pairs; unused slots stay ~0 (dropped)
  if (s) {
    std::vector<uint64_t> ha(s);
    std::vector<uint32_t> hb(s);
    readback(c, ha.data(), sa_.p, s);
    readback(c, hb.data(), sb_.p, s);
    for (uint32_t i = 0; i < s; ++i) mine[2 * i] = ha[i], mine[2 * i + 1] = hb[i];
  }
  std::vector<uint64_t> all(static_cast<size_t>(P) * 2 * kSamplesPerRank);
  T.allgather_host(c, mine.data(), 2 * kSamplesPerRank, all.data());
  std::vector<std::pair<uint64_t, uint32_t>> smp;
  for (size_t i = 0; i < all.size(); i += 2)
    if (all[i + 1] != ~0ull) smp.emplace_back(all[i], static_cast<uint32_t>(all[i + 1]));
  if (smp.empty()) smp.emplace_back(0, 0);
  std::sort(smp.begin(), smp.end());
  std::vector<uint64_t> spa(P - 1);
  std::vector<uint32_t> spb(P - 1);
  for (int q = 1; q < P; ++q) {
    const size_t k = std::min(smp.size() - 1, static_cast<size_t>(q) * smp.size() / P);
    spa[q - 1] = smp[k].first;
    spb[q - 1] = smp[k].second;
  }
  DBuf<uint64_t> dspa(c, P - 1);
  DBuf<uint32_t> dspb(c, P - 1);
  h2d(c, dspa.p, spa.data(), P - 1);
  h2d(c, dspb.p, spb.data(), P - 1);
  DBuf<uint64_t> oa(c, std::max<uint64_t>(1, cnt));
  DBuf<uint32_t> ob(c, std::max<uint64_t>(1, cnt));
  std::vector<uint64_t> counts(P);
  partition(c, a.p, v.p, cnt, 0, dspa.p, dspb.p, static_cast<uint32_t>(P - 1), nullptr, static_cast<uint32_t>(P), oa.p, ob.p,
            counts.data());
  a.release();
  v.release();
  uint64_t rcnt = 0;
  route(c, T, oa.p, ob.p, counts.data(), a, &v, rcnt);
  cnt = rcnt;
  sort(c, a.p, v.p, cnt, key_bits);
}

// (id << 32 | i) or (lcp << 32 | k) to the owner of its low / high half under `bounds`
void to_owners(Ctx* c, Transport& T, const uint64_t* p, uint64_t cnt, const DBuf<uint64_t>& bounds, DBuf<uint64_t>& back,
               uint64_t& rcnt) {
  DBuf<uint64_t> oa(c, std::max<uint64_t>(1, cnt));
  std::vector<uint64_t> counts(T.P);
  partition(c, p, nullptr, cnt, 1, nullptr, nullptr, 0, bounds.p, static_cast<uint32_t>(T.P), oa.p, nullptr, counts.data());
  route<uint64_t>(c, T, oa.p, nullptr, counts.data(), back, nullptr, rcnt);
}

}  // namespace

// SPMD: every rank calls this with the replicated text (tokens + [term], int32 on its device,
// tokens in [0, term)).  cap = max L_max + 1 for mining; 0xFFFFFFFF = full suffix array.
void build(Ctx* c, Transport& T, const int32_t* text, uint64_t n, int32_t term, uint32_t cap, bool want_lcp, Slice& out) {
  const int P = T.P, r = T.r;
  const uint64_t np = n + 1;
  if (np >= 0x7FFFFFFFull) fail(ITT_E_INVALID_ARGUMENT, "dist: n + 1 must stay below 2^31 - 1");
  const char* fe = std::getenv("ITT_DSA_FORCE_DIST");  // =1: the sample-sort rounds even at one rank (tests)
  const bool force = fe && *fe == '1';
  if (P == 1 && !force) {  // nothing to distribute: the single-device capped doubling (sa.cu)
    SuffixState s;
    radix::Scratch rs;
    ScanScratch sc;
    build_suffix_array(c, text, n, term, s, want_lcp, rs, sc, cap, /*known_alphabet=*/true);
    out.kbase = 0;
    out.count = np;
    out.groups = 0;
    out.rounds = s.rounds;
    out.h_final = s.h_final;
    out.cap = s.cap;
    out.sa = std::move(s.sa);
    if (want_lcp) out.lcp = std::move(s.lcp);
    return;
  }
  std::vector<uint64_t> bl(P + 1);
  for (int q = 0; q <= P; ++q) bl[q] = static_cast<uint64_t>(q) * np / P;
  const uint64_t lo = bl[r], hi = bl[r + 1], cnt0 = hi - lo;
  DBuf<uint64_t> bounds(c, P + 1);
  h2d(c, bounds.p, bl.data(), P + 1);
  const int sym_bits = bits_for(static_cast<uint64_t>(term));
  const int k = std::max(1, 64 / sym_bits);
  uint64_t cnt = cnt0;
  DBuf<uint64_t> a(c, std::max<uint64_t>(1, cnt));
  DBuf<uint32_t> v(c, std::max<uint64_t>(1, cnt));
  keys(c, text, np, lo, cnt, sym_bits, k, nullptr, nullptr, 0, 0, a.p, v.p);
  int key_bits = std::min(64, sym_bits * k);
  uint32_t h = static_cast<uint32_t>(k);
  int rounds = 0;
  uint64_t G = 0;
  DBuf<uint64_t> packed;
  std::vector<uint64_t> table(2 * P);
  for (;;) {
    sample_sort(c, T, a, v, cnt, key_bits);
    const uint64_t mine[2] = {cnt, last_of(c, a.p, cnt)};
    T.allgather_host(c, mine, 2, table.data());
    const auto pv = prev_nonempty(table, r);
    packed.alloc(c, std::max<uint64_t>(1, cnt));
    const uint64_t ng = ids(c, a.p, v.p, cnt, pv.first, pv.second, 0, packed.p);
    std::vector<uint64_t> ngs(P);
    T.allgather_host(c, &ng, 1, ngs.data());
    G = std::accumulate(ngs.begin(), ngs.end(), uint64_t{0});
    const uint64_t offset = std::accumulate(ngs.begin(), ngs.begin() + r, uint64_t{0});
    if (offset) ids(c, a.p, v.p, cnt, pv.first, pv.second, static_cast<uint32_t>(offset), packed.p);
    a.release();
    v.release();
    if (G == np || h >= cap) break;
    // (id, i) back to the owner of i
    DBuf<uint64_t> back;
    uint64_t nback = 0;
    to_owners(c, T, packed.p, cnt, bounds, back, nback);
    packed.release();
    DBuf<uint32_t> rank(c, std::max<uint64_t>(1, cnt0));
    scatter_hi(c, back.p, nback, lo, rank.p);
    back.release();
    // halo: ranks of positions [lo + h, min(hi + h, np)) from their owners, one slice per source
    std::vector<uint64_t> sc(P, 0), rc(P, 0);
    uint64_t first = lo;
    bool have_first = false;
    for (int q = 0; q < P; ++q) {  // what I send to q: my positions inside [bl[q] + h, bl[q+1] + h)
      const uint64_t s0 = std::max(bl[q] + h, lo), e0 = std::min(std::min(bl[q + 1] + h, hi), np);
      if (e0 > s0) {
        sc[q] = e0 - s0;
        if (!have_first) first = s0, have_first = true;
      }
      const uint64_t t0 = std::max(lo + h, bl[q]), t1 = std::min(std::min(hi + h, bl[q + 1]), np);  // what q sends me
      rc[q] = t1 > t0 ? t1 - t0 : 0;
    }
    const uint64_t n2 = std::accumulate(rc.begin(), rc.end(), uint64_t{0});
    DBuf<uint32_t> rank2(c, std::max<uint64_t>(1, n2));
    T.alltoallv(c, rank.p + (first - lo), sc.data(), rank2.p, rc.data(), 4);
    const int b = bits_for(G);
    cnt = cnt0;
    a.alloc(c, std::max<uint64_t>(1, cnt));
    v.alloc(c, std::max<uint64_t>(1, cnt));
    keys(c, text, np, lo, cnt, sym_bits, k, rank.p, rank2.p, n2, b, a.p, v.p);
    key_bits = bits_for(G - 1) + b;
    ++rounds;
    if (static_cast<uint64_t>(h) * 2 > 0xFFFFFFFFull) break;
    h *= 2;
  }
  const uint64_t last = last_of(c, packed.p, cnt);
  const uint64_t mine[2] = {cnt, last};
  T.allgather_host(c, mine, 2, table.data());
  uint64_t kbase = 0;
  for (int q = 0; q < r; ++q) kbase += table[2 * q];
  out.kbase = kbase;
  out.count = cnt;
  out.groups = G;
  out.rounds = rounds;
  out.h_final = h;
  out.cap = G == np ? 0xFFFFFFFFu : cap;
  out.sa.alloc(c, std::max<uint64_t>(1, cnt));
  if (cnt) launch(c, "dsa_low32", cnt * 12.0, k_low32, dim3(grid_for(cnt, 256)), dim3(256), 0, packed.p, cnt, out.sa.p);
  if (!want_lcp) return;
  const auto pv = prev_nonempty(table, r);
  DBuf<uint64_t> ra(c, std::max<uint64_t>(1, cnt));
  DBuf<uint32_t> rb(c, std::max<uint64_t>(1, cnt));
  lcp_requests(c, packed.p, cnt, kbase, pv.first, pv.second, ra.p, rb.p);
  DBuf<uint64_t> oa(c, std::max<uint64_t>(1, cnt));
  DBuf<uint32_t> ob(c, std::max<uint64_t>(1, cnt));
  std::vector<uint64_t> counts(P);
  partition(c, ra.p, rb.p, cnt, 1, nullptr, nullptr, 0, bounds.p, static_cast<uint32_t>(P), oa.p, ob.p, counts.data());
  ra.release();
  rb.release();
  DBuf<uint64_t> qa;
  DBuf<uint32_t> qb;
  uint64_t nq = 0;
  route(c, T, oa.p, ob.p, counts.data(), qa, &qb, nq);
  oa.release();
  ob.release();
  DBuf<uint64_t> plcp(c, std::max<uint64_t>(1, cnt0));
  kasai(c, text, np, lo, cnt0, qa.p, qb.p, out.cap, plcp.p);
  qa.release();
  qb.release();
  std::vector<uint64_t> kb(P + 1, 0);
  for (int q = 0; q < P; ++q) kb[q + 1] = kb[q] + table[2 * q];
  DBuf<uint64_t> kbounds(c, P + 1);
  h2d(c, kbounds.p, kb.data(), P + 1);
  DBuf<uint64_t> back;
  uint64_t nback = 0;
  to_owners(c, T, plcp.p, cnt0, kbounds, back, nback);
  out.lcp.alloc(c, std::max<uint64_t>(1, cnt));
  scatter_hi(c, back.p, nback, kbase, out.lcp.p);
}

// ------------------------------------------------------------------ analyze over G ranks
struct Provider {
  itt_ctx* ctx;      // this rank's context for the distributed steps
  Transport* T;
  int root;
  Slice last;
};

// root and servers: one distributed SA over the broadcast text, slices gathered on the root
void provide_round(Provider& pv, uint64_t n, int32_t term, uint32_t cap, DBuf<int32_t>& text, uint32_t* sa, uint32_t* lcp) {
  Ctx* c = &pv.ctx->c;
  Transport& T = *pv.T;
  T.bcast_dev(c, text.p, (n + 1) * 4, pv.root);
  Slice s;
  build(c, T, text.p, n, term, cap, true, s);
  // gather: every rank sends its slice to the root only
  std::vector<uint64_t> counts(T.P);
  T.allgather_host(c, &s.count, 1, counts.data());
  std::vector<uint64_t> sc(T.P, 0), rc(T.P, 0);
  sc[pv.root] = s.count;
  if (T.r == pv.root) rc = counts;
  T.alltoallv(c, s.sa.p, sc.data(), sa, rc.data(), 4);
  T.alltoallv(c, s.lcp.p, sc.data(), lcp, rc.data(), 4);
  c->sync();
  pv.last = std::move(s);
}

}  // namespace dsa
}  // namespace itt

using namespace itt;

struct itt_comm {
  std::unique_ptr<dsa::Transport> t;
};
struct itt_dsa_provider {
  dsa::Provider p;
};

namespace {
template <typename F>
int dguarded(itt_ctx* ctx, F&& f) {
  if (!ctx) return ITT_E_INVALID_ARGUMENT;
  Ctx* c = &ctx->c;
  try {
    ITT_CUDA(cudaSetDevice(c->device));
    c->arena_top = 0;
    c->upload_top = 0;
    f(c);
    c->sync();
    c->last_error.clear();
    return ITT_OK;
  } catch (const Error& e) {
    c->last_error = e.what();
    cudaStreamSynchronize(c->stream);
    c->pending.clear();
    return e.status;
  } catch (const std::exception& e) {
    c->last_error = e.what();
    return ITT_E_CUDA;
  }
}
}  // namespace

extern "C" {

int itt_comm_nccl_unique_id(uint8_t* id) {
  if (!id) return ITT_E_INVALID_ARGUMENT;
  try {
    dsa::nccl::UniqueId u;
    dsa::nccl::check(dsa::nccl::api().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, sizeof(u.internal));
    return ITT_OK;
  } catch (const Error& e) {
    return e.status;
  }
}

int itt_comm_create_nccl(itt_ctx* ctx, int nranks, int rank, const uint8_t* id, itt_comm** out) {
  if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) return ITT_E_INVALID_ARGUMENT;
  *out = nullptr;
  return dguarded(ctx, [&](Ctx* c) {
    auto* m = new itt_comm;
    try {
      m->t = std::make_unique<dsa::NcclTransport>(c, nranks, rank, id);
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
  });
}

int itt_comm_create_local(int nranks, itt_comm** comms) {
  if (!comms || nranks < 1) return ITT_E_INVALID_ARGUMENT;
  auto board = std::make_shared<dsa::Board>(nranks);
  for (int q = 0; q < nranks; ++q) {
    comms[q] = new itt_comm;
    comms[q]->t = std::make_unique<dsa::LocalTransport>(board, q);
  }
  return ITT_OK;
}

int itt_comm_abort(itt_comm* comm) {  // virtual ranks: release the others after a failure
  if (!comm) return ITT_E_INVALID_ARGUMENT;
  if (auto* l = dynamic_cast<dsa::LocalTransport*>(comm->t.get())) l->b->abort();
  return ITT_OK;
}

int itt_comm_destroy(itt_comm* comm) {
  delete comm;
  return ITT_OK;
}

int itt_dsa_build(itt_ctx* ctx, itt_comm* comm, const int32_t* text, uint64_t n, int32_t term, uint32_t cap, int want_lcp,
                  uint32_t** sa, uint32_t** lcp, uint64_t* kbase, uint64_t* count, itt_dsa_info* info) {
  if (!comm || !text || !sa || !kbase || !count) return ITT_E_INVALID_ARGUMENT;
  *sa = nullptr;
  if (lcp) *lcp = nullptr;
  return dguarded(ctx, [&](Ctx* c) {
    dsa::Slice s;
    dsa::build(c, *comm->t, text, n, term, cap, want_lcp != 0, s);
    // hand the slices out as plain device allocations (itt_device_free)
    const uint64_t m = std::max<uint64_t>(1, s.count);
    uint32_t* o = nullptr;
    ITT_CUDA(cudaMalloc(&o, m * 4));
    ITT_CUDA(cudaMemcpyAsync(o, s.sa.p, m * 4, cudaMemcpyDeviceToDevice, c->stream));
    *sa = o;
    if (want_lcp && lcp) {
      uint32_t* l = nullptr;
      ITT_CUDA(cudaMalloc(&l, m * 4));
      ITT_CUDA(cudaMemcpyAsync(l, s.lcp.p, m * 4, cudaMemcpyDeviceToDevice, c->stream));
      *lcp = l;
    }
    *kbase = s.kbase;
    *count = s.count;
    if (info) *info = itt_dsa_info{s.rounds, 0, s.groups, s.h_final, s.cap};
  });
}

int itt_dsa_provider_create(itt_ctx* ctx, itt_comm* comm, int root, itt_dsa_provider** out) {
  if (!ctx || !comm || !out || root < 0 || root >= comm->t->P) return ITT_E_INVALID_ARGUMENT;
  *out = new itt_dsa_provider{dsa::Provider{ctx, comm->t.get(), root, {}}};
  return ITT_OK;
}

int itt_dsa_provider_destroy(itt_dsa_provider* p) {
  delete p;
  return ITT_OK;
}

// itt_analyze_opts.sa_provider on the root (sa_user = the provider)
int itt_dsa_provide(void* user, const int32_t* tokens, uint64_t n, int32_t term, uint32_t cap, uint32_t* sa, uint32_t* lcp) {
  auto* p = static_cast<itt_dsa_provider*>(user);
  if (!p || p->p.T->r != p->p.root) return ITT_E_INVALID_ARGUMENT;
  return dguarded(p->p.ctx, [&](Ctx* c) {
    uint64_t hdr[3] = {n, static_cast<uint64_t>(static_cast<uint32_t>(term)), cap};
    p->p.T->bcast_host(c, hdr, 3, p->p.root);
    DBuf<int32_t> text(c, n + 1);
    if (n) ITT_CUDA(cudaMemcpyAsync(text.p, tokens, n * 4, cudaMemcpyDeviceToDevice, c->stream));
    ITT_CUDA(cudaMemcpyAsync(text.p + n, &hdr[1], 4, cudaMemcpyHostToDevice, c->stream));
    c->sync();
    dsa::provide_round(p->p, n, term, cap, text, sa, lcp);
  });
}

int itt_dsa_serve(itt_dsa_provider* p) {  // the other ranks, until the root's itt_dsa_stop
  if (!p) return ITT_E_INVALID_ARGUMENT;
  for (;;) {
    uint64_t hdr[3] = {0, 0, 0};
    bool stop = false;
    const int rc = dguarded(p->p.ctx, [&](Ctx* c) {
      p->p.T->bcast_host(c, hdr, 3, p->p.root);
      if (hdr[0] == ~0ull) {
        stop = true;
        return;
      }
      DBuf<int32_t> text(c, hdr[0] + 1);
      dsa::provide_round(p->p, hdr[0], static_cast<int32_t>(static_cast<uint32_t>(hdr[1])), static_cast<uint32_t>(hdr[2]),
                         text, nullptr, nullptr);
    });
    if (rc) return rc;
    if (stop) return ITT_OK;
  }
}

int itt_dsa_stop(itt_dsa_provider* p) {
  if (!p) return ITT_E_INVALID_ARGUMENT;
  return dguarded(p->p.ctx, [&](Ctx* c) {
    uint64_t hdr[3] = {~0ull, 0, 0};
    p->p.T->bcast_host(c, hdr, 3, p->p.root);
  });
}

int itt_dsa_last_info(itt_dsa_provider* p, itt_dsa_info* info) {
  if (!p || !info) return ITT_E_INVALID_ARGUMENT;
  const dsa::Slice& s = p->p.last;
  *info = itt_dsa_info{s.rounds, 0, s.groups, s.h_final, s.cap};
  return ITT_OK;
}

}  // extern "C"
