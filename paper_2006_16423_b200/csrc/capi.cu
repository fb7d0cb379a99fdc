// capi.cu — the C-ABI (include/dsg_b200.h) over the sm_100a kernels.
//
// dsg_dp_solve replaces MaxloadDp (/root/reference/proj/src/dp_solver.cpp:
// 116-405) behind the same contract: same validation and error order as the
// MaxloadDp constructor (133-166), same budget semantics (ideals.cpp:69),
// same optimum and the same fewest-devices rule (337-351).  The host part is
// O(|V|^2/64): flatten the Graph, convert every weight to int64 fixed point
// at the common denominator D (exact: the DP only adds, subtracts, maxes and
// mins), build adjacency bitsets, upload.  Everything O(#ideals) or more runs
// on the device: enumeration (enumerate.cu), descriptors (describe.cu), and
// one transition + finalize launch per lattice level (transition.cu).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <unordered_map>
#include <vector>

#include "dsg_b200.h"
#include "dsg_device.cuh"
#include "dsg_internal.h"

#define DSG_TIME_KERNELS_FLAG DSG_FLAG_TIME_KERNELS

// device->host copy on the solve's stream, counted for the e2e record
#define D2H_3(dst, src, bytes)                                                           \
  do {                                                                                   \
    ctx.d2h_bytes += (int64_t)(bytes);                                                   \
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx.stream));            \
  } while (0)
#define D2H(...) D2H_3(__VA_ARGS__)

namespace dsg {

static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

}  // namespace dsg

namespace {

using namespace dsg;
using i128 = __int128;
using Clock = std::chrono::steady_clock;

struct Fail {
  int status;
  std::string msg;
  int64_t limit = 0;
};

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      throw Fail{DSG_CUDA_ERROR, std::string(#x) + " (capi.cu:" + std::to_string(__LINE__) + \
                                     "): " + cudaGetErrorString(e_)};                  \
  } while (0)

// DSG_DEBUG_SYNC=1: synchronise after a launch group and name it in the
// error (debugging aid; the sanitizer is not available on the GPU pool)
#define debug_sync(ctx, what)                                                              \
  do {                                                                                     \
    static const bool on_ = std::getenv("DSG_DEBUG_SYNC") != nullptr;                      \
    if (on_) {                                                                             \
      cudaError_t e_ = cudaStreamSynchronize((ctx).stream);                                \
      if (e_ != cudaSuccess)                                                               \
        throw Fail{DSG_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e_)};     \
    }                                                                                      \
  } while (0)

double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

// DSG_PREP_TRACE=1: host timestamps of a solve's steps on stderr (diagnostics)
void host_mark(const char* what) {
  static const bool on = std::getenv("DSG_PREP_TRACE") != nullptr;
  if (!on) return;
  static Clock::time_point last = Clock::now();
  const auto now = Clock::now();
  std::fprintf(stderr, "host %-14s +%.3f ms\n", what, ms_since(last));
  last = now;
}

// ------------------------------------------------------------ device arena
// Named device buffers reused across solves on one device (grow-only), so a
// repeated solve does no cudaMalloc.  One context per device, one solve at a
// time per device (the mutex); independent devices run concurrently.
struct DeviceCtx {
  int device = -1;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  std::map<std::string, std::pair<void*, size_t>> bufs;
  void* pinned = nullptr;
  size_t pinned_cap = 0;
  int64_t h2d_bytes = 0, d2h_bytes = 0;  // per solve, for the bench's e2e record
  cudaEvent_t ev_end = nullptr;

  void* get(const std::string& name, size_t bytes) {
    if (bytes == 0) bytes = 8;
    auto& b = bufs[name];
    if (b.second < bytes) {
      if (b.first) CK(cudaFree(b.first));
      b.first = nullptr;
      size_t cap = std::max(bytes, b.second + b.second / 2);
      CK(cudaMalloc(&b.first, cap));
      b.second = cap;
    }
    return b.first;
  }
  void release_prefix(const std::string& prefix) {
    for (auto it = bufs.begin(); it != bufs.end();) {
      if (it->first.compare(0, prefix.size(), prefix) == 0) {
        if (it->second.first) cudaFree(it->second.first);
        it = bufs.erase(it);
      } else {
        ++it;
      }
    }
    for (auto it = pinned_named.begin(); it != pinned_named.end();) {
      if (it->first.compare(0, prefix.size(), prefix) == 0) {
        if (it->second.first) cudaFreeHost(it->second.first);
        it = pinned_named.erase(it);
      } else {
        ++it;
      }
    }
  }
  template <typename T>
  T* get_t(const std::string& name, size_t count) {
    return static_cast<T*>(get(name, count * sizeof(T)));
  }
  // pinned device->host landing areas (per pipeline prefix) for a solve's
  // small results: copies into them stay asynchronous (a D2H into pageable
  // memory waits for the copy)
  std::map<std::string, std::pair<void*, size_t>> pinned_named;
  void* rb(const std::string& name, size_t bytes) {
    auto& b = pinned_named[name];
    if (b.second < bytes) {
      if (b.first) cudaFreeHost(b.first);
      b.first = nullptr;
      CK(cudaMallocHost(&b.first, bytes));
      b.second = bytes;
    }
    return b.first;
  }
  void* host(size_t bytes) {
    if (pinned_cap < bytes) {
      if (pinned) cudaFreeHost(pinned);
      pinned = nullptr;
      size_t cap = std::max(bytes, pinned_cap * 2);
      CK(cudaMallocHost(&pinned, cap));
      pinned_cap = cap;
    }
    return pinned;
  }
};

std::mutex g_ctx_mu;
std::map<int, std::unique_ptr<DeviceCtx>> g_ctx;

DeviceCtx& context(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw Fail{DSG_CUDA_ERROR, std::string("no CUDA device: ") + cudaGetErrorString(e)};
  if (device < 0) CK(cudaGetDevice(&device));
  if (device >= count) throw Fail{DSG_CUDA_ERROR, "device ordinal out of range"};
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  auto& p = g_ctx[device];
  if (!p) {
    p = std::make_unique<DeviceCtx>();
    p->device = device;
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      throw Fail{DSG_CUDA_ERROR, "libdsg_b200 is built for sm_100a (B200); found sm_" +
                                     std::to_string(prop.major * 10 + prop.minor)};
    p->sm_count = prop.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
  }
  return *p;
}

// ------------------------------------------------------------ host prepare
struct Q {  // exact rational
  int64_t num = 0, den = 1;
  bool inf = false;
};

int64_t gcd64(int64_t a, int64_t b) {
  // binary GCD (no divisions); |INT64_MIN| is taken as 2^63 unsigned
  uint64_t x = a < 0 ? 0ull - (uint64_t)a : (uint64_t)a;
  uint64_t y = b < 0 ? 0ull - (uint64_t)b : (uint64_t)b;
  if (!x) return (int64_t)y;
  if (!y) return (int64_t)x;
  const int sh = __builtin_ctzll(x | y);
  x >>= __builtin_ctzll(x);
  do {
    y >>= __builtin_ctzll(y);
    if (x > y) std::swap(x, y);
    y -= x;
  } while (y);
  return (int64_t)(x << sh);
}

Q to_q(dsg_rat r) {
  Q q;
  if (r.den == 0) {
    if (r.num <= 0) throw Fail{DSG_INVALID, "invalid rational"};
    q.inf = true;
    return q;
  }
  if (r.num == INT64_MIN || r.den == INT64_MIN) {
    // the one case whose negation leaves int64: 128-bit path
    i128 n = r.num, d = r.den;
    if (d < 0) {
      n = -n;
      d = -d;
    }
    i128 g = gcd64((int64_t)(n < 0 ? -n : n), (int64_t)d);
    if (g > 1) {
      n /= g;
      d /= g;
    }
    if (n > INT64_MAX || n < INT64_MIN || d > INT64_MAX) throw Fail{DSG_OVERFLOW, "rational overflow"};
    q.num = (int64_t)n;
    q.den = (int64_t)d;
    return q;
  }
  int64_t n = r.num, d = r.den;
  if (d < 0) {
    n = -n;
    d = -d;
  }
  const int64_t g = gcd64(n, d);
  if (g > 1) {
    n /= g;
    d /= g;
  }
  q.num = n;
  q.den = d;
  return q;
}

// Adjacency lists in CSR form, filled in edge order (as push_back would).
struct Adjl {
  std::vector<int> off, adj;
  struct Range {
    const int *b, *e;
    const int* begin() const { return b; }
    const int* end() const { return e; }
    size_t size() const { return (size_t)(e - b); }
  };
  Range operator[](int v) const { return {adj.data() + off[v], adj.data() + off[v + 1]}; }
};

struct Prepared {
  int n = 0, W = 0, K = 0, L = 0, C = 0;
  bool training = false;
  std::vector<int32_t> ids;
  std::vector<int64_t> cpu, acc, comm, mem;
  std::vector<uint8_t> unsup, comminf, in_universe, bw;
  std::vector<uint64_t> succ_real, pred_real, pred_u, succ_u, twins, bw_succ, bw_from, bw_to,
      bwset;
  std::vector<int32_t> out_off, out_adj, in_off, in_adj;
  std::vector<int32_t> pu_off, pu_adj, su_off, su_adj;  // universe CSR, unique
  int64_t D = 1;
  int value_bits = 64;
  int64_t mlim = 0;
  int memcheck = 0;
  int interleave = 0;
  bool has_bw = false;
  bool inf_cpu_mem = false;  // deferred std::domain_error("subtracting infinity")
  bool neg_comm = false;     // some finite comm_time < 0 (acc >= proc fails under Sum)
  bool repl = false;         // solve_maxload_replicated
  int repl_combine = 0;
  int64_t repl_bn = 1, repl_bd = 1;
  int repl_sign = 1;
};

void set_bit(std::vector<uint64_t>& m, int row, int W, int v) {
  m[(size_t)row * W + (v >> 6)] |= 1ull << (v & 63);
}

// Graph::Graph + MaxloadDp ctor checks (graph.cpp:132-158, dp_solver.cpp:133-166)
Prepared prepare(int mode, const dsg_graph* g, const dsg_config* cfg, const uint8_t* within,
                 bool enumerate_only, int flags) {
  Prepared P;
  // DSG_PREP_TRACE=1: host ms per prepare step on stderr (diagnostics)
  static const bool prep_trace = std::getenv("DSG_PREP_TRACE") != nullptr;
  auto prep_t = Clock::now();
#define PREP_MARK(name)                                                      \
  do {                                                                       \
    if (prep_trace) {                                                        \
      std::fprintf(stderr, "prep %-10s %.3f ms\n", name, ms_since(prep_t)); \
      prep_t = Clock::now();                                                 \
    }                                                                        \
  } while (0)
  if (!g || g->n_nodes < 0) throw Fail{DSG_INVALID, "invalid graph"};
  const int n = g->n_nodes;
  if (n > kMaxWords * 64)
    throw Fail{DSG_UNSUPPORTED, "graphs above " + std::to_string(kMaxWords * 64) + " nodes"};
  P.n = n;
  P.W = std::max(1, (n + 63) / 64);
  const int W = P.W;
  P.ids.assign(g->ids, g->ids + n);
  // external id -> dense index, first wins: a direct table when the ids are
  // dense enough, else a hash map
  int32_t id_lo = 0, id_hi = -1;
  for (int i = 0; i < n; ++i) {
    id_lo = i ? std::min(id_lo, g->ids[i]) : g->ids[i];
    id_hi = i ? std::max(id_hi, g->ids[i]) : g->ids[i];
  }
  const bool direct = n > 0 && (int64_t)id_hi - id_lo < 4 * (int64_t)n + 64;
  std::vector<int> table;
  std::unordered_map<int32_t, int> index;
  if (direct) {
    table.assign((size_t)((int64_t)id_hi - id_lo + 1), -1);
    for (int i = 0; i < n; ++i)
      if (table[g->ids[i] - id_lo] < 0) table[g->ids[i] - id_lo] = i;
  } else {
    index.reserve(n * 2 + 1);
    for (int i = 0; i < n; ++i) index.emplace(g->ids[i], i);
  }
  auto idx_of = [&](int32_t id) {
    if (direct) return id < id_lo || id > id_hi ? -1 : table[id - id_lo];
    auto it = index.find(id);
    return it == index.end() ? -1 : it->second;
  };
  // resolved edges (dangling ends dropped), then CSR lists by counting
  std::vector<int> ef, et;
  ef.reserve(g->n_edges + g->n_artificial);
  et.reserve(g->n_edges + g->n_artificial);
  for (int e = 0; e < g->n_edges; ++e) {
    int f = idx_of(g->edge_from[e]), t = idx_of(g->edge_to[e]);
    if (f < 0 || t < 0) continue;
    ef.push_back(f);
    et.push_back(t);
  }
  const size_t n_real = ef.size();
  for (int e = 0; e < g->n_artificial; ++e) {
    int f = idx_of(g->art_from[e]), t = idx_of(g->art_to[e]);
    if (f < 0 || t < 0) continue;
    ef.push_back(f);
    et.push_back(t);
  }
  auto build_adj = [&](size_t m, const std::vector<int>& from, const std::vector<int>& to,
                       Adjl& out) {
    out.off.assign(n + 1, 0);
    out.adj.resize(m);
    for (size_t e = 0; e < m; ++e) ++out.off[from[e] + 1];
    for (int v = 0; v < n; ++v) out.off[v + 1] += out.off[v];
    std::vector<int> pos(out.off.begin(), out.off.end() - 1);
    for (size_t e = 0; e < m; ++e) out.adj[pos[from[e]]++] = to[e];
  };
  Adjl out_real, in_real, out_all, in_all;
  build_adj(n_real, ef, et, out_real);
  build_adj(n_real, et, ef, in_real);
  build_adj(ef.size(), ef, et, out_all);
  build_adj(ef.size(), et, ef, in_all);
  P.bw.assign(n, 0);
  for (int i = 0; i < n; ++i) P.bw[i] = g->is_backward ? (g->is_backward[i] != 0) : 0;
  P.has_bw = std::any_of(P.bw.begin(), P.bw.end(), [](uint8_t b) { return b != 0; });

  // weights (validated even for enumeration, as the Graph holds Rats)
  std::vector<Q> qc(n), qa(n), qm(n), qmem(n);
  for (int i = 0; i < n; ++i) {
    qc[i] = to_q(g->cpu_time[i]);
    qa[i] = to_q(g->acc_time[i]);
    qm[i] = to_q(g->comm_time[i]);
    qmem[i] = to_q(g->mem_size[i]);
  }

  PREP_MARK("weights");
  // acyclicity over real + artificial edges (the reference assumes a
  // validated DAG; a cycle would leave the universe unreachable)
  {
    std::vector<int> indeg(n, 0), ready;
    for (int v = 0; v < n; ++v)
      for (int w : out_all[v]) ++indeg[w];
    for (int v = 0; v < n; ++v)
      if (!indeg[v]) ready.push_back(v);
    int seen = 0;
    while (!ready.empty()) {
      int v = ready.back();
      ready.pop_back();
      ++seen;
      for (int w : out_all[v])
        if (--indeg[w] == 0) ready.push_back(w);
    }
    if (seen != n) throw Fail{DSG_INVALID, "graph has a cycle (validate_dag first)"};
  }

  PREP_MARK("acyclic");
  std::vector<std::vector<int>> paired_bw(n);
  P.in_universe.assign(n, 0);
  if (enumerate_only) {
    for (int v = 0; v < n; ++v) P.in_universe[v] = within ? (within[v] != 0) : 1;
  } else {
    P.K = cfg->accelerators;
    P.L = cfg->cpus;
    if (mode == DSG_MODE_REPLICATED) {  // dp_solver.cpp:397-405
      if (!cfg->has_bandwidth) throw Fail{DSG_MISSING_BANDWIDTH, "replication requires a bandwidth value"};
      if (P.has_bw) throw Fail{DSG_INVALID, "replicated solve expects an inference graph"};
    }
    if (P.K + P.L < 1) throw Fail{DSG_INVALID, "need at least one device"};
    if (P.K < 0 || P.L < 0) throw Fail{DSG_INVALID, "negative device count"};
    if (mode == DSG_MODE_REPLICATED) {
      const Q b = to_q(cfg->bandwidth);
      if (b.inf) throw Fail{DSG_INVALID, "dividing by infinity"};
      if (b.num == 0 && P.K >= 2) throw Fail{DSG_INVALID, "division by zero"};
      P.repl = true;
      P.repl_combine = cfg->replication_combine == DSG_REPL_MAX ? 1 : 0;
      P.repl_bn = b.num < 0 ? -b.num : (b.num == 0 ? 1 : b.num);
      P.repl_bd = b.den;
      P.repl_sign = b.num < 0 ? -1 : 1;
    }
    P.C = (P.K + 1) * (P.L + 1);
    P.training = mode == DSG_MODE_TRAINING;
    if (P.training) {
      for (int v = 0; v < n; ++v) P.in_universe[v] = !P.bw[v];
      for (int b = 0; b < n; ++b) {
        if (!P.bw[b]) continue;
        int32_t pid = g->forward_pair ? g->forward_pair[b] : DSG_NO_PAIR;
        if (pid == DSG_NO_PAIR)
          throw Fail{DSG_INVALID,
                     "training solve requires every backward node to be paired (run "
                     "preprocessing first)"};
        int f = idx_of(pid);
        if (f < 0) throw Fail{DSG_INVALID, "forward_pair references missing node"};
        paired_bw[f].push_back(b);
      }
    } else {
      std::fill(P.in_universe.begin(), P.in_universe.end(), 1);
    }
  }

  // nodes the DP ever adds to a block: universe + paired backward twins
  std::vector<uint8_t> added(n, 0);
  for (int v = 0; v < n; ++v) {
    if (!P.in_universe[v]) continue;
    added[v] = 1;
    for (int b : paired_bw[v]) added[b] = 1;
  }
  for (int v = 0; v < n; ++v)
    if (added[v] && (qc[v].inf || qmem[v].inf)) P.inf_cpu_mem = true;

  PREP_MARK("universe");
  // ---- fixed point at the common denominator D (exact)
  int64_t D64 = 1;  // <= 2^62 throughout
  auto lcm_in = [&](const Q& q) {
    if (q.inf || q.den == 1 || D64 % q.den == 0) return;
    const int64_t gg = gcd64(D64, q.den);
    const i128 nd = (i128)(D64 / gg) * q.den;
    if (nd > ((i128)1 << 62)) throw Fail{DSG_OVERFLOW, "common denominator overflow"};
    D64 = (int64_t)nd;
  };
  for (int v = 0; v < n; ++v) {
    lcm_in(qc[v]);
    lcm_in(qa[v]);
    lcm_in(qm[v]);
    lcm_in(qmem[v]);
  }
  Q qlim;
  if (!enumerate_only) {
    qlim = to_q(cfg->memory_limit);
    lcm_in(qlim);
  }
  // replication divides by r <= K and by the bandwidth: scale every value by
  // S = lcm(1..K) * |b_num| so base/r and (r-1)*mem*b_den/(r*b_num) stay
  // exact integers (replicated_load, dp_solver.cpp:100-108)
  i128 S = 1, lcmK = 1;
  if (P.repl) {
    for (int r = 2; r <= P.K; ++r) {
      lcmK = lcmK / gcd64((int64_t)lcmK, r) * r;
      if (lcmK > ((i128)1 << 40)) throw Fail{DSG_OVERFLOW, "replication scale overflow"};
    }
    S = lcmK * P.repl_bn;
    if (S > ((i128)1 << 50)) throw Fail{DSG_OVERFLOW, "replication scale overflow"};
  }
  const i128 D = D64;
  if (D * S > ((i128)1 << 62)) throw Fail{DSG_OVERFLOW, "common denominator overflow"};
  P.D = (int64_t)(D * S);
  auto fx = [&](const Q& q) -> i128 { return q.inf ? 0 : (i128)q.num * (D64 / q.den) * S; };
  P.cpu.assign(n, 0);
  P.acc.assign(n, 0);
  P.comm.assign(n, 0);
  P.mem.assign(n, 0);
  P.unsup.assign(n, 0);
  P.comminf.assign(n, 0);
  i128 bound = 0;
  auto absq = [](i128 x) { return x < 0 ? -x : x; };
  for (int v = 0; v < n; ++v) {
    i128 c = fx(qc[v]), a = fx(qa[v]), m = fx(qm[v]), s = fx(qmem[v]);
    bound += absq(c) + absq(a) + 2 * absq(m) + absq(s);
    if (bound > ((i128)1 << 62)) throw Fail{DSG_OVERFLOW, "fixed-point weight sum overflow"};
    P.cpu[v] = (int64_t)c;
    P.acc[v] = (int64_t)a;
    P.comm[v] = (int64_t)m;
    P.mem[v] = (int64_t)s;
    P.unsup[v] = qa[v].inf;
    P.comminf[v] = qm[v].inf;
    if (!qm[v].inf && qm[v].num < 0) P.neg_comm = true;
  }
  if (P.repl) {
    // sync terms reach (K-1)/K * Σ|mem| * b_den / |b_num| on top of the loads
    i128 mem_total = 0;
    for (int v = 0; v < n; ++v) mem_total += absq((i128)P.mem[v]);
    bound += 2 * (mem_total / P.repl_bn + 1) * P.repl_bd;
    if (bound > ((i128)1 << 62)) throw Fail{DSG_OVERFLOW, "fixed-point weight sum overflow"};
  }
  P.value_bits = (bound < ((i128)1 << 30) && !(flags & DSG_FLAG_FORCE_INT64)) ? 32 : 64;
  if (!enumerate_only) {
    P.memcheck = qlim.inf ? 0 : 1;
    if (!qlim.inf) {
      i128 m = fx(qlim);
      i128 cap = bound + 1;
      P.mlim = (int64_t)std::max(-cap, std::min(cap, m));
    }
    P.interleave = cfg->interleaving;
    if (P.interleave < 0 || P.interleave > 2) throw Fail{DSG_INVALID, "bad interleaving mode"};
  }

  PREP_MARK("fixedpoint");
  // ---- adjacency bitsets and CSR
  const size_t NW = (size_t)n * W;
  // [n][W] rows only where a kernel reads them: pred_real never (lists
  // serve), twins only for training, bw_succ only with backward nodes
  // (succ_real, pred_u and succ_u rows are built on the device from the
  // lists: launch_adj_bits in upload_graph)
  P.pred_real.assign(W, 0);
  P.twins.assign(P.training ? NW : (size_t)W, 0);
  P.bw_succ.assign(P.has_bw ? NW : (size_t)W, 0);
  P.bwset.assign(W, 0);
  P.out_off.assign(n + 1, 0);
  P.in_off.assign(n + 1, 0);
  for (int v = 0; v < n; ++v) {
    P.out_off[v + 1] = P.out_off[v] + (int)out_real[v].size();
    P.in_off[v + 1] = P.in_off[v] + (int)in_real[v].size();
    for (int b : paired_bw[v]) set_bit(P.twins, v, W, b);
    if (P.bw[v]) {
      P.bwset[v >> 6] |= 1ull << (v & 63);
      for (int w : out_all[v])
        if (P.bw[w]) set_bit(P.bw_succ, v, W, w);
    }
  }
  PREP_MARK("bitsets");
  P.out_adj.assign(out_real.adj.begin(), out_real.adj.end());
  P.in_adj.assign(in_real.adj.begin(), in_real.adj.end());
  if (P.out_adj.empty()) P.out_adj.push_back(0);
  if (P.in_adj.empty()) P.in_adj.push_back(0);
  // the same universe adjacency as lists: sorted, unique (as a bit scan of
  // pred_u / succ_u would give)
  auto to_csr = [&](const Adjl& lists, std::vector<int32_t>& off, std::vector<int32_t>& adj) {
    off.assign(n + 1, 0);
    adj.clear();
    adj.reserve(lists.adj.size());
    for (int v = 0; v < n; ++v) {
      const size_t b0 = adj.size();
      if (P.in_universe[v])
        for (int u : lists[v])
          if (P.in_universe[u]) adj.push_back(u);
      std::sort(adj.begin() + b0, adj.end());
      adj.erase(std::unique(adj.begin() + b0, adj.end()), adj.end());
      off[v + 1] = (int32_t)adj.size();
    }
    if (adj.empty()) adj.push_back(0);
  };
  to_csr(in_all, P.pu_off, P.pu_adj);
  to_csr(out_all, P.su_off, P.su_adj);
  PREP_MARK("csr");
  // reachability_within(g, backward) for the general training gate
  // (graph.cpp:291-345): rows in reverse topological order
  if (P.training && P.has_bw) {
    P.bw_from.assign(NW, 0);
    P.bw_to.assign(NW, 0);
    std::vector<int> indeg(n, 0), order, ready;
    for (int v = 0; v < n; ++v)
      if (P.bw[v])
        for (int w : out_all[v])
          if (P.bw[w]) ++indeg[w];
    for (int v = n - 1; v >= 0; --v)
      if (P.bw[v] && !indeg[v]) ready.push_back(v);
    while (!ready.empty()) {
      int v = ready.back();
      ready.pop_back();
      order.push_back(v);
      for (int w : out_all[v])
        if (P.bw[w] && --indeg[w] == 0) ready.push_back(w);
    }
    for (auto it = order.rbegin(); it != order.rend(); ++it) {
      int u = *it;
      set_bit(P.bw_from, u, W, u);
      for (int w : out_all[u]) {
        if (!P.bw[w]) continue;
        for (int k = 0; k < W; ++k) P.bw_from[(size_t)u * W + k] |= P.bw_from[(size_t)w * W + k];
      }
    }
    for (int u = 0; u < n; ++u) {
      if (!P.bw[u]) continue;
      for (int k = 0; k < W; ++k)
        for (uint64_t x = P.bw_from[(size_t)u * W + k]; x; x &= x - 1)
          set_bit(P.bw_to, (k << 6) | __builtin_ctzll(x), W, u);
    }
  } else {
    P.bw_from.assign(W, 0);
    P.bw_to.assign(W, 0);
  }
  PREP_MARK("reach");
#undef PREP_MARK
  return P;
}

template <typename T>
T* upload(DeviceCtx& ctx, const std::string& name, const std::vector<T>& v) {
  T* d = ctx.get_t<T>(name, std::max<size_t>(v.size(), 1));
  if (!v.empty()) {
    CK(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, ctx.stream));
    ctx.h2d_bytes += (int64_t)(v.size() * sizeof(T));
  }
  return d;
}

struct DeviceGraph {
  DevGraph g;
  uint8_t* in_universe;
  int32_t *pu_off, *pu_adj, *su_off, *su_adj;
};

// Every host array of the prepared graph packed into the context's pinned
// staging buffer and moved with ONE host->device copy into one device buffer
// (two dozen pageable cudaMemcpyAsync calls cost ~0.2 ms per solve).
struct Packer {
  std::vector<std::pair<const void*, size_t>> parts;
  std::vector<size_t> offs;
  size_t total = 0;
  template <typename T>
  size_t add(const std::vector<T>& v) {
    const size_t off = total;
    const size_t bytes = std::max<size_t>(v.size(), 1) * sizeof(T);
    parts.push_back({v.empty() ? nullptr : v.data(), v.size() * sizeof(T)});
    offs.push_back(off);
    total = off + ((bytes + 15) & ~(size_t)15);
    return off;
  }
};

DeviceGraph upload_graph(DeviceCtx& ctx, const Prepared& P, const std::string& prefix) {
  Packer pk;
  const size_t o_cpu = pk.add(P.cpu), o_acc = pk.add(P.acc), o_comm = pk.add(P.comm),
               o_mem = pk.add(P.mem), o_unsup = pk.add(P.unsup), o_comminf = pk.add(P.comminf),
               o_pr = pk.add(P.pred_real), o_tw = pk.add(P.twins), o_bws = pk.add(P.bw_succ),
               o_bwf = pk.add(P.bw_from), o_bwt = pk.add(P.bw_to), o_bwset = pk.add(P.bwset),
               o_oo = pk.add(P.out_off), o_oa = pk.add(P.out_adj), o_io = pk.add(P.in_off),
               o_ia = pk.add(P.in_adj), o_univ = pk.add(P.in_universe), o_puo = pk.add(P.pu_off),
               o_pua = pk.add(P.pu_adj), o_suo = pk.add(P.su_off), o_sua = pk.add(P.su_adj);
  char* host = static_cast<char*>(ctx.host(pk.total));
  for (size_t i = 0; i < pk.parts.size(); ++i)
    if (pk.parts[i].second) std::memcpy(host + pk.offs[i], pk.parts[i].first, pk.parts[i].second);
  char* dev = static_cast<char*>(ctx.get(prefix + "graph", pk.total));
  CK(cudaMemcpyAsync(dev, host, pk.total, cudaMemcpyHostToDevice, ctx.stream));
  ctx.h2d_bytes += (int64_t)pk.total;
  // (the staging buffer is next written by the next solve's upload, after
  // this solve's final synchronisation)
  DeviceGraph d;
  DevGraph& g = d.g;
  g.n = P.n;
  g.W = P.W;
  g.cpu = reinterpret_cast<const int64_t*>(dev + o_cpu);
  g.acc = reinterpret_cast<const int64_t*>(dev + o_acc);
  g.comm = reinterpret_cast<const int64_t*>(dev + o_comm);
  g.mem = reinterpret_cast<const int64_t*>(dev + o_mem);
  g.unsup = reinterpret_cast<const uint8_t*>(dev + o_unsup);
  g.comminf = reinterpret_cast<const uint8_t*>(dev + o_comminf);
  g.pred_real = reinterpret_cast<const uint64_t*>(dev + o_pr);
  g.twins = reinterpret_cast<const uint64_t*>(dev + o_tw);
  g.bw_succ = reinterpret_cast<const uint64_t*>(dev + o_bws);
  g.bw_from = reinterpret_cast<const uint64_t*>(dev + o_bwf);
  g.bw_to = reinterpret_cast<const uint64_t*>(dev + o_bwt);
  g.bwset = reinterpret_cast<const uint64_t*>(dev + o_bwset);
  g.out_real_off = reinterpret_cast<const int32_t*>(dev + o_oo);
  g.out_real_adj = reinterpret_cast<const int32_t*>(dev + o_oa);
  g.in_real_off = reinterpret_cast<const int32_t*>(dev + o_io);
  g.in_real_adj = reinterpret_cast<const int32_t*>(dev + o_ia);
  d.in_universe = reinterpret_cast<uint8_t*>(dev + o_univ);
  d.pu_off = reinterpret_cast<int32_t*>(dev + o_puo);
  d.pu_adj = reinterpret_cast<int32_t*>(dev + o_pua);
  d.su_off = reinterpret_cast<int32_t*>(dev + o_suo);
  d.su_adj = reinterpret_cast<int32_t*>(dev + o_sua);
  // [n][W] adjacency rows from the lists, on the device (C4: 0.9 MB of host
  // bit setting and H2D per solve before)
  const size_t NW = (size_t)std::max(1, P.n) * P.W;
  uint64_t* rows = ctx.get_t<uint64_t>(prefix + "adj.rows", 3 * NW);
  CK(cudaMemsetAsync(rows, 0, 3 * NW * sizeof(uint64_t), ctx.stream));
  launch_adj_bits(P.n, P.W, d.pu_off, d.pu_adj, d.su_off, d.su_adj, g.out_real_off, g.out_real_adj,
                  rows, rows + NW, rows + 2 * NW, ctx.stream);
  g.pred_u = rows;
  g.succ_u = rows + NW;
  g.succ_real = rows + 2 * NW;
  return d;
}

// ------------------------------------------------------------ enumeration
struct Lattice {
  int64_t I = 0;
  int n_levels = 0;
  std::vector<int64_t> level_off;  // host copy, n_levels + 1
  uint64_t* sbits = nullptr;       // sorted, device
  uint64_t* smax = nullptr;        // maximal elements of each ideal, same order
  const int* lvl_pre = nullptr;    // each level's common word prefix (null: not computed)
};

Lattice enumerate_device(DeviceCtx& ctx, const Prepared& P, const DeviceGraph& dg, int64_t budget,
                         bool hash_mode, const std::string& pfx) {
  const int W = P.W;
  const int64_t budget_eff = std::max<int64_t>(budget, 1);
  int64_t cap = std::min<int64_t>(budget_eff + 1, std::max<int64_t>(4096, (int64_t(1) << 22) / W));
  int64_t cand_cap = hash_mode ? cap * 4 : 0;
  EnumStatus* st_d = ctx.get_t<EnumStatus>("enum.status", 1);
  int64_t* lvl_d = ctx.get_t<int64_t>("enum.level_off", (size_t)P.n + 3);
  for (int attempt = 0; attempt < 8; ++attempt) {
    EnumLaunch L{};
    L.W = W;
    L.n = P.n;
    L.pred_u = dg.g.pred_u;
    L.succ_u = dg.g.succ_u;
    L.in_universe = dg.in_universe;
    L.pu_off = dg.pu_off;
    L.pu_adj = dg.pu_adj;
    L.su_off = dg.su_off;
    L.su_adj = dg.su_adj;
    L.n_pu = (int)P.pu_off[P.n];
    L.n_su = (int)P.su_off[P.n];
    L.bits = ctx.get_t<uint64_t>("enum.bits", (size_t)cap * W);
    L.maxm = ctx.get_t<uint64_t>("enum.maxm", (size_t)cap * W);
    L.addm = ctx.get_t<uint64_t>("enum.addm", (size_t)cap * W);
    L.level_of = ctx.get_t<int32_t>("enum.level_of", (size_t)cap);
    L.spill_par = ctx.get_t<int32_t>("enum.spill_par", (size_t)cap);
    L.spill_v = ctx.get_t<int32_t>("enum.spill_v", (size_t)cap);
    L.cap = cap;
    L.budget = budget_eff;
    L.level_off = lvl_d;
    L.status = st_d;
    L.hash_mode = hash_mode ? 1 : 0;
    if (hash_mode) {
      L.cand_bits = ctx.get_t<uint64_t>("enum.cbits", (size_t)cand_cap * W);
      L.cand_maxm = ctx.get_t<uint64_t>("enum.cmaxm", (size_t)cand_cap * W);
      L.cand_addm = ctx.get_t<uint64_t>("enum.caddm", (size_t)cand_cap * W);
      L.cand_cap = cand_cap;
      int64_t tc = 1024;
      while (tc < 2 * cand_cap) tc <<= 1;
      L.table = ctx.get_t<int64_t>("enum.table", (size_t)tc);
      L.table_cap = tc;
    }
    CK(cudaMemsetAsync(st_d, 0, sizeof(EnumStatus), ctx.stream));
    L.resume = 0;
    launch_enumerate(L, ctx.stream);
    CK(cudaGetLastError());
    debug_sync(ctx, "enumerate");
    EnumStatus st;
    D2H(&st, st_d, sizeof st);
    host_mark("enum-sync-in");
    CK(cudaStreamSynchronize(ctx.stream));
    host_mark("enum-sync-out");
    if (st.code == 4) {
      // a level wider than one CTA's frontier: the cluster walk continues
      // from it (enumerate.cu enumerate_cluster_kernel)
      CK(cudaMemsetAsync(&st_d->code, 0, sizeof(int32_t), ctx.stream));
      L.resume = 1;
      launch_enumerate(L, ctx.stream);
      CK(cudaGetLastError());
      debug_sync(ctx, "enumerate (cluster)");
      D2H(&st, st_d, sizeof st);
      CK(cudaStreamSynchronize(ctx.stream));
    }
    if (st.code == 1) throw Fail{DSG_BUDGET, "ideal budget exceeded", budget};
    if (st.code == 2) {
      cap = std::min<int64_t>(budget_eff + 1, std::max(cap * 2, st.needed + st.needed / 2));
      if (hash_mode) cand_cap = std::max(cand_cap, cap * 4);
      continue;
    }
    if (st.code == 3) {
      cand_cap = std::max(cand_cap * 2, st.needed * 2);
      continue;
    }
    Lattice lat;
    lat.I = st.total;
    lat.n_levels = st.n_levels;
    lat.level_off.resize(lat.n_levels + 1);
    D2H(lat.level_off.data(), lvl_d, sizeof(int64_t) * (lat.n_levels + 1));
    lat.sbits = ctx.get_t<uint64_t>(pfx + "lat.sbits", (size_t)lat.I * W);
    lat.smax = ctx.get_t<uint64_t>(pfx + "lat.smax", (size_t)lat.I * W);
    int64_t max_level = 0;
    for (int s = 0; s < lat.n_levels; ++s)
      max_level = std::max(max_level, lat.level_off[s + 1] - lat.level_off[s]);
    int64_t* perm_a = ctx.get_t<int64_t>("enum.perm_a", (size_t)lat.I);
    int64_t* perm_b = ctx.get_t<int64_t>("enum.perm_b", (size_t)lat.I);
    int* lvl_pre = ctx.get_t<int>(pfx + "lat.lvl_pre", (size_t)lat.n_levels + 1);
    lat.lvl_pre = launch_lex_rank(W, lat.I, L.bits, L.maxm, L.level_of, lvl_d, lat.sbits, lat.smax,
                                  max_level, perm_a, perm_b, lvl_pre, lat.n_levels, ctx.stream)
                      ? lvl_pre
                      : nullptr;
    CK(cudaGetLastError());
    debug_sync(ctx, "lex rank");
    return lat;
  }
  throw Fail{DSG_CUDA_ERROR, "enumeration capacity retries exhausted"};
}

void fill_msg(char* dst, const std::string& s) {
  std::strncpy(dst, s.c_str(), 255);
  dst[255] = 0;
}

// one end-of-pipeline event per device context (phase 2 records it)
cudaEvent_t pl_ev_end(DeviceCtx& ctx) {
  if (!ctx.ev_end) CK(cudaEventCreate(&ctx.ev_end));
  return ctx.ev_end;
}

struct Pipeline;
void write_trace(DeviceCtx& ctx, const Pipeline& pl, const char* path);

// One solve's small device->host results, landing in pinned memory (followed
// by the traceback arrays: kinds [maxb], loads [maxb], block bits [maxb][W]).
struct Readback {
  int64_t n_cov;
  int64_t totals[kNumCounts];
  int32_t cov_bad;
  int32_t flags[2];  // stop, watchdog
  int32_t tables_bad;
  unsigned long long pairs;
  TraceState tb;
};

// ------------------------------------------------------------ solve
// Phase 1: lattice, descriptors, chunk plan, DP buffers.  Phase 2: reset, all
// DP levels (one persistent cooperative launch), traceback.  Every solve runs
// both phases (nothing is cached between solves); buffers are named per
// session so their addresses stay stable across solves of the same graph —
// which is what lets a sharded session (one process per GPU) exchange CUDA
// IPC handles of its dp / bp / level-counter buffers once and then run every
// solve with the finalizers of all ranks storing rows into all ranks' tables
// over NVLink (persistent.cu).
struct Pipeline {
  std::string pfx;
  Lattice lat;
  int64_t I = 0;
  DescribeLaunch D{};
  LevelLaunch LL{};
  PersistPlan PP{};
  PersistInfo pinfo{};
  bool persistent = true;
  std::vector<int64_t> n_chunks, chunk_len, item_base;
  int4* items_d = nullptr;  // readiness-ordered work items (device)
  ItemBuild item_build{};
  std::vector<int32_t> mode;
  int64_t total_tiles = 0, total_items = 0;
  unsigned* ctl = nullptr;  // [0] stop, [1] err, [32 + s] level s done
  size_t ctl_words = 0;
  int rank = 0, world = 1;
  // virtual shards (dsg_options::shard_count > 1): all `world` ranks run in
  // this process's one cooperative launch, each with its own tables
  bool virt = false;
  std::vector<std::vector<int4>> run_lists;  // chain-runner items per (virtual) rank
  std::vector<VRank> vranks;  // host copy; [0] aliases the tables above
  VRank* vranks_d = nullptr;
  int* tables_bad = nullptr;  // replica comparison after the solve
  std::vector<void*> peer_dp;
  std::vector<int32_t*> peer_bp;
  int64_t* level_off_d = nullptr;
  int32_t* level_of_d = nullptr;
  std::vector<unsigned*> peer_done;
  std::vector<void*> ipc_opened;
  double t_enum_ms = 0, t_desc_ms = 0;
  Readback* rbk = nullptr;  // pinned, this pipeline's
};

// The persistent plan's host tables (chunk plan, run lists, mode table,
// virtual-rank records, peer lists) staged in pinned memory and moved with ONE
// host->device copy into one device buffer (a dozen pageable copies cost
// ~0.1 ms of host time with the GPU idle).  Each table's device pointer is
// written through `out` at flush().
struct PlanStage {
  struct Ent {
    const void* src;
    size_t bytes, off;
    void** out;
  };
  std::vector<Ent> ents;
  size_t total = 0;
  template <typename T>
  void add(const T* src, size_t count, T** out) {
    const size_t bytes = count * sizeof(T);
    ents.push_back({src, bytes, total, reinterpret_cast<void**>(out)});
    total += (std::max<size_t>(bytes, 8) + 15) & ~(size_t)15;
  }
  template <typename T>
  void add(const std::vector<T>& v, T** out) {
    add(v.data(), v.size(), out);
  }
  void flush(DeviceCtx& ctx, const std::string& pfx, cudaStream_t st) {
    if (!total) return;
    uint8_t* host = static_cast<uint8_t*>(ctx.rb(pfx + "plan", total));
    uint8_t* dev = static_cast<uint8_t*>(ctx.get(pfx + "pp.plan", total));
    for (const Ent& e : ents) {
      if (e.bytes) std::memcpy(host + e.off, e.src, e.bytes);
      *e.out = dev + e.off;
    }
    CK(cudaMemcpyAsync(dev, host, total, cudaMemcpyHostToDevice, st));
    ctx.h2d_bytes += (int64_t)total;
  }
};

void phase1(DeviceCtx& ctx, const Prepared& P, const DeviceGraph& dg, const dsg_options* opt,
            Pipeline& pl) {
  const int flags = opt->flags;
  cudaStream_t st = ctx.stream;
  const std::string& pfx = pl.pfx;
  const int W = P.W, K = P.K, Lc = P.L, C = P.C;
  const int vb = P.value_bits;
  const size_t vsz = vb == 32 ? 4 : 8;
  if (opt->shard_count > 1) {
    // virtual shards: the multi-GPU wavefront's ranks emulated in one launch
    if (opt->shard_count > DSG_MAX_SHARDS) throw Fail{DSG_INVALID, "shard_count above DSG_MAX_SHARDS"};
    if (pl.world > 1 && !pl.virt)
      throw Fail{DSG_UNSUPPORTED, "virtual shards inside a multi-GPU sharded session"};
    if (flags & DSG_FLAG_LEVEL_LAUNCH)
      throw Fail{DSG_UNSUPPORTED, "virtual shards need the persistent level kernel"};
    pl.virt = true;
    pl.world = opt->shard_count;
    pl.rank = 0;
  }
  const auto t1 = Clock::now();
  pl.lat = enumerate_device(ctx, P, dg, opt->ideal_budget, (flags & DSG_FLAG_HASH_ENUM) != 0, pfx);
  const Lattice& lat = pl.lat;
  pl.t_enum_ms = ms_since(t1);
  if (P.inf_cpu_mem) throw Fail{DSG_INVALID, "subtracting infinity"};
  const int64_t I = lat.I;
  pl.I = I;

  // level of every ordinal (dependency waits, covers, traceback)
  pl.level_off_d = ctx.get_t<int64_t>(pfx + "pp.level_off", lat.level_off.size() + 1);
  CK(cudaMemcpyAsync(pl.level_off_d, lat.level_off.data(), sizeof(int64_t) * lat.level_off.size(),
                     cudaMemcpyHostToDevice, st));
  ctx.h2d_bytes += (int64_t)(sizeof(int64_t) * lat.level_off.size());
  pl.level_of_d = ctx.get_t<int32_t>(pfx + "pp.level_of", (size_t)I);
  launch_level_of(pl.level_off_d, lat.n_levels, I, pl.level_of_d, st);
  // lower covers (the newest-level sources of every target, no subset scan)
  int64_t* cov_off = ctx.get_t<int64_t>(pfx + "lat.cov_off", (size_t)I + 1);
  launch_cover_count(W, I, lat.smax, cov_off, st);
  launch_scan_counts(cov_off, I, 1, st);
  {
    const int maxb = K + Lc + 1;
    pl.rbk = static_cast<Readback*>(ctx.rb(pfx + "rb", sizeof(Readback) + 16 +
                                                          (size_t)maxb * (4 + 8 + 8 * W)));
    std::memset(pl.rbk, 0, sizeof(Readback));
  }
  Readback& rbk = *pl.rbk;
  D2H(&rbk.n_cov, cov_off + I, sizeof(int64_t));

  // ---- descriptors
  const auto t2 = Clock::now();
  DescribeLaunch& D = pl.D;
  D = DescribeLaunch{};
  D.g = dg.g;
  D.training = P.training ? 1 : 0;
  D.has_bw = (P.training && P.has_bw) ? 1 : 0;
  D.value_bits = vb;
  D.I = I;
  D.sbits = lat.sbits;
  D.AW = (W + 1) & ~1;
  D.abits = ctx.get_t<uint64_t>(pfx + "d.abits", (size_t)I * D.AW);
  D.intbits = ctx.get_t<uint64_t>(pfx + "d.intbits", P.training ? (size_t)I * W : 1);
  D.pfx_cpu = ctx.get(pfx + "d.cpu", I * vsz);
  D.pfx_acc = ctx.get(pfx + "d.acc", I * vsz);
  D.pfx_mem = ctx.get(pfx + "d.mem", I * vsz);
  D.unsup = ctx.get_t<int32_t>(pfx + "d.unsup", I);
  D.fw = ctx.get(pfx + "d.fw", I * vsz);
  D.fwinf = ctx.get_t<int32_t>(pfx + "d.fwinf", I);
  D.upset = ctx.get_t<uint8_t>(pfx + "d.upset", I);
  D.srec = ctx.get_t<SrcRec>(pfx + "d.srec", I);
  D.counts = ctx.get_t<int64_t>(pfx + "d.counts", (size_t)kNumCounts * (I + 1));
  CK(cudaMemsetAsync(D.counts, 0, sizeof(int64_t) * kNumCounts * (I + 1), st));
  launch_describe(D, false, st);
  launch_scan_counts(D.counts, I, kNumCounts, st);
  for (int k = 0; k < kNumCounts; ++k)
    D2H(&rbk.totals[k], D.counts + (size_t)k * (I + 1) + I, sizeof(int64_t));
  host_mark("cnt-sync-in");
  CK(cudaStreamSynchronize(st));  // pool sizes: the one synchronisation after the lattice
  host_mark("cnt-sync-out");
  CK(cudaGetLastError());
  const int64_t* totals = rbk.totals;
  const int64_t n_cov = rbk.n_cov;
  if (totals[kCntF] > INT32_MAX || totals[kCntN] > INT32_MAX || totals[kCntLItems] > INT32_MAX)
    throw Fail{DSG_UNSUPPORTED, "frontier tables exceed 2^31 entries"};
  D.chunks = ctx.get_t<FChunk>(pfx + "d.chunks", totals[kCntChunks]);
  D.fpool = ctx.get(pfx + "d.fpool", totals[kCntF] * vsz);
  D.nitems = ctx.get_t<NItem>(pfx + "d.nitems", totals[kCntN]);
  D.pitems = ctx.get_t<PItem>(pfx + "d.pitems", totals[kCntP]);
  D.lentries = ctx.get_t<LEntry>(pfx + "d.lentries", totals[kCntL]);
  D.litems = ctx.get_t<MaskItem>(pfx + "d.litems", totals[kCntLItems]);
  launch_describe(D, true, st);
  CK(cudaGetLastError());
  if (n_cov > INT32_MAX) throw Fail{DSG_UNSUPPORTED, "cover lists exceed 2^31 entries"};
  int32_t* cov = ctx.get_t<int32_t>(pfx + "lat.cov", (size_t)n_cov + 1);
  int* cov_err = ctx.get_t<int>(pfx + "lat.cov_err", 1);
  CK(cudaMemsetAsync(cov_err, 0, sizeof(int), st));
  launch_cover_fill(W, I, lat.sbits, lat.smax, pl.level_of_d, pl.level_off_d, cov_off, cov,
                    lat.lvl_pre, cov_err, st);
  pl.t_desc_ms = ms_since(t2);

  // ---- DP tables and launch parameters
  pl.persistent = !(flags & DSG_FLAG_LEVEL_LAUNCH);
  LevelLaunch& LL = pl.LL;
  LL = LevelLaunch{};
  LL.value_bits = vb;
  LL.training = P.training ? 1 : 0;
  LL.has_bw = D.has_bw;
  LL.fastgate = (flags & DSG_FLAG_NO_FASTGATE) ? 0 : 1;
  LL.K = K;
  LL.L = Lc;
  LL.C = C;
  LL.W = W;
  LL.mlim = P.mlim;
  LL.memcheck = P.memcheck;
  LL.interleave = P.interleave;
  LL.repl = P.repl ? 1 : 0;
  LL.repl_combine = P.repl_combine;
  LL.repl_bn = P.repl_bn;
  LL.repl_bd = P.repl_bd;
  LL.repl_sign = P.repl_sign;
  // the exact pruning assumes acc(B) >= proc(B), which negative comm weights
  // break under Interleaving::Sum (graph.cpp:457-467): no pruning then
  LL.no_prune = (P.neg_comm && P.interleave == DSG_INTERLEAVE_SUM) ? 1 : 0;
  if ((i128)I * (K + 2) >= ((i128)1 << 31))
    throw Fail{DSG_UNSUPPORTED, "ideal count x (accelerators + 2) exceeds the 31-bit argmin"};
  LL.abits = D.abits;
  LL.AW = D.AW;
  LL.intbits = D.intbits;
  LL.pfx_cpu = D.pfx_cpu;
  LL.pfx_acc = D.pfx_acc;
  LL.pfx_mem = D.pfx_mem;
  LL.unsup = D.unsup;
  LL.fw = D.fw;
  LL.fwinf = D.fwinf;
  LL.upset = D.upset;
  LL.srec = D.srec;
  LL.chunk_off = D.counts + (size_t)kCntChunks * (I + 1);
  LL.chunks = D.chunks;
  LL.fpool = D.fpool;
  LL.nitems = D.nitems;
  LL.p_off = D.counts + (size_t)kCntP * (I + 1);
  LL.pitems = D.pitems;
  LL.l_off = D.counts + (size_t)kCntL * (I + 1);
  LL.lentries = D.lentries;
  LL.litems = D.litems;
  LL.bwset = dg.g.bwset;
  LL.bw_from = dg.g.bw_from;
  LL.bw_to = dg.g.bw_to;
  LL.n_nodes = P.n;
  LL.cov_off = cov_off;
  LL.cov = cov;
  {
    int64_t* cmax = ctx.get_t<int64_t>(pfx + "d.cmax", 4 * (size_t)((I + kChunkMaxLen - 1) / kChunkMaxLen) + 4);
    launch_chunk_max(D.srec, I, cmax, st);
    LL.cmax = cmax;
  }
  LL.dp = ctx.get(pfx + "dp.values", (size_t)I * C * vsz + 64);  // + staging slack
  LL.bp = nullptr;  // values only; the traceback re-derives the argmins
  LL.pair_counter = ctx.get_t<unsigned long long>(pfx + "dp.pairs", 1);
  LL.stats = ctx.get_t<unsigned long long>(pfx + "dp.stats", 8);

  // ---- chunk plan
  pl.pinfo = PersistInfo{};
  if (pl.persistent) {
    PersistPlan q{};  // what sizes the CTA's shared memory (see the chunk plan)
    q.chunk_len0 = q.chunk_len1 = 64;
    if (const char* e = std::getenv("DSG_CHUNK_LEN")) q.chunk_len0 = std::max(4, std::atoi(e));
    if (const char* e = std::getenv("DSG_CHUNK_LEN1")) q.chunk_len1 = std::max(4, std::atoi(e));
    q.stage = 1;
    if (const char* e = std::getenv("DSG_STAGE")) q.stage = std::atoi(e) != 0;
    query_persistent(LL, q, &pl.pinfo);
    if (pl.pinfo.blocks <= 0) {
      // the CTA's shared memory does not fit (very large (K+1)(L+1) with
      // 64-bit values): the per-level driver needs none of it
      if (pl.virt) throw Fail{DSG_UNSUPPORTED, "virtual shards: persistent kernel does not fit"};
      pl.persistent = false;
    } else if (opt->reserved > 0) {
      pl.pinfo.blocks = std::min(pl.pinfo.blocks, opt->reserved);
    }
    // every virtual rank needs at least one CTA
    if (pl.virt) pl.pinfo.blocks = std::max(pl.pinfo.blocks, pl.world);
  }
  const int64_t target_items =
      pl.persistent ? std::max(1, pl.pinfo.blocks) : (int64_t)ctx.sm_count * 8;
  pl.n_chunks.assign(lat.n_levels, 1);
  pl.chunk_len.assign(lat.n_levels, 1);
  pl.mode.assign(lat.n_levels, 0);
  pl.item_base.assign(lat.n_levels + 1, 0);
  std::vector<int64_t> tile_base(lat.n_levels, 0);
  std::vector<int64_t> chunk_lo, chunk_base(lat.n_levels, 0);
  size_t part_elems = 1;
  pl.total_tiles = 0;
  pl.total_items = 0;
  // persistent, mode 0 (>= 16 targets): (32-target group, chunk) CTA items
  // whose 4 warps split the chunk; mode 1 (< 16 targets): (target, chunk)
  // items with one source per thread.  Items are claimed in readiness order
  // (see the item list below).  Per-level path: 128-target tiles x uniform
  // chunks of >= 16 sources.
  const int64_t kSmallLevel = 16;
  // mode 0: old sources (levels <= s-2) in short implicit chunks (chunk c =
  // sources [c*len, (c+1)*len), len 64: measured best on C2/C3 once the
  // newest level moved to the cover chunk; 48 / 96 are 3-5 % slower) — with
  // readiness-ordered claims the scan stays balanced and no long item sits
  // on the critical path; mode 1: old sources in cost-balanced chunks of
  // <= 128 (explicit boundaries).  Both: one cover chunk for level s-1.
  int64_t chunk_len0 = 64, chunk_len1 = 64;
  int grade = 1;
  if (const char* e = std::getenv("DSG_GRADE")) grade = std::max(1, std::atoi(e));
  int grade1 = 5;  // mode 1: recent old levels chunked per level (C4 with 24 runners: 3 -> 4.75 ms,
                   // 5 -> 4.53 ms; C1-C3, C5 flat)
  if (const char* e = std::getenv("DSG_GRADE1")) grade1 = std::max(0, std::atoi(e));
  int64_t fin_fold_max = 32;  // mode 1: the finisher folds level s-2 up to this size
  if (const char* e = std::getenv("DSG_FIN_FOLD")) fin_fold_max = std::max(0, std::atoi(e));
  int runner_max_t = 16;  // chain runner: finishers of mode-1 levels with <= this many targets
                          // (C4 DP: 4 -> 5.21 ms, 8 -> 4.99, 12..64 -> 4.93; C1-C3, C5 flat)
  if (const char* e = std::getenv("DSG_RUNNER_T")) runner_max_t = std::max(0, std::atoi(e));
  int fold_levels = 1;  // measured on C4: folding s-3 too costs the finisher more than it saves
  if (const char* e = std::getenv("DSG_FOLD_LEVELS")) fold_levels = std::max(0, std::atoi(e));
  int runners = 16;  // runner CTAs per rank (C4: 16 < 8 < 4 runners in DP ms)
  const char* runners_env = std::getenv("DSG_RUNNERS");
  if (runners_env) runners = std::max(1, std::atoi(runners_env));
  // the runners' finishers wait for chunks only the other CTAs claim: keep
  // the runner off unless most of the grid is left for them
  if (!pl.persistent || pl.pinfo.blocks < 4 * runners * pl.world) runner_max_t = 0;
  // chain blocks (persistent_impl.cuh): runs of single-target levels whose
  // predecessor level is single-target too, folded by one runner CTA with the
  // recent rows in shared memory; the staging area must hold the block state
  // off by default: measured on C4 (DP 4.86 ms without; 8.6 / 7.2 / 6.5 / 6.7 ms with F = 16 / 8 /
  // 4 / 2) and C1 (0.33 vs 0.44-0.51 ms) — a chain level costs ~2 us of CTA-wide barriers and
  // dependent shared-memory steps on an SM shared with six scanning CTAs, more than the L2 hand-off
  // between runner CTAs it removes
  int chain_fmax = 0;  // levels folded by a chain level (its old chunks end before them)
  if (const char* e = std::getenv("DSG_CHAIN_F")) chain_fmax = std::max(0, std::atoi(e));
  bool chain_on = runner_max_t > 0 && chain_fmax > 0 && !P.repl && C <= kTileTargets;
  {
    const int n_stage = (int)std::max(chunk_len0, chunk_len1);
    const size_t staging = std::getenv("DSG_STAGE") && std::atoi(std::getenv("DSG_STAGE")) == 0
                               ? 0
                               : 16 + (size_t)n_stage * (LL.AW * 8 + sizeof(SrcRec) + (size_t)C * vsz) + 32;
    if (chain_smem_need(C, LL.AW, W, vsz) > staging) chain_on = false;
  }
  std::vector<int> chain_f(lat.n_levels, -1);  // F of a chain level, -1: not one
  for (int s = 3; chain_on && s < lat.n_levels; ++s) {
    if (lat.level_off[s + 1] - lat.level_off[s] != 1 || lat.level_off[s] - lat.level_off[s - 1] != 1)
      continue;
    int F = 0;
    while (F < std::min(chain_fmax, s - 2) &&
           lat.level_off[s - 1] - lat.level_off[s - 2 - F] <= kChainSrcMax - 1)
      ++F;
    chain_f[s] = F;
  }
  unsigned poll_ns_max = 128;  // measured: 128 ns <= 256 ns (C1 -4 %, C3 -1 %, C4 -1 %, C2 =) and beats 1 us
  if (const char* e = std::getenv("DSG_CHUNK_LEN")) chunk_len0 = std::max(4, std::atoi(e));
  if (const char* e = std::getenv("DSG_CHUNK_LEN1")) chunk_len1 = std::max(4, std::atoi(e));
  if (const char* e = std::getenv("DSG_POLL_NS")) poll_ns_max = (unsigned)std::max(32, std::atoi(e));
  for (int s = 1; s < lat.n_levels; ++s) {
    const int64_t T = lat.level_off[s + 1] - lat.level_off[s];
    const int64_t S = lat.level_off[s];
    int64_t units, min_chunk;
    if (!pl.persistent) {
      units = (T + kTileTargets - 1) / kTileTargets;
      min_chunk = 16;
    } else if (T < kSmallLevel) {
      pl.mode[s] = 1;
      units = T;
      min_chunk = kTileTargets;
    } else {
      units = (T + 31) / 32;
      min_chunk = 4;
    }
    int64_t chunks = std::max<int64_t>(1, (target_items + units - 1) / units);
    // The newest level's sources are handled by ONE cover chunk (the last
    // chunk): each target's lower covers (enumerate.cu) are exactly its
    // nested sources in level s-1, so that critical chunk evaluates a handful
    // of pairs instead of scanning the whole level.
    if (pl.persistent && pl.mode[s] == 0) {
      // as mode0_chunk (persistent.cu): old levels, graded recent levels, cover
      const int G = std::min(grade, s - 1);
      const int64_t Rg = lat.level_off[s - 1 - G];
      chunks = (Rg + chunk_len0 - 1) / chunk_len0 + 1;
      for (int d = G; d >= 1; --d) {
        const int64_t len = std::min(chunk_len0, chunk_len1 << (d - 1));
        chunks += (lat.level_off[s - d] - lat.level_off[s - 1 - d] + len - 1) / len;
      }
      chunk_base[s] = -1;
      pl.chunk_len[s] = chunk_len0;
    } else if (pl.persistent) {
      // mode 1: sources below level s-1-G1 in cost-balanced chunks of <= 128
      // (one per thread); each of the G1 most recent old levels s-1-G1 ..
      // s-2 in chunks of its own, so the item that waits for level s-2 (on
      // the level-to-level chain of a narrow lattice) holds only that
      // level's few sources; then the cover chunk (the finisher)
      const int G1 = chain_f[s] >= 0 ? chain_f[s] : std::max(0, std::min(grade1, s - 2));
      const int64_t R = s >= 2 ? lat.level_off[s - 1] : 0;
      const int64_t Rg = s >= 2 ? lat.level_off[s - 1 - G1] : 0;
      chunk_base[s] = (int64_t)chunk_lo.size();
      const int64_t oc = (Rg + kTileTargets - 1) / kTileTargets;
      const int64_t olen = oc ? (Rg + oc - 1) / oc : 1;
      for (int64_t c = 0; c < oc; ++c) chunk_lo.push_back(std::min(Rg, c * olen));
      chunks = oc;
      // the F most recent old levels s-2 .. s-1-F, when small, are folded by
      // the finisher itself (mode 1 + F): no separate items — and no arrival
      // round trips — between those levels and level s
      int F = 0;
      while (F < std::min(G1, fold_levels) &&
             lat.level_off[s - 1] - lat.level_off[s - 2 - F] <= fin_fold_max)
        ++F;
      if (chain_f[s] >= 0) F = chain_f[s];
      pl.mode[s] = 1 + F;
      for (int j = s - 1 - G1; j <= s - 2 - F && G1 > 0; ++j) {
        const int64_t lo = lat.level_off[j], n = lat.level_off[j + 1] - lo;
        const int64_t nc = (n + kTileTargets - 1) / kTileTargets, len = (n + nc - 1) / nc;
        for (int64_t c = 0; c < nc; ++c) chunk_lo.push_back(lo + c * len);
        chunks += nc;
      }
      chunk_lo.push_back(lat.level_off[s - 1 - F]);
      chunks += 1;
      pl.chunk_len[s] = 0;
    } else {
      chunks = std::min<int64_t>(chunks, std::max<int64_t>(1, S / min_chunk));
      const int64_t len = (S + chunks - 1) / chunks;
      chunks = (S + len - 1) / len;
      pl.chunk_len[s] = len;
    }
    pl.n_chunks[s] = chunks;
    tile_base[s] = pl.total_tiles;
    pl.total_tiles += units;
    pl.item_base[s] = pl.total_items;
    pl.total_items += units * chunks;
    part_elems = std::max(part_elems, (size_t)(chunks * C * T));
  }
  pl.item_base[lat.n_levels] = pl.total_items;
  if (pl.persistent) {
    // the dataflow kernel merges every chunk into the target's keys with a
    // value atomicMin (both item shapes): no partials
    part_elems = 1;
  }
  LL.part_val = ctx.get(pfx + "dp.part_val", part_elems * vsz);
  LL.part_arg = nullptr;
  if (!pl.persistent) return;

  // ---- persistent plan (device copies)
  PersistPlan& PP = pl.PP;
  PP = PersistPlan{};
  PP.n_levels = lat.n_levels;
  PlanStage stage;
  auto up64 = [&](const std::vector<int64_t>& v, const int64_t** out) {
    stage.add(v.data(), v.size(), const_cast<int64_t**>(out));
  };
  PP.level_off = pl.level_off_d;
  PP.level_of = pl.level_of_d;
  up64(pl.n_chunks, &PP.n_chunks);
  up64(pl.chunk_len, &PP.chunk_len);
  up64(chunk_lo, &PP.chunk_lo);
  up64(chunk_base, &PP.chunk_base);
  up64(tile_base, &PP.tile_base);
  PP.chunk_len0 = (int)chunk_len0;
  PP.stage = 1;
  if (const char* e = std::getenv("DSG_STAGE")) PP.stage = std::atoi(e) != 0;
  PP.chunk_len1 = (int)chunk_len1;
  PP.dead_skip = 1;
  if (const char* e = std::getenv("DSG_DEAD_SKIP")) PP.dead_skip = std::atoi(e) != 0;

  PP.grade = grade;
  PP.poll_ns_max = poll_ns_max;
  // narrow-level cell polls spin (few pollers, each on the level-to-level
  // chain): C1 DP 0.42 -> 0.37 ms, C4 4.97 -> 4.89 ms, C2/C3/C5 flat
  PP.fin_poll_ns = 0;
  if (const char* e = std::getenv("DSG_FIN_POLL_NS")) PP.fin_poll_ns = (unsigned)std::max(0, std::atoi(e));
  // work items in readiness order, built on the device (launch_build_items):
  // buckets by dep = level of the chunk's last source, critical items first;
  // a sharded solve lists only this rank's units (virtual shards: one list
  // per rank)
  std::vector<int64_t> rank_items(pl.virt ? pl.world : 1, 0);
  std::vector<int64_t> pair_off(lat.n_levels + 1, 0);  // staged: lives until the flush
  const int64_t* pair_off_d = nullptr;
  {
    for (int l = 1; l < lat.n_levels; ++l) pair_off[l + 1] = pair_off[l] + pl.n_chunks[l];
    auto runner_level = [&](int l) {
      return runner_max_t > 0 && pl.mode[l] != 0 &&
             lat.level_off[l + 1] - lat.level_off[l] <= runner_max_t;
    };
    auto items_of_rank = [&](int rank) {
      int64_t total = 0;
      for (int l = 1; l < lat.n_levels; ++l) {
        const int64_t T = lat.level_off[l + 1] - lat.level_off[l];
        const int64_t units = pl.mode[l] == 0 ? (T + 31) / 32 : T;
        const int64_t units_r =
            pl.world > 1 ? (units > rank ? (units - rank + pl.world - 1) / pl.world : 0) : units;
        total += (pl.n_chunks[l] - (runner_level(l) ? 1 : 0)) * units_r;
      }
      return total;
    };
    // the chain runners' lists, per rank (units u % world == rank): the
    // finishers of narrow mode-1 levels, and the chain blocks (a chain level
    // run: up to kChainBlk levels per block, a block's levels' old chunks all
    // reading levels before the block), in level order; runner i takes
    // segment i (header: run_items[i].y = start of segment i, i <= runners),
    // a whole chain in one segment, the rest round-robin
    // a lattice that is mostly narrow levels (C4: 1,469 of 1,517) keeps more
    // finishers in flight with 24 runners (C4 DP -1.7 %; C1 flat; C2, whose
    // narrow levels are a minority, keeps 16)
    if (!runners_env && runner_max_t > 0) {
      int narrow = 0;
      for (int l = 1; l < lat.n_levels; ++l) narrow += runner_level(l) ? 1 : 0;
      if (2 * narrow > lat.n_levels && pl.pinfo.blocks >= 4 * 24 * pl.world) runners = 24;
    }
    pl.run_lists.assign(pl.virt ? pl.world : 1, {});
    int chain_blk = 8;  // levels per chain block (<= persistent_impl.cuh kChainBlk)
    if (const char* e = std::getenv("DSG_CHAIN_BLK")) chain_blk = std::max(1, std::min(8, std::atoi(e)));
    for (size_t r = 0; r < pl.run_lists.size(); ++r) {
      const int rank = pl.virt ? (int)r : pl.rank;
      std::vector<std::vector<int4>> seg(runners);
      int rr = 0;
      for (int l = 1; l < lat.n_levels; ++l) {
        if (!runner_level(l)) continue;
        const int64_t T = lat.level_off[l + 1] - lat.level_off[l];
        if (chain_f[l] >= 0) {
          if (rank != 0) continue;  // single-target levels: unit 0, rank 0
          int b = l;
          while (b + 1 < lat.n_levels && chain_f[b + 1] >= 0) ++b;
          auto& sg = seg[rr++ % runners];
          for (int blk = l; blk <= b;) {
            int e = blk;
            while (e + 1 <= b && e + 1 - blk < chain_blk && (e + 1) - 2 - chain_f[e + 1] < blk) ++e;
            // .w: the run's first level (its rows onwards sit in the runner's ring)
            sg.push_back(make_int4(blk, -(e - blk + 1), (int)(pl.n_chunks[blk] - 1), l));
            blk = e + 1;
          }
          l = b;
          continue;
        }
        for (int64_t u = pl.world > 1 ? rank : 0; u < T; u += pl.world)
          seg[rr++ % runners].push_back(make_int4(l, (int)u, (int)(pl.n_chunks[l] - 1), l - 1));
      }
      std::vector<int4>& out = pl.run_lists[r];
      out.assign(runners + 1, make_int4(-1, 0, 0, 0));
      for (int i = 0; i < runners; ++i) {
        out[i].y = (int)out.size();
        out.insert(out.end(), seg[i].begin(), seg[i].end());
      }
      out[runners].y = (int)out.size();
    }
    PP.chain = chain_on ? (std::getenv("DSG_CHAIN_DEBUG") ? 2 : 1) : 0;
    for (size_t r = 0; r < rank_items.size(); ++r)
      rank_items[r] = items_of_rank(pl.virt ? (int)r : pl.rank);
    pl.total_items = rank_items[0];
    ItemBuild B{};
    B.runner_max_t = runner_max_t;
    B.lag = 1 << 30;
    if (const char* e = std::getenv("DSG_SCHED_LAG")) B.lag = std::max(1, std::atoi(e));
    // dedicated cover-item CTAs (needs >= 2 CTAs: one of each role; one
    // queue per rank with virtual shards)
    int crit_ctas = 0;
    if (const char* e = std::getenv("DSG_CRIT_CTAS")) crit_ctas = std::max(0, std::atoi(e));
    if (crit_ctas >= pl.pinfo.blocks) crit_ctas = pl.pinfo.blocks / 2;
    if (pl.virt) crit_ctas = 0;
    B.split = crit_ctas > 0 ? 1 : 0;
    PP.crit_ctas = crit_ctas;
    B.n_levels = lat.n_levels;
    up64(pair_off, &pair_off_d);  // into the builds after the flush
    B.n_pairs = pair_off[lat.n_levels];
    B.cnt = ctx.get_t<unsigned long long>(pfx + "pp.item_cnt", 4 * (size_t)lat.n_levels + 1);
    B.items = ctx.get_t<int4>(pfx + "pp.items", (size_t)pl.total_items + 1);
    B.rank = pl.rank;
    B.world = pl.world;
    PP.items = B.items;
    PP.total_items = pl.total_items;
    PP.crit_end = B.cnt + 2 * (size_t)lat.n_levels - 1;  // end of the last cover key
    pl.items_d = B.items;
    pl.item_build = B;  // launched after the plan is on the device
  }
  PP.tile_count = ctx.get_t<unsigned>(pfx + "pp.tile_count", (size_t)pl.total_tiles + 1);
  pl.ctl_words = (size_t)lat.n_levels + 64;
  pl.ctl = ctx.get_t<unsigned>(pfx + "pp.ctl", pl.ctl_words);
  PP.stop = reinterpret_cast<int*>(pl.ctl);
  PP.err = reinterpret_cast<int*>(pl.ctl + 1);
  PP.next = reinterpret_cast<unsigned long long*>(pl.ctl + 2);  // ctl[2..3], zeroed per solve
  PP.crit_next = reinterpret_cast<unsigned long long*>(pl.ctl + 4);  // ctl[4..5]
  PP.done = pl.ctl + 32;
  PP.keys = ctx.get_t<unsigned long long>(pfx + "pp.keys", (size_t)I * C);  // value atomics
  PP.virt = 0;
  PP.vrank = nullptr;
  PP.runner_max_t = runner_max_t;
  PP.runners = runners;
  PP.run_total = (int64_t)pl.run_lists[0].size();
  stage.add(pl.run_lists[0], const_cast<int4**>(&PP.run_items));
  stage.add(pl.mode, const_cast<int32_t**>(&PP.mode));
  std::vector<ItemBuild> rank_builds;
  if (pl.virt) {
    // virtual ranks 1..world-1: everything a rank owns on its own GPU
    pl.vranks.assign(pl.world, VRank{});
    rank_builds.assign(pl.world, pl.item_build);
    for (int r = 1; r < pl.world; ++r) {
      const std::string vp = pfx + "v" + std::to_string(r) + ".";
      ItemBuild& B = rank_builds[r];
      B.rank = r;
      B.items = ctx.get_t<int4>(vp + "items", (size_t)rank_items[r] + 1);
      VRank& v = pl.vranks[r];
      v.items = B.items;
      v.total_items = rank_items[r];
      v.ctl = ctx.get_t<unsigned>(vp + "ctl", pl.ctl_words);
      v.tile_count = ctx.get_t<unsigned>(vp + "tile_count", (size_t)pl.total_tiles + 1);
      v.keys = ctx.get_t<unsigned long long>(vp + "keys", (size_t)I * C);
      v.dp = ctx.get(vp + "dp", (size_t)I * C * vsz + 64);
      v.run_total = (int64_t)pl.run_lists[r].size();
      stage.add(pl.run_lists[r], const_cast<int4**>(&v.run_items));
    }
    pl.tables_bad = ctx.get_t<int>(pfx + "pp.tables_bad", 1);
  }
  // peer tables: this GPU only, until a sharded session attaches its peers
  // (virtual shards: every rank's replica in this process)
  if (pl.virt) {
    pl.peer_dp.assign(pl.world, nullptr);
    pl.peer_bp.assign(pl.world, nullptr);
    pl.peer_done.assign(pl.world, nullptr);
    for (int r = 1; r < pl.world; ++r) {
      pl.peer_dp[r] = pl.vranks[r].dp;
      pl.peer_done[r] = pl.vranks[r].ctl + 32;
    }
    pl.peer_dp[0] = LL.dp;
    pl.peer_done[0] = PP.done;
  } else if (pl.world == 1) {
    pl.peer_dp.assign(1, LL.dp);
    pl.peer_bp.assign(1, LL.bp);
    pl.peer_done.assign(1, PP.done);
  }
  stage.add(pl.peer_dp, const_cast<void***>(&PP.peer_dp));
  stage.add(pl.peer_bp, const_cast<int32_t***>(&PP.peer_bp));
  stage.add(pl.peer_done, const_cast<unsigned***>(&PP.peer_done));
  stage.flush(ctx, pfx, st);  // every table above, one copy
  // the virtual-rank records hold the (now known) run-list pointers
  if (pl.virt) {
    pl.vranks[0] = VRank{PP.items, pl.total_items, pl.ctl, PP.tile_count, PP.keys, LL.dp,
                         PP.run_items, PP.run_total};
    pl.vranks_d = ctx.get_t<VRank>(pfx + "pp.vranks", pl.world);
    VRank* vh = static_cast<VRank*>(ctx.rb(pfx + "vranks", sizeof(VRank) * pl.world));
    std::memcpy(vh, pl.vranks.data(), sizeof(VRank) * pl.world);
    CK(cudaMemcpyAsync(pl.vranks_d, vh, sizeof(VRank) * pl.world, cudaMemcpyHostToDevice, st));
    PP.virt = 1;
    PP.vrank = pl.vranks_d;
  }
  pl.item_build.pair_off = pair_off_d;
  for (ItemBuild& B : rank_builds) B.pair_off = pair_off_d;
  launch_build_items(PP, pl.item_build, st);
  for (int r = 1; pl.virt && r < pl.world; ++r) launch_build_items(PP, rank_builds[r], st);
  CK(cudaGetLastError());
  // checked after the solve's one final synchronisation
  D2H(&pl.rbk->cov_bad, cov_err, sizeof(int));
  PP.rank = pl.rank;
  PP.world = pl.world;
}

void write_trace(DeviceCtx& ctx, const Pipeline& pl, const char* path) {
  // debug trace (DSG_TRACE_FILE): header, per-level plan, per-item timestamps
  std::vector<uint64_t> tr((size_t)(pl.total_items + pl.PP.run_total) * 4);
  CK(cudaMemcpyAsync(tr.data(), pl.PP.trace, sizeof(uint64_t) * tr.size(), cudaMemcpyDeviceToHost,
                     ctx.stream));
  CK(cudaStreamSynchronize(ctx.stream));
  if (FILE* f = std::fopen(path, "wb")) {
    int64_t hdr[4] = {pl.lat.n_levels, pl.total_items + pl.PP.run_total, pl.pinfo.blocks, pl.rank};
    std::fwrite(hdr, sizeof hdr, 1, f);
    std::fwrite(pl.lat.level_off.data(), sizeof(int64_t), pl.lat.level_off.size(), f);
    std::fwrite(pl.item_base.data(), sizeof(int64_t), pl.item_base.size(), f);
    std::vector<int4> items((size_t)pl.total_items);
    CK(cudaMemcpy(items.data(), pl.items_d, sizeof(int4) * items.size(), cudaMemcpyDeviceToHost));
    items.insert(items.end(), pl.run_lists[0].begin(), pl.run_lists[0].end());
    std::fwrite(items.data(), sizeof(int4), items.size(), f);
    std::fwrite(pl.n_chunks.data(), sizeof(int64_t), pl.n_chunks.size(), f);
    std::vector<int64_t> m64(pl.mode.begin(), pl.mode.end());
    std::fwrite(m64.data(), sizeof(int64_t), m64.size(), f);
    std::fwrite(tr.data(), sizeof(uint64_t), tr.size(), f);
    std::fclose(f);
  }
}

// Per-solve state: counters, merge keys, the empty ideal's dp row.
void reset_tables(DeviceCtx& ctx, const Prepared& P, Pipeline& pl) {
  cudaStream_t st = ctx.stream;
  const int vb = P.value_bits;
  CK(cudaMemsetAsync(pl.LL.pair_counter, 0, sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(pl.LL.stats, 0, 8 * sizeof(unsigned long long), st));
  // persistent: every row PENDING until final (narrow-level items poll the
  // cells they read instead of a level counter), then the empty ideal's row
  if (pl.persistent) launch_fill_pending(vb, pl.LL.dp, pl.I * P.C, st);
  launch_init_empty(vb, P.K, P.L, pl.LL.dp, st);
  if (pl.persistent) {
    CK(cudaMemsetAsync(pl.PP.tile_count, 0, sizeof(unsigned) * (pl.total_tiles + 1), st));
    CK(cudaMemsetAsync(pl.ctl, 0, sizeof(unsigned) * pl.ctl_words, st));
    // level 0 (the empty ideal) is final before the launch
    launch_fill_u32(pl.PP.done, 1, 1u, st);
    launch_fill_inf(vb, pl.PP.keys, pl.I * P.C, st);
    // virtual ranks 1..world-1: the same per-rank reset every GPU does
    for (size_t r = 1; pl.virt && r < pl.vranks.size(); ++r) {
      const VRank& v = pl.vranks[r];
      launch_fill_pending(vb, v.dp, pl.I * P.C, st);
      launch_init_empty(vb, P.K, P.L, v.dp, st);
      CK(cudaMemsetAsync(v.tile_count, 0, sizeof(unsigned) * (pl.total_tiles + 1), st));
      CK(cudaMemsetAsync(v.ctl, 0, sizeof(unsigned) * pl.ctl_words, st));
      launch_fill_u32(v.ctl + 32, 1, 1u, st);
      launch_fill_inf(vb, v.keys, pl.I * P.C, st);
    }
    if (pl.virt) CK(cudaMemsetAsync(pl.tables_bad, 0, sizeof(int), st));
  }
}

void phase2(DeviceCtx& ctx, const Prepared& P, const dsg_options* opt, Pipeline& pl,
            dsg_result* res, Clock::time_point t0) {
  const int flags = opt->flags;
  cudaStream_t st = ctx.stream;
  const bool timing = (flags & DSG_TIME_KERNELS_FLAG) != 0;
  const bool has_deadline = opt->deadline_seconds > 0;
  const auto deadline = t0 + std::chrono::nanoseconds((int64_t)(opt->deadline_seconds * 1e9));
  const Lattice& lat = pl.lat;
  const int64_t I = pl.I;
  const int W = P.W, K = P.K, Lc = P.L, C = P.C;
  const int vb = P.value_bits;
  LevelLaunch& LL = pl.LL;
  void* dp = LL.dp;
  // this pass's readback fields (cov_bad belongs to phase 1, maybe in flight)
  pl.rbk->tb = TraceState{};
  pl.rbk->flags[0] = pl.rbk->flags[1] = 0;
  pl.rbk->tables_bad = 0;
  pl.rbk->pairs = 0;

  cudaEvent_t ev_desc, ev_dp;
  CK(cudaEventCreate(&ev_desc));
  CK(cudaEventCreate(&ev_dp));
  std::vector<cudaEvent_t> kev, dl_ev;
  const int kDeadlineStride = 8;
  if (pl.persistent) {
    PersistPlan& PP = pl.PP;
    PP.deadline_ns = 0;
    if (has_deadline) {
      uint64_t* gt_d = ctx.get_t<uint64_t>(pl.pfx + "pp.gt", 1);
      uint64_t gt = 0;
      launch_read_globaltimer(gt_d, st);
      D2H(&gt, gt_d, sizeof gt);
      CK(cudaStreamSynchronize(st));
      const int64_t left =
          std::chrono::duration_cast<std::chrono::nanoseconds>(deadline - Clock::now()).count();
      PP.deadline_ns = (int64_t)gt + std::max<int64_t>(left, 1);
    }
    const char* trace_file = std::getenv("DSG_TRACE_FILE");
    PP.trace = nullptr;
    if (trace_file && *trace_file) {
      const size_t n_tr = (size_t)(pl.total_items + PP.run_total) * 4;
      PP.trace = ctx.get_t<uint64_t>(pl.pfx + "pp.trace", n_tr);
      CK(cudaMemsetAsync(PP.trace, 0, sizeof(uint64_t) * n_tr, st));
    }
    CK(cudaEventRecord(ev_desc, st));
    host_mark("dp-launch");
    launch_persistent(LL, PP, st, &pl.pinfo);
    if (pl.pinfo.launch_error != 0)
      throw Fail{DSG_CUDA_ERROR, std::string("cooperative launch failed: ") +
                                     cudaGetErrorString((cudaError_t)pl.pinfo.launch_error)};
    CK(cudaGetLastError());
    CK(cudaEventRecord(ev_dp, st));
    if (PP.trace) write_trace(ctx, pl, trace_file);
    D2H(pl.rbk->flags, PP.stop, sizeof pl.rbk->flags);
    if (pl.virt) {
      // every rank's replica must equal rank 0's byte for byte: each row
      // was stored into every table by the rank that finalized it
      const size_t bytes = (size_t)I * C * (vb == 32 ? 4 : 8);
      for (int r = 1; r < pl.world; ++r)
        launch_compare_tables(pl.vranks[0].dp, pl.vranks[r].dp, bytes, pl.tables_bad, st);
      D2H(&pl.rbk->tables_bad, pl.tables_bad, sizeof(int));
    }
    // stop / watchdog / replica checks wait for the final synchronisation;
    // the traceback reads the stop flags on the device and stands down
  } else {
    CK(cudaEventRecord(ev_desc, st));
    for (int s = 1; s < lat.n_levels; ++s) {
      LL.t_lo = lat.level_off[s];
      LL.t_hi = lat.level_off[s + 1];
      LL.s_hi = lat.level_off[s];
      LL.n_chunks = pl.n_chunks[s];
      LL.chunk_len = pl.chunk_len[s];
      if (timing) {
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        CK(cudaEventRecord(a, st));
        launch_transition(LL, st);
        CK(cudaEventRecord(b, st));
        kev.push_back(a);
        kev.push_back(b);
      } else {
        launch_transition(LL, st);
      }
      launch_finalize(LL, st);
      if (has_deadline && s % kDeadlineStride == 0) {
        // keep at most two strides in flight so the clock tracks the device
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventRecord(e, st));
        dl_ev.push_back(e);
        if (dl_ev.size() >= 2) {
          CK(cudaEventSynchronize(dl_ev[dl_ev.size() - 2]));
          if (Clock::now() > deadline) {
            CK(cudaStreamSynchronize(st));
            for (auto x : dl_ev) cudaEventDestroy(x);
            for (auto x : kev) cudaEventDestroy(x);
            cudaEventDestroy(ev_desc);
            cudaEventDestroy(ev_dp);
            throw Fail{DSG_DEADLINE, "time limit reached"};
          }
        }
      }
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(ev_dp, st));
  }
  res->persistent_blocks = pl.persistent ? pl.pinfo.blocks : 0;

  // ---- traceback (rank 0 of a sharded run holds every row)
  Readback& rbk = *pl.rbk;
  D2H(&rbk.pairs, LL.pair_counter, sizeof rbk.pairs);
#ifdef DSG_PAIR_STATS
  {
    unsigned long long sv[4];
    CK(cudaMemcpyAsync(sv, LL.stats, sizeof sv, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::fprintf(stderr, "DSG_PAIR_STATS {\"count_only\": %llu, \"candidate_test_dropped\": %llu, "
                 "\"frontier_walks\": %llu, \"minmax_updates\": %llu}\n", sv[0], sv[1], sv[2], sv[3]);
  }
#endif
  const bool do_traceback = pl.rank == 0;
  const int maxb = K + Lc + 1;
  int32_t* cpus = reinterpret_cast<int32_t*>(pl.rbk + 1);
  int64_t* loads = reinterpret_cast<int64_t*>(
      reinterpret_cast<uintptr_t>(cpus + maxb + 1) & ~uintptr_t(7));
  uint64_t* bbits = reinterpret_cast<uint64_t*>(loads + maxb);
  if (do_traceback) {
    TraceBuffers tbuf;
    tbuf.state = ctx.get_t<TraceState>(pl.pfx + "tb.state", 1);
    tbuf.n_parts = std::max(1, ctx.sm_count * 2);
    tbuf.part_v = ctx.get(pl.pfx + "tb.part_v", (size_t)tbuf.n_parts * 8);
    tbuf.part_g = ctx.get_t<int32_t>(pl.pfx + "tb.part_g", tbuf.n_parts);
    tbuf.ords = ctx.get_t<int64_t>(pl.pfx + "tb.ords", maxb);
    tbuf.prevs = ctx.get_t<int64_t>(pl.pfx + "tb.prevs", maxb);
    tbuf.kinds = ctx.get_t<int32_t>(pl.pfx + "tb.kinds", maxb);
    tbuf.block_bits = ctx.get_t<uint64_t>(pl.pfx + "tb.bits", (size_t)maxb * W);
    tbuf.loads = ctx.get_t<int64_t>(pl.pfx + "tb.loads", maxb);
    tbuf.abort = pl.persistent ? pl.PP.stop : nullptr;
    launch_traceback(LL, pl.level_of_d, pl.level_off_d, I, ctx.sm_count, tbuf, st);
    D2H(&rbk.tb, tbuf.state, sizeof rbk.tb);
    D2H(cpus, tbuf.kinds, sizeof(int32_t) * maxb);
    D2H(bbits, tbuf.block_bits, sizeof(uint64_t) * maxb * W);
    D2H(loads, tbuf.loads, sizeof(int64_t) * maxb);
  }
  if (flags & DSG_FLAG_KEEP_TABLES) {
    res->words = W;
    res->ideal_bits = (uint64_t*)std::malloc(sizeof(uint64_t) * (size_t)I * W + 8);
    D2H(res->ideal_bits, lat.sbits, sizeof(uint64_t) * (size_t)I * W);
    res->dp_values = (int64_t*)std::malloc(sizeof(int64_t) * (size_t)I * C + 8);
    if (vb == 64) D2H(res->dp_values, dp, sizeof(int64_t) * (size_t)I * C);
  }
  CK(cudaEventRecord(pl_ev_end(ctx), st));
  host_mark("fin-sync-in");
  CK(cudaStreamSynchronize(st));  // the solve's one synchronisation after the lattice
  host_mark("fin-sync-out");
  CK(cudaGetLastError());
  const TraceState& tb = rbk.tb;
  const unsigned long long pairs = rbk.pairs;
  if (rbk.cov_bad) throw Fail{DSG_CUDA_ERROR, "lower-cover lookup failed"};
  if (pl.persistent) {
    if (rbk.flags[1]) throw Fail{DSG_CUDA_ERROR, "dataflow watchdog fired"};
    if (rbk.flags[0]) throw Fail{DSG_DEADLINE, "time limit reached"};
    if (rbk.tables_bad) throw Fail{DSG_LOGIC, "virtual shard dp replicas differ"};
  }
  if ((flags & DSG_FLAG_KEEP_TABLES) && vb == 32) {
    std::vector<int32_t> tmp((size_t)I * C);
    ctx.d2h_bytes += (int64_t)(sizeof(int32_t) * tmp.size());
    CK(cudaMemcpy(tmp.data(), dp, sizeof(int32_t) * tmp.size(), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < tmp.size(); ++i)
      res->dp_values[i] = tmp[i] == VTraits<int32_t>::INF ? INT64_MAX : (int64_t)tmp[i];
  }
  float dp_ms = 0, tb_ms = 0;
  cudaEventElapsedTime(&dp_ms, ev_desc, ev_dp);
  // traceback + result copies: the dp pass's end to the pipeline's end event
  cudaEventElapsedTime(&tb_ms, ev_dp, pl_ev_end(ctx));
  res->t_traceback_ms = tb_ms;
  double kern_ms = 0;
  for (size_t i = 0; i + 1 < kev.size(); i += 2) {
    float x = 0;
    cudaEventElapsedTime(&x, kev[i], kev[i + 1]);
    kern_ms += x;
  }
  for (auto x : kev) cudaEventDestroy(x);
  for (auto x : dl_ev) cudaEventDestroy(x);
  cudaEventDestroy(ev_desc);
  cudaEventDestroy(ev_dp);
  res->t_dp_ms = dp_ms;
  // persistent: the one cooperative launch spans ev_desc..ev_dp
  res->t_transition_kernel_ms = pl.persistent ? dp_ms : kern_ms;
  res->n_pairs = (int64_t)pairs;
  res->n_ideals = I;
  res->n_levels = lat.n_levels;
  res->value_bits = vb;
  res->denominator = P.D;
  res->t_enumerate_ms = pl.t_enum_ms;
  res->t_describe_ms = pl.t_desc_ms;
  if (!do_traceback) return;
  if (tb.status == 2) throw Fail{DSG_INFEASIBLE, "no feasible assignment exists"};
  if (tb.status != 1) throw Fail{DSG_LOGIC, "dp reconstruction stuck"};

  // ---- result
  const int64_t g = gcd64(tb.best_value, P.D);
  res->objective.num = tb.best_value / (g ? g : 1);
  res->objective.den = P.D / (g ? g : 1);
  res->best_k = tb.best_k;
  res->block_loads = 1;
  res->best_l = tb.best_l;
  res->n_blocks = tb.n_blocks;
  res->blocks = (dsg_block*)std::calloc((size_t)std::max(1, tb.n_blocks), sizeof(dsg_block));
  res->members = (int32_t*)std::malloc(sizeof(int32_t) * (size_t)(P.n + 1));
  int off = 0;
  for (int b = 0; b < tb.n_blocks; ++b) {
    dsg_block& blk = res->blocks[b];
    blk.cpu = cpus[b] & 1;
    blk.repl = cpus[b] >> 1;
    blk.offset = off;
    blk.load_num = loads[b];
    for (int w = 0; w < W; ++w) {
      uint64_t x = bbits[(size_t)b * W + w];
      while (x) {
        const int bit = __builtin_ctzll(x);
        x &= x - 1;
        res->members[off++] = w * 64 + bit;
      }
    }
    blk.n_members = off - blk.offset;
  }
}

// Full device pipeline with event timing of the whole thing.
void run_device(DeviceCtx& ctx, const Prepared& P, const DeviceGraph& dg, const dsg_options* opt,
                Pipeline& pl, dsg_result* res, Clock::time_point t0, bool reset) {
  const int64_t launches0 = dsg::g_launches.load();
  ctx.d2h_bytes = 0;
  cudaEvent_t ev_start;
  CK(cudaEventCreate(&ev_start));
  CK(cudaEventRecord(ev_start, ctx.stream));
  phase1(ctx, P, dg, opt, pl);
  if (reset) reset_tables(ctx, P, pl);
  phase2(ctx, P, opt, pl, res, t0);
  float dev_ms = 0;
  cudaEventElapsedTime(&dev_ms, ev_start, pl_ev_end(ctx));
  cudaEventDestroy(ev_start);
  res->t_device_ms = dev_ms;
  res->t_total_ms = ms_since(t0);
  res->kernel_launches = dsg::g_launches.load() - launches0;
  res->h2d_bytes = ctx.h2d_bytes;
  res->d2h_bytes = ctx.d2h_bytes;
}

void solve(int mode, const dsg_graph* graph, const dsg_config* config, const dsg_options* opt,
           dsg_result* res) {
  const auto t0 = Clock::now();
  dsg_options defaults;
  dsg_default_options(&defaults);
  if (!opt) opt = &defaults;
  host_mark("solve-start");
  Prepared P = prepare(mode, graph, config, nullptr, false, opt->flags);
  host_mark("prepared");
  DeviceCtx& ctx = context(opt->device);
  std::lock_guard<std::mutex> lk(ctx.mu);
  CK(cudaSetDevice(ctx.device));
  ctx.h2d_bytes = 0;
  DeviceGraph dg = upload_graph(ctx, P, "g.");
  res->t_prepare_ms = ms_since(t0);
  host_mark("uploaded");
  Pipeline pl;
  run_device(ctx, P, dg, opt, pl, res, t0, true);
}

}  // namespace

// A prepared solve whose graph stays resident on the device (bench: timing
// with inputs already in HBM), optionally one shard of a multi-GPU solve.
struct dsg_session {
  Prepared P;
  DeviceCtx* ctx = nullptr;
  DeviceGraph dg;
  dsg_options opt;
  Pipeline pl;
  bool sharded = false;
  bool reset_done = false;
};

namespace {
std::atomic<int> g_session_ids{0};

template <typename F>
int guarded(dsg_result* result, F&& f) {
  try {
    f();
    result->status = DSG_OK;
  } catch (const Fail& e) {
    result->status = e.status;
    result->budget_limit = e.limit;
    fill_msg(result->message, e.msg);
  } catch (const std::exception& e) {
    result->status = DSG_LOGIC;
    fill_msg(result->message, e.what());
  }
  return result->status;
}
}  // namespace

extern "C" {

dsg_session* dsg_session_create(int32_t mode, const dsg_graph* graph, const dsg_config* config,
                                const dsg_options* options, dsg_result* status_out) {
  std::memset(status_out, 0, sizeof *status_out);
  dsg_session* s = nullptr;
  guarded(status_out, [&] {
    auto t0 = Clock::now();
    std::unique_ptr<dsg_session> sp(new dsg_session());
    dsg_default_options(&sp->opt);
    if (options) sp->opt = *options;
    sp->P = prepare(mode, graph, config, nullptr, false, sp->opt.flags);
    sp->ctx = &context(sp->opt.device);
    std::lock_guard<std::mutex> lk(sp->ctx->mu);
    CK(cudaSetDevice(sp->ctx->device));
    sp->pl.pfx = "s" + std::to_string(g_session_ids.fetch_add(1)) + ".";
    sp->dg = upload_graph(*sp->ctx, sp->P, sp->pl.pfx);
    CK(cudaStreamSynchronize(sp->ctx->stream));
    status_out->t_prepare_ms = ms_since(t0);
    s = sp.release();
  });
  return s;
}

int dsg_session_run(dsg_session* s, dsg_result* result) {
  std::memset(result, 0, sizeof *result);
  return guarded(result, [&] {
    if (!s) throw Fail{DSG_INVALID, "null session"};
    std::lock_guard<std::mutex> lk(s->ctx->mu);
    CK(cudaSetDevice(s->ctx->device));
    s->ctx->h2d_bytes = 0;  // inputs are resident
    if (s->sharded) {
      // dsg_session_shard_reset ran phase 1 + the reset on every rank, and
      // the caller passed a cross-rank barrier since
      if (!s->reset_done) throw Fail{DSG_INVALID, "sharded run without dsg_session_shard_reset"};
      s->reset_done = false;
      const int64_t launches0 = dsg::g_launches.load();
      s->ctx->d2h_bytes = 0;
      cudaEvent_t ev_start;
      CK(cudaEventCreate(&ev_start));
      CK(cudaEventRecord(ev_start, s->ctx->stream));
      phase2(*s->ctx, s->P, &s->opt, s->pl, result, Clock::now());
      float ms = 0;
      cudaEventElapsedTime(&ms, ev_start, pl_ev_end(*s->ctx));
      cudaEventDestroy(ev_start);
      result->t_device_ms = ms;
      result->kernel_launches = dsg::g_launches.load() - launches0;
      result->d2h_bytes = s->ctx->d2h_bytes;
      return;
    }
    run_device(*s->ctx, s->P, s->dg, &s->opt, s->pl, result, Clock::now(), true);
  });
}

int dsg_session_shard_prepare(dsg_session* s, int32_t rank, int32_t world,
                              dsg_shard_handle* handle_out, dsg_result* status_out) {
  std::memset(status_out, 0, sizeof *status_out);
  std::memset(handle_out, 0, sizeof *handle_out);
  return guarded(status_out, [&] {
    if (!s) throw Fail{DSG_INVALID, "null session"};
    if (world < 1 || rank < 0 || rank >= world || world > DSG_MAX_SHARDS)
      throw Fail{DSG_INVALID, "bad rank / world"};
    if (s->opt.flags & DSG_FLAG_LEVEL_LAUNCH)
      throw Fail{DSG_UNSUPPORTED, "sharding needs the persistent level kernel"};
    std::lock_guard<std::mutex> lk(s->ctx->mu);
    CK(cudaSetDevice(s->ctx->device));
    s->sharded = true;  // world == 1 too: same reset / run protocol
    s->pl.rank = rank;
    s->pl.world = world;
    // placeholder peer tables (self) so phase 1 can size them
    s->pl.peer_dp.assign(world, nullptr);
    s->pl.peer_bp.assign(world, nullptr);
    s->pl.peer_done.assign(world, nullptr);
    phase1(*s->ctx, s->P, s->dg, &s->opt, s->pl);
    handle_out->rank = rank;
    handle_out->device = s->ctx->device;
    handle_out->n_ideals = s->pl.I;
    CK(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle_out->dp), s->pl.LL.dp));
    CK(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle_out->ctl), s->pl.ctl));
  });
}

int dsg_session_shard_attach(dsg_session* s, const dsg_shard_handle* all, dsg_result* status_out) {
  std::memset(status_out, 0, sizeof *status_out);
  return guarded(status_out, [&] {
    if (!s) throw Fail{DSG_INVALID, "null session"};
    std::lock_guard<std::mutex> lk(s->ctx->mu);
    CK(cudaSetDevice(s->ctx->device));
    Pipeline& pl = s->pl;
    for (int r = 0; r < pl.world; ++r) {
      if (all[r].rank != r) throw Fail{DSG_INVALID, "shard handles out of rank order"};
      if (all[r].n_ideals != pl.I) throw Fail{DSG_INVALID, "shards disagree on the lattice"};
      if (r == pl.rank) {
        pl.peer_dp[r] = pl.LL.dp;
        pl.peer_bp[r] = pl.LL.bp;
        pl.peer_done[r] = pl.PP.done;
        continue;
      }
      void *d = nullptr, *c = nullptr;
      CK(cudaIpcOpenMemHandle(&d, *reinterpret_cast<const cudaIpcMemHandle_t*>(all[r].dp),
                              cudaIpcMemLazyEnablePeerAccess));
      CK(cudaIpcOpenMemHandle(&c, *reinterpret_cast<const cudaIpcMemHandle_t*>(all[r].ctl),
                              cudaIpcMemLazyEnablePeerAccess));
      pl.ipc_opened.push_back(d);
      pl.ipc_opened.push_back(c);
      pl.peer_dp[r] = d;
      pl.peer_bp[r] = nullptr;
      pl.peer_done[r] = static_cast<unsigned*>(c) + 32;
    }
  });
}

int dsg_session_shard_reset(dsg_session* s, dsg_result* status_out) {
  std::memset(status_out, 0, sizeof *status_out);
  return guarded(status_out, [&] {
    if (!s) throw Fail{DSG_INVALID, "null session"};
    std::lock_guard<std::mutex> lk(s->ctx->mu);
    CK(cudaSetDevice(s->ctx->device));
    const void* dp0 = s->pl.LL.dp;
    cudaEvent_t ev_start;
    CK(cudaEventCreate(&ev_start));
    CK(cudaEventRecord(ev_start, s->ctx->stream));
    s->ctx->d2h_bytes = 0;
    phase1(*s->ctx, s->P, s->dg, &s->opt, s->pl);  // recomputed every solve
    if (s->pl.LL.dp != dp0) throw Fail{DSG_LOGIC, "shard tables moved; re-attach"};
    reset_tables(*s->ctx, s->P, s->pl);
    CK(cudaEventRecord(pl_ev_end(*s->ctx), s->ctx->stream));
    CK(cudaEventSynchronize(pl_ev_end(*s->ctx)));
    float ms = 0;
    cudaEventElapsedTime(&ms, ev_start, pl_ev_end(*s->ctx));
    cudaEventDestroy(ev_start);
    status_out->t_device_ms = ms;
    status_out->t_enumerate_ms = s->pl.t_enum_ms;
    status_out->t_describe_ms = s->pl.t_desc_ms;
    status_out->d2h_bytes = s->ctx->d2h_bytes;
    s->reset_done = true;
  });
}

int dsg_session_reload(dsg_session* s, const dsg_graph* graph, const dsg_config* config,
                       dsg_result* status_out) {
  std::memset(status_out, 0, sizeof *status_out);
  return guarded(status_out, [&] {
    if (!s) throw Fail{DSG_INVALID, "null session"};
    const auto t0 = Clock::now();
    Prepared P = prepare(s->P.training ? DSG_MODE_TRAINING : (s->P.repl ? DSG_MODE_REPLICATED
                                                                          : DSG_MODE_INFERENCE),
                         graph, config, nullptr, false, s->opt.flags);
    std::lock_guard<std::mutex> lk(s->ctx->mu);
    CK(cudaSetDevice(s->ctx->device));
    s->ctx->h2d_bytes = 0;
    s->P = std::move(P);
    s->dg = upload_graph(*s->ctx, s->P, s->pl.pfx);
    CK(cudaStreamSynchronize(s->ctx->stream));
    status_out->h2d_bytes = s->ctx->h2d_bytes;
    status_out->t_prepare_ms = ms_since(t0);
  });
}

void dsg_session_destroy(dsg_session* s) {
  if (!s) return;
  if (s->ctx) {
    std::lock_guard<std::mutex> lk(s->ctx->mu);
    cudaSetDevice(s->ctx->device);
    for (void* p : s->pl.ipc_opened) cudaIpcCloseMemHandle(p);
    s->ctx->release_prefix(s->pl.pfx);
  }
  delete s;
}

void dsg_default_options(dsg_options* o) {
  std::memset(o, 0, sizeof *o);
  o->ideal_budget = DSG_DEFAULT_IDEAL_BUDGET;
  o->deadline_seconds = 0;
  o->device = -1;
  o->shard_count = 0;
  o->flags = 0;
}

const char* dsg_version(void) { return "dsg_b200 1 (sm_100a)"; }

int dsg_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return c;
}

int64_t dsg_kernel_launch_count(void) { return dsg::g_launches.load(); }

int dsg_dp_solve(int32_t mode, const dsg_graph* graph, const dsg_config* config,
                 const dsg_options* options, dsg_result* result) {
  std::memset(result, 0, sizeof *result);
  try {
    solve(mode, graph, config, options, result);
    result->status = DSG_OK;
  } catch (const Fail& f) {
    result->status = f.status;
    result->budget_limit = f.limit;
    fill_msg(result->message, f.msg);
  } catch (const std::exception& e) {
    result->status = DSG_LOGIC;
    fill_msg(result->message, e.what());
  }
  return result->status;
}

void dsg_result_free(dsg_result* r) {
  if (!r) return;
  std::free(r->blocks);
  std::free(r->members);
  std::free(r->ideal_bits);
  std::free(r->dp_values);
  r->blocks = nullptr;
  r->members = nullptr;
  r->ideal_bits = nullptr;
  r->dp_values = nullptr;
}

int dsg_enumerate_ideals(const dsg_graph* graph, const uint8_t* within, int64_t budget,
                         const dsg_options* options, dsg_ideals* out) {
  std::memset(out, 0, sizeof *out);
  const auto t0 = Clock::now();
  try {
    dsg_options defaults;
    dsg_default_options(&defaults);
    const dsg_options* opt = options ? options : &defaults;
    Prepared P = prepare(DSG_MODE_INFERENCE, graph, nullptr, within, true, opt->flags);
    DeviceCtx& ctx = context(opt->device);
    std::lock_guard<std::mutex> lk(ctx.mu);
    CK(cudaSetDevice(ctx.device));
    DeviceGraph dg = upload_graph(ctx, P, "g.");
    Lattice lat = enumerate_device(ctx, P, dg, budget, (opt->flags & DSG_FLAG_HASH_ENUM) != 0, "e.");
    out->count = lat.I;
    out->words = P.W;
    out->bits = (uint64_t*)std::malloc(sizeof(uint64_t) * (size_t)lat.I * P.W + 8);
    // ctx.stream is non-blocking: a legacy-stream copy would not wait for it
    CK(cudaMemcpyAsync(out->bits, lat.sbits, sizeof(uint64_t) * (size_t)lat.I * P.W,
                       cudaMemcpyDeviceToHost, ctx.stream));
    CK(cudaStreamSynchronize(ctx.stream));
    out->n_levels = lat.n_levels;
    out->level_offsets = (int64_t*)std::malloc(sizeof(int64_t) * (lat.n_levels + 1));
    std::memcpy(out->level_offsets, lat.level_off.data(), sizeof(int64_t) * (lat.n_levels + 1));
    out->status = DSG_OK;
  } catch (const Fail& f) {
    out->status = f.status;
    out->budget_limit = f.limit;
    fill_msg(out->message, f.msg);
  } catch (const std::exception& e) {
    out->status = DSG_LOGIC;
    fill_msg(out->message, e.what());
  }
  out->t_ms = ms_since(t0);
  return out->status;
}

void dsg_ideals_free(dsg_ideals* out) {
  if (!out) return;
  std::free(out->bits);
  std::free(out->level_offsets);
  out->bits = nullptr;
  out->level_offsets = nullptr;
}

}  // extern "C"
