// transition.cu — per-level launches (DSG_FLAG_LEVEL_LAUNCH cross-check
// path), dp initialisation and the traceback.
//
// Per-level path: one transition_kernel launch per level; a CTA owns a tile
// of 128 target ideals (one per thread) and a contiguous chunk of source
// ordinals; all 32 lanes walk the same source (broadcast loads) through the
// fused scan of scan.cuh; finalize_kernel reduces the per-chunk minima and
// applies monotone_pass (dp_solver.cpp:180-193).  The default driver is the
// persistent dataflow kernel (persistent.cu); this path shares the scan but
// nothing else, so the parity tests run both.
//
// Traceback (dp_solver.cpp:332-380).  The DP kernels keep values only; the
// traceback re-derives the argmin of the ≤ K+L cells on the optimal path:
// for cell (ord, k, l), traceback_search scans every source of `ord` on the
// whole GPU and keeps the lexicographically smallest (value, src*(K+2)+code)
// — code r for an accelerator block on r replicas, K+1 for a CPU block —
// which is the reference's first-found improvement when sources are walked
// in ordinal order (dp_solver.cpp:205-230); traceback_decide then replays
// monotone_pass's strict tests to tell a block from a waste move (kinds
// 3/4) and steps to the predecessor.
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdlib>

#include "scan.cuh"

namespace dsg {

namespace {

using namespace scan;

// lattices up to this many ideal words (ideals x W) trace back in one
// single-CTA launch (C1: 0.10 -> 0.05 ms; C4's 96K words are faster on the grid)
constexpr int64_t kTracebackCtaMax = 16384;

template <typename V, int LP1, int KP1MAX, bool TRAIN>
__global__ void __launch_bounds__(kTileTargets) transition_kernel(const LevelLaunch a) {
  constexpr bool kGeneric = LP1 == 0;
  constexpr int CMAX = kGeneric ? 1 : LP1 * KP1MAX;
  constexpr int TS = kTileTargets;
  extern __shared__ __align__(16) unsigned char smem[];
  const int W = a.W, C = a.C;
  uint64_t* s_tgt = reinterpret_cast<uint64_t*>(smem);
  uint64_t* s_int = s_tgt + (size_t)a.AW * TS;  // target column padded to AW
  V* s_best = reinterpret_cast<V*>(s_int + (TRAIN ? (size_t)W * TS : 0));
  const int tid = threadIdx.x;
  const int64_t T = a.t_hi - a.t_lo;
  const Target<V> x = load_target<V, TRAIN, TS>(a, a.t_lo, a.t_hi, blockIdx.x, tid, s_tgt + tid,
                                                s_int + tid);
  V best[CMAX];
  init_cells<V, LP1, KP1MAX, TS>(C, best, s_best + tid);
  __syncwarp();
  const int64_t s0 = (int64_t)blockIdx.y * a.chunk_len;
  const int64_t s1 = min(s0 + a.chunk_len, a.s_hi);
  unsigned nested = scan_sources<V, LP1, KP1MAX, TRAIN, TS, true, TS>(
      a, x, s0, s1, 1, s_tgt + tid, s_int + tid, best, s_best + tid);
  if (x.active) {
    V* pv = (V*)a.part_val;
    const size_t base = (size_t)blockIdx.y * C;
#pragma unroll
    for (int c = 0; c < (kGeneric ? 0 : CMAX); ++c)
      if (c < C) pv[(base + c) * T + x.tl] = best[c];
    if (kGeneric)
      for (int c = 0; c < C; ++c) pv[(base + c) * T + x.tl] = s_best[c * TS + tid];
  }
  for (int off = 16; off > 0; off >>= 1) nested += __shfl_xor_sync(0xffffffffu, nested, off);
  if ((tid & 31) == 0 && nested) atomicAdd(a.pair_counter, (unsigned long long)nested);
}

template <typename V>
__global__ void finalize_kernel(const LevelLaunch a) {
  constexpr V INF = VTraits<V>::INF;
  const int64_t T = a.t_hi - a.t_lo;
  const int64_t tl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tl >= T) return;
  const int64_t t = a.t_lo + tl;
  const int C = a.C;
  V* dpt = (V*)a.dp + (size_t)t * C;
  const V* pv = (const V*)a.part_val;
  for (int c = 0; c < C; ++c) {
    V v = INF;
    for (int64_t ch = 0; ch < a.n_chunks; ++ch) v = min(v, pv[((size_t)ch * C + c) * T + tl]);
    dpt[c] = v;
  }
  monotone_strided(dpt, 1, a.K, a.L);
}

// dp[∅][0][0] = 0 followed by monotone_pass(0) (dp_solver.cpp:325-326)
template <typename V>
__global__ void init_empty_kernel(int C, V* dp) {
  for (int c = threadIdx.x; c < C; c += blockDim.x) dp[c] = 0;
}

// level of every ordinal: largest s with level_off[s] <= o
__global__ void level_of_kernel(const int64_t* __restrict__ level_off, int n_levels, int64_t I,
                                int32_t* __restrict__ level_of) {
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= I) return;
  int lo = 0, hi = n_levels - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (level_off[mid] <= o) lo = mid;
    else hi = mid - 1;
  }
  level_of[o] = lo;
}

template <typename V>
__global__ void fill_inf_kernel(V* p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = VTraits<V>::INF;
}

template <typename V>
__global__ void fill_pending_kernel(V* p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = VTraits<V>::PENDING;
}

__global__ void read_globaltimer_kernel(uint64_t* out) { *out = globaltimer(); }

__global__ void compare_tables_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                                      size_t n, int* bad) {
  bool diff = false;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    diff |= a[i] != b[i];
  if (__syncthreads_or(diff) && threadIdx.x == 0) atomicExch(bad, 1);
}

__global__ void fill_u32_kernel(unsigned* p, int64_t n, unsigned value) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = value;
}

// ---------------------------------------------------------------- traceback

// Fewest-devices cell (dp_solver.cpp:337-351); one thread.
template <typename V>
__global__ void traceback_init_kernel(int64_t I, int K, int L, const V* dp, TraceState* st,
                                      const int* abort) {
  constexpr V INF = VTraits<V>::INF;
  if (abort && (abort[0] | abort[1])) {
    // the dp pass stopped early (deadline / watchdog): the host raises it
    st->status = 3;
    st->n_blocks = 0;
    return;
  }
  const int lp1 = L + 1, C = (K + 1) * lp1;
  const V* row = dp + (size_t)(I - 1) * C;
  const V best = row[K * lp1 + L];
  st->best_value = (int64_t)best;
  st->n_blocks = 0;
  st->arrivals = 0;
  if (best == INF) {
    st->status = 2;  // infeasible
    return;
  }
  int bk = K, bl = L;
  bool found = false;
  for (int total = 0; total <= K + L && !found; ++total) {
    for (int k = max(0, total - L); k <= min(K, total); ++k) {
      const int l = total - k;
      if (row[k * lp1 + l] == best) {
        bk = k;
        bl = l;
        found = true;
        break;
      }
    }
  }
  st->best_k = bk;
  st->best_l = bl;
  st->ord = I - 1;
  st->k = bk;
  st->l = bl;
  st->status = (I - 1 == 0 && bk == 0 && bl == 0) ? 1 : 0;
}

template <typename V>
__device__ void traceback_decide(int K, int L, int W, int AW, const V* dp, const uint64_t* abits,
                                 V dv, int32_t dg, TraceState* st, int64_t* ords,
                                 int64_t* prevs, int32_t* kinds, uint64_t* block_bits);

// The direct (pre-monotone) minimum of cell (ord, k, l) and its smallest
// argmin, one partial per CTA; sources are spread over the whole grid.
template <typename V, bool TRAIN>
__global__ void __launch_bounds__(256) traceback_search_kernel(const LevelLaunch a,
                                                               TraceState* st,
                                                               const int32_t* level_of,
                                                               const int64_t* level_off,
                                                               V* part_v, int32_t* part_g,
                                                               int64_t* ords, int64_t* prevs,
                                                               int32_t* kinds,
                                                               uint64_t* block_bits,
                                                               int64_t* loads) {
  constexpr V INF = VTraits<V>::INF;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ V red_v[256];
  __shared__ int32_t red_g[256];
  if (st->status != 0) return;
  const int W = a.W, K = a.K, lp1 = a.L + 1;
  const int64_t ord = st->ord;
  const int k = st->k, l = st->l;
  uint64_t* tA = reinterpret_cast<uint64_t*>(smem);
  uint64_t* tInt = tA + W;
  for (int w = threadIdx.x; w < W; w += blockDim.x) {
    tA[w] = a.abits[(size_t)ord * a.AW + w];
    if (TRAIN) tInt[w] = a.intbits[(size_t)ord * W + w];
  }
  __syncthreads();
  const Target<V> x = target_scalars<V, TRAIN>(a, ord, 0, true);
  const int64_t S = level_off[level_of[ord]];
  const V* dp = (const V*)a.dp;
  V bv = INF;
  int32_t bg = INT_MAX;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < S;
       s += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t* sA = a.abits + (size_t)s * a.AW;
    bool nested = true;
    for (int w = 0; w < W && nested; ++w) nested = (sA[w] & ~tA[w]) == 0ull;
    if (!nested) continue;
    bool gated;
    V acc, cpu, mem_blk;
    pair_cost<V, TRAIN, 1>(a, x, s, tA, tInt, gated, acc, cpu, mem_blk);
    if (gated) continue;
    const V* sdp = dp + (size_t)s * a.C;
    const int32_t base = (int32_t)(s * (K + 2));
    if (k >= 1 && acc != INF) {
      const int rmax = a.repl ? k : 1;
      for (int rr = 1; rr <= rmax; ++rr) {
        const V load = rr == 1 ? acc : replicated<V>(a, acc, mem_blk, rr);
        vmin_arg(bv, bg, vmax(sdp[(k - rr) * lp1 + l], load), base + rr);
      }
    }
    if (l >= 1) vmin_arg(bv, bg, vmax(sdp[k * lp1 + l - 1], cpu), base + K + 1);
  }
  red_v[threadIdx.x] = bv;
  red_g[threadIdx.x] = bg;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off) {
      V v = red_v[threadIdx.x];
      int32_t g = red_g[threadIdx.x];
      vmin_arg(v, g, red_v[threadIdx.x + off], red_g[threadIdx.x + off]);
      red_v[threadIdx.x] = v;
      red_g[threadIdx.x] = g;
    }
    __syncthreads();
  }
  // the last CTA to arrive reduces the partials and takes the step
  // (threadFenceReduction pattern: no separate decide launch per step)
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    part_v[blockIdx.x] = red_v[0];
    part_g[blockIdx.x] = red_g[0];
    __threadfence();
    s_last = atomicAdd(&st->arrivals, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  bv = INF;
  bg = INT_MAX;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x)
    vmin_arg(bv, bg, __ldcg(part_v + i), __ldcg(part_g + i));
  red_v[threadIdx.x] = bv;
  red_g[threadIdx.x] = bg;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off) {
      V v = red_v[threadIdx.x];
      int32_t g = red_g[threadIdx.x];
      vmin_arg(v, g, red_v[threadIdx.x + off], red_g[threadIdx.x + off]);
      red_v[threadIdx.x] = v;
      red_g[threadIdx.x] = g;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    st->arrivals = 0;
    const int nb = st->n_blocks;
    traceback_decide<V>(a.K, a.L, a.W, a.AW, dp, a.abits, red_v[0], red_g[0], st, ords, prevs,
                        kinds, block_bits);
    if (st->n_blocks > nb) {
      // the block's per-device load, recomputed from the closed forms (what
      // make_canonical_split reports, graph.cpp:573-621)
      bool gated;
      V acc, cpu, mem_blk;
      pair_cost<V, TRAIN, 1>(a, x, prevs[nb], tA, tInt, gated, acc, cpu, mem_blk);
      const int kind = kinds[nb];
      V load = (kind & 1) ? cpu : acc;
      if (!(kind & 1) && (kind >> 1) > 1 && acc != INF) load = replicated<V>(a, acc, mem_blk, kind >> 1);
      loads[nb] = load == INF ? INT64_MAX : (int64_t)load;
    }
  }
}

// Replay monotone_pass's strict tests for cell (ord, k, l) given its direct
// minimum (dv, argmin dg), and step.  Run by one thread of the last search CTA.
template <typename V>
__device__ void traceback_decide(int K, int L, int W, int AW, const V* dp, const uint64_t* abits,
                                 V dv, int32_t dg, TraceState* st, int64_t* ords,
                                 int64_t* prevs, int32_t* kinds, uint64_t* block_bits) {
  constexpr V INF = VTraits<V>::INF;
  const int lp1 = L + 1, C = (K + 1) * lp1;
  const int64_t ord = st->ord;
  int k = st->k, l = st->l;
  const V* row = dp + (size_t)ord * C;
  const int c = k * lp1 + l;
  V w = dv;
  int kind = 0;  // 0 block, 3 waste accelerator, 4 waste CPU
  if (k > 0 && row[c - lp1] < w) {
    w = row[c - lp1];
    kind = 3;
  }
  if (l > 0 && row[c - 1] < w) {
    w = row[c - 1];
    kind = 4;
  }
  if (w != row[c] || w == INF) {
    st->status = 3;  // dp reconstruction stuck (dp_solver.cpp:357)
    return;
  }
  int64_t next = ord;
  if (kind == 3) {
    --k;
  } else if (kind == 4) {
    --l;
  } else {
    const int64_t prev = dg / (K + 2);
    const int code = dg % (K + 2);
    const int cpu = code == K + 1;
    const int repl = cpu ? 1 : code;
    const int nb = st->n_blocks;
    ords[nb] = ord;
    prevs[nb] = prev;
    kinds[nb] = cpu | (repl << 1);
    for (int x = 0; x < W; ++x)
      block_bits[(size_t)nb * W + x] = abits[(size_t)ord * AW + x] & ~abits[(size_t)prev * AW + x];
    st->n_blocks = nb + 1;
    if (cpu) --l;
    else k -= repl;
    next = prev;
  }
  st->ord = next;
  st->k = k;
  st->l = l;
  if (next == 0 && k == 0 && l == 0) st->status = 1;
}

// Small lattices: every traceback step in ONE single-CTA launch (no launch
// and grid-reduction round trip per step): the CTA scans the current
// target's sources, reduces to the smallest (value, argmin), and thread 0
// takes the step and recomputes the block's load, then the next step.
template <typename V, bool TRAIN>
__global__ void __launch_bounds__(1024) traceback_cta_kernel(const LevelLaunch a, TraceState* st,
                                                             const int32_t* level_of,
                                                             const int64_t* level_off,
                                                             int64_t* ords, int64_t* prevs,
                                                             int32_t* kinds, uint64_t* block_bits,
                                                             int64_t* loads) {
  constexpr V INF = VTraits<V>::INF;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ V red_v[32];
  __shared__ int32_t red_g[32];
  uint64_t* tA = reinterpret_cast<uint64_t*>(smem);
  uint64_t* tInt = tA + a.W;
  const int W = a.W, K = a.K, lp1 = a.L + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  while (true) {
    __syncthreads();
    if (st->status != 0) return;
    const int64_t ord = st->ord;
    const int k = st->k, l = st->l;
    for (int w = threadIdx.x; w < W; w += blockDim.x) {
      tA[w] = a.abits[(size_t)ord * a.AW + w];
      if (TRAIN) tInt[w] = a.intbits[(size_t)ord * W + w];
    }
    __syncthreads();
    const Target<V> x = target_scalars<V, TRAIN>(a, ord, 0, true);
    const int64_t S = level_off[level_of[ord]];
    const V* dp = (const V*)a.dp;
    V bv = INF;
    int32_t bg = INT_MAX;
    for (int64_t s = threadIdx.x; s < S; s += blockDim.x) {
      const uint64_t* sA = a.abits + (size_t)s * a.AW;
      bool nested = true;
      for (int w = 0; w < W && nested; ++w) nested = (sA[w] & ~tA[w]) == 0ull;
      if (!nested) continue;
      bool gated;
      V acc, cpu, mem_blk;
      pair_cost<V, TRAIN, 1>(a, x, s, tA, tInt, gated, acc, cpu, mem_blk);
      if (gated) continue;
      const V* sdp = dp + (size_t)s * a.C;
      const int32_t base = (int32_t)(s * (K + 2));
      if (k >= 1 && acc != INF) {
        const int rmax = a.repl ? k : 1;
        for (int rr = 1; rr <= rmax; ++rr) {
          const V load = rr == 1 ? acc : replicated<V>(a, acc, mem_blk, rr);
          vmin_arg(bv, bg, vmax(sdp[(k - rr) * lp1 + l], load), base + rr);
        }
      }
      if (l >= 1) vmin_arg(bv, bg, vmax(sdp[k * lp1 + l - 1], cpu), base + K + 1);
    }
    for (int off = 16; off > 0; off >>= 1) {
      const V v2 = __shfl_xor_sync(0xffffffffu, bv, off);
      const int32_t g2 = __shfl_xor_sync(0xffffffffu, bg, off);
      vmin_arg(bv, bg, v2, g2);
    }
    if (lane == 0) {
      red_v[warp] = bv;
      red_g[warp] = bg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < nw; ++w) vmin_arg(bv, bg, red_v[w], red_g[w]);
      const int nb = st->n_blocks;
      traceback_decide<V>(a.K, a.L, a.W, a.AW, dp, a.abits, bv, bg, st, ords, prevs, kinds,
                          block_bits);
      if (st->n_blocks > nb) {
        bool gated;
        V acc, cpu, mem_blk;
        pair_cost<V, TRAIN, 1>(a, x, prevs[nb], tA, tInt, gated, acc, cpu, mem_blk);
        const int kind = kinds[nb];
        V load = (kind & 1) ? cpu : acc;
        if (!(kind & 1) && (kind >> 1) > 1 && acc != INF) load = replicated<V>(a, acc, mem_blk, kind >> 1);
        loads[nb] = load == INF ? INT64_MAX : (int64_t)load;
      }
    }
  }
}

template <typename V, int LP1, int KP1MAX, bool TRAIN>
void launch_tile(const LevelLaunch& L, dim3 grid, cudaStream_t st) {
  size_t smem = (size_t)(L.AW + (TRAIN ? L.W : 0)) * kTileTargets * sizeof(uint64_t);
  if (LP1 == 0) smem += (size_t)L.C * kTileTargets * sizeof(V);
  auto kern = transition_kernel<V, LP1, KP1MAX, TRAIN>;
  // per device context: set on every launch (a second device needs it too)
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, kTileTargets, smem, st>>>(L);
}

template <typename V, bool TRAIN>
void dispatch_tile(const LevelLaunch& L, dim3 grid, cudaStream_t st) {
  const int lp1 = L.L + 1, kp1 = L.K + 1;
  // replication and unprunable weights: generic cells (no pruning)
  if (L.repl || L.no_prune) return launch_tile<V, 0, 0, TRAIN>(L, grid, st);
  if (lp1 == 1 && kp1 <= 9) return launch_tile<V, 1, 9, TRAIN>(L, grid, st);
  if (lp1 == 1 && kp1 <= 17) return launch_tile<V, 1, 17, TRAIN>(L, grid, st);
  if (lp1 == 2 && kp1 <= 9) return launch_tile<V, 2, 9, TRAIN>(L, grid, st);
  if (lp1 == 3 && kp1 <= 9) return launch_tile<V, 3, 9, TRAIN>(L, grid, st);
  if (lp1 == 5 && kp1 <= 9) return launch_tile<V, 5, 9, TRAIN>(L, grid, st);
  return launch_tile<V, 0, 0, TRAIN>(L, grid, st);
}

template <typename V>
void traceback_t(const LevelLaunch& L, const int32_t* level_of, const int64_t* level_off,
                 int64_t I, int sm_count, TraceBuffers& b, cudaStream_t st) {
  traceback_init_kernel<V><<<1, 1, 0, st>>>(I, L.K, L.L, (const V*)L.dp, b.state, b.abort);
  count_launch();
  const int grid = b.n_parts;
  const size_t smem = (size_t)L.W * sizeof(uint64_t) * 2;
  static const int64_t cta_max = [] {
    const char* e = std::getenv("DSG_TB_CTA_MAX");
    return e ? (int64_t)std::atoll(e) : kTracebackCtaMax;
  }();
  if (I * L.W <= cta_max) {
    if (L.training)
      traceback_cta_kernel<V, true><<<1, 1024, smem, st>>>(L, b.state, level_of, level_off, b.ords,
                                                           b.prevs, b.kinds, b.block_bits, b.loads);
    else
      traceback_cta_kernel<V, false><<<1, 1024, smem, st>>>(L, b.state, level_of, level_off, b.ords,
                                                            b.prevs, b.kinds, b.block_bits, b.loads);
    count_launch();
    return;
  }
  for (int step = 0; step <= L.K + L.L; ++step) {
    if (L.training)
      traceback_search_kernel<V, true><<<grid, 256, smem, st>>>(
          L, b.state, level_of, level_off, (V*)b.part_v, b.part_g, b.ords, b.prevs, b.kinds,
          b.block_bits, b.loads);
    else
      traceback_search_kernel<V, false><<<grid, 256, smem, st>>>(
          L, b.state, level_of, level_off, (V*)b.part_v, b.part_g, b.ords, b.prevs, b.kinds,
          b.block_bits, b.loads);
    count_launch();
  }
  (void)sm_count;
}

}  // namespace

void launch_transition(const LevelLaunch& L, cudaStream_t st) {
  const int64_t T = L.t_hi - L.t_lo;
  dim3 grid((unsigned)((T + kTileTargets - 1) / kTileTargets), (unsigned)L.n_chunks, 1);
  if (L.value_bits == 32) {
    if (L.training) dispatch_tile<int32_t, true>(L, grid, st);
    else dispatch_tile<int32_t, false>(L, grid, st);
  } else {
    if (L.training) dispatch_tile<int64_t, true>(L, grid, st);
    else dispatch_tile<int64_t, false>(L, grid, st);
  }
  count_launch();
}

void launch_finalize(const LevelLaunch& L, cudaStream_t st) {
  const int64_t T = L.t_hi - L.t_lo;
  const int threads = 128;
  const unsigned blocks = (unsigned)((T + threads - 1) / threads);
  if (L.value_bits == 32) finalize_kernel<int32_t><<<blocks, threads, 0, st>>>(L);
  else finalize_kernel<int64_t><<<blocks, threads, 0, st>>>(L);
  count_launch();
}

void launch_init_empty(int value_bits, int K, int L, void* dp, cudaStream_t st) {
  const int C = (K + 1) * (L + 1);
  if (value_bits == 32) init_empty_kernel<int32_t><<<1, 128, 0, st>>>(C, (int32_t*)dp);
  else init_empty_kernel<int64_t><<<1, 128, 0, st>>>(C, (int64_t*)dp);
  count_launch();
}

void launch_fill_pending(int value_bits, void* p, int64_t n, cudaStream_t st) {
  const int blocks = (int)std::min<int64_t>(1024, (n + 255) / 256 + 1);
  if (value_bits == 32) fill_pending_kernel<int32_t><<<blocks, 256, 0, st>>>((int32_t*)p, n);
  else fill_pending_kernel<int64_t><<<blocks, 256, 0, st>>>((int64_t*)p, n);
  count_launch();
}

void launch_fill_inf(int value_bits, void* p, int64_t n, cudaStream_t st) {
  const int blocks = (int)std::min<int64_t>(1024, (n + 255) / 256 + 1);
  if (value_bits == 32) fill_inf_kernel<int32_t><<<blocks, 256, 0, st>>>((int32_t*)p, n);
  else fill_inf_kernel<int64_t><<<blocks, 256, 0, st>>>((int64_t*)p, n);
  count_launch();
}

void launch_level_of(const int64_t* level_off, int n_levels, int64_t I, int32_t* level_of,
                     cudaStream_t st) {
  if (I <= 0) return;
  level_of_kernel<<<(unsigned)((I + 255) / 256), 256, 0, st>>>(level_off, n_levels, I, level_of);
  count_launch();
}

void launch_fill_u32(unsigned* p, int64_t n, unsigned value, cudaStream_t st) {
  fill_u32_kernel<<<1, 256, 0, st>>>(p, n, value);
  count_launch();
}

void launch_compare_tables(const void* a, const void* b, size_t bytes, int* bad, cudaStream_t st) {
  const size_t n = bytes / 4;  // tables are whole int32 / int64 rows
  const unsigned blocks = (unsigned)std::min<size_t>(1024, (n + 255) / 256 + 1);
  compare_tables_kernel<<<blocks, 256, 0, st>>>((const uint32_t*)a, (const uint32_t*)b, n, bad);
  count_launch();
}

void launch_read_globaltimer(uint64_t* out, cudaStream_t st) {
  read_globaltimer_kernel<<<1, 1, 0, st>>>(out);
  count_launch();
}

void launch_traceback(const LevelLaunch& L, const int32_t* level_of, const int64_t* level_off,
                      int64_t I, int sm_count, TraceBuffers& b, cudaStream_t st) {
  if (L.value_bits == 32) traceback_t<int32_t>(L, level_of, level_off, I, sm_count, b, st);
  else traceback_t<int64_t>(L, level_of, level_off, I, sm_count, b, st);
}

}  // namespace dsg
