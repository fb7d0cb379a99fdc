// transition.cu — per-level launches (DSG_FLAG_LEVEL_LAUNCH cross-check
// path), dp initialisation and traceback.
//
// One transition_kernel launch per level: a CTA owns a tile of 128 target
// ideals (one per thread) and a contiguous chunk of source ordinals; all
// 32 lanes walk the same source (broadcast loads) through the fused scan of
// scan.cuh; per-chunk (value, arg) partials are reduced in chunk order by
// finalize_kernel, which then applies monotone_pass (dp_solver.cpp:180-193).
// The default driver is the persistent cooperative kernel (persistent.cu);
// this path shares the scan but nothing else, so the parity tests run both.
#include <climits>
#include <cstdint>

#include "scan.cuh"

namespace dsg {

namespace {

using namespace scan;

template <typename V, int LP1, int KP1MAX, bool TRAIN>
__global__ void __launch_bounds__(kTileTargets) transition_kernel(const LevelLaunch a) {
  constexpr bool kGeneric = LP1 == 0;
  constexpr int CMAX = kGeneric ? 1 : LP1 * KP1MAX;
  constexpr int TS = kTileTargets;
  extern __shared__ __align__(16) unsigned char smem[];
  const int W = a.W, C = a.C;
  uint64_t* s_tgt = reinterpret_cast<uint64_t*>(smem);
  uint64_t* s_int = s_tgt + (size_t)W * TS;
  V* s_best = reinterpret_cast<V*>(s_int + (TRAIN ? (size_t)W * TS : 0));
  int32_t* s_arg = reinterpret_cast<int32_t*>(s_best + (kGeneric ? (size_t)C * TS : 0));
  const int tid = threadIdx.x;
  const int64_t T = a.t_hi - a.t_lo;
  const Target<V> x = load_target<V, TRAIN, TS>(a, a.t_lo, a.t_hi, blockIdx.x, tid, s_tgt + tid,
                                                s_int + tid);
  V best[CMAX];
  int32_t barg[CMAX];
  init_cells<V, LP1, KP1MAX, TS>(C, best, barg, s_best + tid, s_arg + tid);
  __syncwarp();
  const int64_t s0 = (int64_t)blockIdx.y * a.chunk_len;
  const int64_t s1 = min(s0 + a.chunk_len, a.s_hi);
  unsigned nested = scan_sources<V, LP1, KP1MAX, TRAIN, TS, true, TS>(
      a, x, s0, s1, 1, s_tgt + tid, s_int + tid, best, barg, s_best + tid, s_arg + tid);
  if (x.active) {
    V* pv = (V*)a.part_val;
    const size_t base = (size_t)blockIdx.y * C;
#pragma unroll
    for (int c = 0; c < (kGeneric ? 0 : CMAX); ++c) {
      if (c < C) {
        pv[(base + c) * T + x.tl] = best[c];
        a.part_arg[(base + c) * T + x.tl] = barg[c];
      }
    }
    if (kGeneric) {
      for (int c = 0; c < C; ++c) {
        pv[(base + c) * T + x.tl] = s_best[c * TS + tid];
        a.part_arg[(base + c) * T + x.tl] = s_arg[c * TS + tid];
      }
    }
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
  int32_t* bpt = a.bp + (size_t)t * C;
  const V* pv = (const V*)a.part_val;
  for (int c = 0; c < C; ++c) {
    V v = INF;
    int32_t g = INT_MAX;
    for (int64_t ch = 0; ch < a.n_chunks; ++ch) {
      const size_t i = ((size_t)ch * C + c) * T + tl;
      vmin_arg(v, g, pv[i], a.part_arg[i]);
    }
    dpt[c] = v;
    bpt[c] = v == INF ? -1 : g;
  }
  monotone_strided(dpt, bpt, 1, a.K, a.L);
}

// dp[∅][0][0] = 0 followed by monotone_pass(0) (dp_solver.cpp:325-326)
template <typename V>
__global__ void init_empty_kernel(int K, int L, V* dp, int32_t* bp) {
  const int C = (K + 1) * (L + 1);
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const int k = c / (L + 1), l = c % (L + 1);
    dp[c] = 0;
    bp[c] = (k == 0 && l == 0) ? -1 : (k > 0 ? -3 : -4);
  }
}

__global__ void read_globaltimer_kernel(uint64_t* out) { *out = globaltimer(); }

__global__ void fill_u32_kernel(unsigned* p, int64_t n, unsigned value) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = value;
}

// Fewest-devices cell + argmin walk (dp_solver.cpp:332-380); one thread.
template <typename V>
__global__ void traceback_kernel(int64_t I, int K, int L, int W, const V* dp, const int32_t* bp,
                                 const uint64_t* abits, TracebackOut* out, int64_t* ords,
                                 int64_t* prevs, int32_t* cpus, uint64_t* block_bits) {
  constexpr V INF = VTraits<V>::INF;
  const int lp1 = L + 1, C = (K + 1) * lp1;
  const int64_t full = I - 1;
  const V* row = dp + (size_t)full * C;
  const V best = row[K * lp1 + L];
  out->best_value = (int64_t)best;
  out->n_blocks = 0;
  if (best == INF) {
    out->status = 1;
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
  out->best_k = bk;
  out->best_l = bl;
  int64_t ord = full;
  int k = bk, l = bl, nb = 0;
  int guard = 2 * (K + L) + 2;
  while (!(ord == 0 && k == 0 && l == 0)) {
    if (--guard < 0 || k < 0 || l < 0) {
      out->status = 2;
      return;
    }
    const int32_t b = bp[(size_t)ord * C + k * lp1 + l];
    if (b == -1 || b < -4) {
      out->status = 2;
      return;
    }
    if (b == -3) {
      --k;
      continue;
    }
    if (b == -4) {
      --l;
      continue;
    }
    // arg = prev*(K+2) + r (accelerator block on r replicas) or + K+1 (CPU)
    const int64_t prev = (int64_t)(b / (K + 2));
    const int code = b % (K + 2);
    const int cpu = code == K + 1;
    const int repl = cpu ? 1 : code;
    if ((!cpu && repl > k) || prev >= ord) {
      out->status = 2;
      return;
    }
    ords[nb] = ord;
    prevs[nb] = prev;
    cpus[nb] = cpu | (repl << 1);
    for (int w = 0; w < W; ++w)
      block_bits[(size_t)nb * W + w] = abits[(size_t)ord * W + w] & ~abits[(size_t)prev * W + w];
    ++nb;
    if (cpu) --l;
    else k -= repl;
    ord = prev;
  }
  out->n_blocks = nb;
  out->status = 0;
}

template <typename V, int LP1, int KP1MAX, bool TRAIN>
void launch_tile(const LevelLaunch& L, dim3 grid, cudaStream_t st) {
  size_t smem = (size_t)L.W * kTileTargets * sizeof(uint64_t) * (TRAIN ? 2 : 1);
  if (LP1 == 0) smem += (size_t)L.C * kTileTargets * (sizeof(V) + sizeof(int32_t));
  auto kern = transition_kernel<V, LP1, KP1MAX, TRAIN>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  kern<<<grid, kTileTargets, smem, st>>>(L);
}

template <typename V, bool TRAIN>
void dispatch_tile(const LevelLaunch& L, dim3 grid, cudaStream_t st) {
  const int lp1 = L.L + 1, kp1 = L.K + 1;
  if (L.repl) return launch_tile<V, 0, 0, TRAIN>(L, grid, st);  // replication: generic cells
  if (lp1 == 1 && kp1 <= 9) return launch_tile<V, 1, 9, TRAIN>(L, grid, st);
  if (lp1 == 1 && kp1 <= 17) return launch_tile<V, 1, 17, TRAIN>(L, grid, st);
  if (lp1 == 2 && kp1 <= 9) return launch_tile<V, 2, 9, TRAIN>(L, grid, st);
  if (lp1 == 3 && kp1 <= 9) return launch_tile<V, 3, 9, TRAIN>(L, grid, st);
  if (lp1 == 5 && kp1 <= 9 && sizeof(V) == 4) return launch_tile<V, 5, 9, TRAIN>(L, grid, st);
  return launch_tile<V, 0, 0, TRAIN>(L, grid, st);
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

void launch_init_empty(int value_bits, int K, int L, void* dp, int32_t* bp, cudaStream_t st) {
  if (value_bits == 32) init_empty_kernel<int32_t><<<1, 128, 0, st>>>(K, L, (int32_t*)dp, bp);
  else init_empty_kernel<int64_t><<<1, 128, 0, st>>>(K, L, (int64_t*)dp, bp);
  count_launch();
}

void launch_fill_u32(unsigned* p, int64_t n, unsigned value, cudaStream_t st) {
  fill_u32_kernel<<<1, 256, 0, st>>>(p, n, value);
  count_launch();
}

void launch_read_globaltimer(uint64_t* out, cudaStream_t st) {
  read_globaltimer_kernel<<<1, 1, 0, st>>>(out);
  count_launch();
}

void launch_traceback(int value_bits, int64_t I, int K, int L, int W, const void* dp,
                      const int32_t* bp, const uint64_t* abits, TracebackOut* out,
                      int64_t* ords, int64_t* prevs, int32_t* cpus, uint64_t* block_bits,
                      cudaStream_t st) {
  if (value_bits == 32)
    traceback_kernel<int32_t><<<1, 1, 0, st>>>(I, K, L, W, (const int32_t*)dp, bp, abits, out, ords,
                                               prevs, cpus, block_bits);
  else
    traceback_kernel<int64_t><<<1, 1, 0, st>>>(I, K, L, W, (const int64_t*)dp, bp, abits, out, ords,
                                               prevs, cpus, block_bits);
  count_launch();
}

}  // namespace dsg
