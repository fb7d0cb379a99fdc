// transition.cu — K2+K3+K4: the fused max-load DP transition for one level.
//
// Replaces the reference's per-target DFS over sub-ideals
// (walk_subideals + apply_candidate, /root/reference/proj/src/dp_solver.cpp:
// 197-317) with a dense, level-synchronous tiling that needs no hash lookups
// and no allocation:
//
//   * every thread OWNS one target ideal I of level s (128 targets per CTA)
//     and keeps its (K+1)(L+1) running (min, argmin) cells in registers;
//   * blockIdx.y selects a contiguous chunk of source ordinals [0, start_s);
//     all 32 lanes walk the SAME source at the same time, so every source
//     read (bitset, prefix sums, frontier table, dp row) is one broadcast
//     load, and the per-source frontier loop is warp-uniform;
//   * K2 (pair enumeration): I' ⊆ I is a W-word AND-NOT test against the
//     target bitset held in shared memory;
//   * K3 (block cost): prefix differences + the source-frontier walk of
//     describe.cu (two 64-bit masks per chunk of <= 64 producers);
//   * K4 (min-max): for each cell, max(dp[I'][k-1][l], acc) and
//     max(dp[I'][k][l-1], cpu) with a strict-< update; the argmin is
//     2*I' + (cpu block), so "smallest (value, arg)" is a total order and the
//     result is independent of how sources are chunked across CTAs/GPUs.
//
// Partial (value, arg) per chunk go to part_*; the finalize kernel reduces
// them in chunk order and applies monotone_pass (dp_solver.cpp:180-193).
#include <climits>
#include <cstdint>

#include "dsg_device.cuh"
#include "dsg_internal.h"

namespace dsg {

namespace {

template <typename V>
__device__ __forceinline__ V vmax(V a, V b) {
  return a > b ? a : b;
}

// combine_interleaving, graph.cpp:457-467
template <typename V>
__device__ __forceinline__ V combine(V in, V proc, V out, int mode) {
  if (mode == 0) return in + proc + out;
  if (mode == 1) return vmax(proc, (V)(in + out));
  return vmax(proc, vmax(in, out));
}

// General backward-contiguity gate (is_contiguous over reachability_within
// of the backward part, graph.cpp:349-363), used when the fast up-set test
// does not apply.
__device__ bool bw_contiguous(const LevelLaunch& a, const uint64_t* __restrict__ tA,
                              const uint64_t* __restrict__ sA) {
  const int W = a.W;
  uint64_t rf[kMaxWords], rt[kMaxWords], B[kMaxWords];
  bool any = false;
  for (int w = 0; w < W; ++w) {
    B[w] = tA[w * kTileTargets] & ~sA[w] & a.bwset[w];
    rf[w] = 0;
    rt[w] = 0;
    any |= B[w] != 0;
  }
  if (!any) return true;
  for (int w = 0; w < W; ++w) {
    uint64_t x = B[w];
    while (x) {
      int b = __ffsll((long long)x) - 1;
      x &= x - 1;
      int u = (w << 6) | b;
      const uint64_t* f = a.bw_from + (size_t)u * W;
      const uint64_t* t = a.bw_to + (size_t)u * W;
      for (int k = 0; k < W; ++k) {
        rf[k] |= f[k];
        rt[k] |= t[k];
      }
    }
  }
  for (int w = 0; w < W; ++w)
    if (rf[w] & rt[w] & ~B[w]) return false;
  return true;
}

// Block cost of B = A(t) \ A(s) on an accelerator (BlockTracker::acc_load,
// dp_solver.cpp:90-97) given the prefix differences; INF when infeasible.
template <typename V, bool TRAIN>
__device__ __forceinline__ V acc_block_cost(const LevelLaunch& a, int64_t s, V proc, V tfw,
                                            int tfwi, const uint64_t* __restrict__ tA,
                                            const uint64_t* __restrict__ tInt, int64_t tl_lo,
                                            int64_t tl_hi) {
  constexpr V INF = VTraits<V>::INF;
  const FChunk* __restrict__ chunks = a.chunks;
  const NItem* __restrict__ nitems = a.nitems;
  const V* __restrict__ fpool = (const V*)a.fpool;
  V cin = 0, csub = 0;
  bool cin_inf = false;
  int cout_inf = tfwi;
  const int64_t c0 = __ldg(a.chunk_off + s), c1 = __ldg(a.chunk_off + s + 1);
  for (int64_t c = c0; c < c1; ++c) {
    const int n_n = __ldg(&chunks[c].n_n);
    const int n_f = __ldg(&chunks[c].n_f);
    const int off_n = __ldg(&chunks[c].off_n);
    const int off_f = __ldg(&chunks[c].off_f);
    const uint64_t infm = __ldg(&chunks[c].infmask);
    uint64_t hit = 0, miss = 0;
    for (int i = 0; i < n_n; ++i) {
      const uint32_t word = __ldg(&nitems[off_n + i].word);
      const uint32_t bit = __ldg(&nitems[off_n + i].bit);
      const uint64_t pm = __ldg(&nitems[off_n + i].predmask);
      const bool in = (tA[word * kTileTargets] >> bit) & 1ull;
      hit |= in ? pm : 0ull;
      miss |= in ? 0ull : pm;
    }
    for (int j = 0; j < n_f; ++j) {
      const V w = __ldg(fpool + off_f + j);
      cin += ((hit >> j) & 1ull) ? w : (V)0;
      csub += ((miss >> j) & 1ull) ? w : (V)0;
    }
    cin_inf |= (hit & infm) != 0ull;
    cout_inf -= __popcll(miss & infm);
  }
  V cout = tfw - csub;
  if (TRAIN) {
    // comm_out += W(P'(A') ∩ Int(A))  (source side, warp-uniform)
    const int64_t p0 = __ldg(a.p_off + s), p1 = __ldg(a.p_off + s + 1);
    for (int64_t p = p0; p < p1; ++p) {
      const PItem* pi = a.pitems + p;
      const uint32_t word = __ldg(&pi->word), bit = __ldg(&pi->bit);
      const bool in = (tInt[word * kTileTargets] >> bit) & 1ull;
      cout += in ? (V)__ldg(&pi->weight) : (V)0;
      cout_inf += (in && __ldg(&pi->inf)) ? 1 : 0;
    }
    // comm_in += W({u in L(A) : succ(u) ∩ A ⊄ A'})  (target side)
    const uint64_t* sA = a.abits + (size_t)s * a.W;
    for (int64_t e = tl_lo; e < tl_hi; ++e) {
      const LEntry le = a.lentries[e];
      bool charged = false;
      for (int i = 0; i < le.n_items; ++i) {
        const MaskItem mi = a.litems[le.off_items + i];
        charged |= (mi.mask & ~__ldg(sA + mi.word)) != 0ull;
      }
      cin += charged ? (V)le.weight : (V)0;
      cin_inf |= charged && le.inf;
    }
  }
  if (cin_inf || cout_inf > 0) return INF;
  return combine<V>(cin, proc, cout, a.interleave);
}

template <typename V, int LP1, int KP1MAX, bool TRAIN>
__global__ void __launch_bounds__(kTileTargets) transition_kernel(const LevelLaunch a) {
  constexpr V INF = VTraits<V>::INF;
  constexpr bool kGeneric = LP1 == 0;
  constexpr int CMAX = kGeneric ? 1 : LP1 * KP1MAX;
  extern __shared__ __align__(16) unsigned char smem[];
  const int W = a.W;
  const int C = a.C;
  uint64_t* s_tgt = reinterpret_cast<uint64_t*>(smem);
  uint64_t* s_int = s_tgt + (size_t)W * kTileTargets;
  V* s_best = reinterpret_cast<V*>(s_int + (TRAIN ? (size_t)W * kTileTargets : 0));
  int32_t* s_arg = reinterpret_cast<int32_t*>(s_best + (kGeneric ? (size_t)C * kTileTargets : 0));

  const int tid = threadIdx.x;
  const int64_t T = a.t_hi - a.t_lo;
  const int64_t tl = (int64_t)blockIdx.x * kTileTargets + tid;
  const bool active = tl < T;
  const int64_t t = a.t_lo + (active ? tl : 0);

  for (int w = 0; w < W; ++w) {
    s_tgt[w * kTileTargets + tid] = active ? a.abits[(size_t)t * W + w] : 0ull;
    if (TRAIN) s_int[w * kTileTargets + tid] = active ? a.intbits[(size_t)t * W + w] : 0ull;
  }
  const uint64_t* tA = s_tgt + tid;
  const uint64_t* tInt = s_int + tid;
  const V tcpu = ((const V*)a.pfx_cpu)[t];
  const V tacc = ((const V*)a.pfx_acc)[t];
  const V tmem = ((const V*)a.pfx_mem)[t];
  const V tfw = ((const V*)a.fw)[t];
  const int tun = a.unsup[t];
  const int tfwi = a.fwinf[t];
  const bool tup = TRAIN ? (a.upset[t] != 0) : true;
  const int64_t tl_lo = TRAIN ? a.l_off[t] : 0;
  const int64_t tl_hi = TRAIN ? a.l_off[t + 1] : 0;
  const V mlim = (V)a.mlim;

  V best[CMAX];
  int32_t barg[CMAX];
#pragma unroll
  for (int c = 0; c < CMAX; ++c) {
    best[c] = INF;
    barg[c] = INT_MAX;
  }
  if (kGeneric) {
    for (int c = 0; c < C; ++c) {
      s_best[c * kTileTargets + tid] = INF;
      s_arg[c * kTileTargets + tid] = INT_MAX;
    }
  }
  __syncwarp();

  const int64_t s0 = (int64_t)blockIdx.y * a.chunk_len;
  const int64_t s1 = min(s0 + a.chunk_len, a.s_hi);
  const V* __restrict__ pcpu = (const V*)a.pfx_cpu;
  const V* __restrict__ pacc = (const V*)a.pfx_acc;
  const V* __restrict__ pmem = (const V*)a.pfx_mem;
  const V* __restrict__ dp = (const V*)a.dp;
  unsigned nested_cnt = 0;

  for (int64_t s = s0; s < s1; ++s) {
    // K2: I' ⊆ I
    const uint64_t* __restrict__ sA = a.abits + (size_t)s * W;
    bool nested = active;
    for (int w = 0; w < W; ++w) nested &= (__ldg(sA + w) & ~tA[w * kTileTargets]) == 0ull;
    if (!__any_sync(0xffffffffu, nested)) continue;
    if (nested) {
      ++nested_cnt;
      bool gate = true;
      if (TRAIN && a.has_bw) {
        if (!(a.fastgate && tup && __ldg(a.upset + s))) gate = bw_contiguous(a, tA, sA);
      }
      if (gate) {
        // K3: block cost
        const V cpu = tcpu - __ldg(pcpu + s);
        V acc = INF;
        bool acc_ok = a.K > 0 && (tun - __ldg(a.unsup + s)) == 0;
        if (acc_ok && a.memcheck) acc_ok = !((V)(tmem - __ldg(pmem + s)) > mlim);
        if (acc_ok)
          acc = acc_block_cost<V, TRAIN>(a, s, (V)(tacc - __ldg(pacc + s)), tfw, tfwi, tA, tInt,
                                         tl_lo, tl_hi);
        // K4: min-max update, strict < keeps the smallest argmin
        const V* __restrict__ sdp = dp + (size_t)s * C;
        const int32_t aa = (int32_t)(2 * s), ac = aa + 1;
        if (!kGeneric) {
#pragma unroll
          for (int c = 0; c < CMAX; ++c) {
            const int k = kGeneric ? 0 : c / (LP1 ? LP1 : 1);
            const int l = kGeneric ? 0 : c % (LP1 ? LP1 : 1);
            if (c < C) {
              if (k >= 1) {
                const V v = vmax(__ldg(sdp + c - LP1), acc);
                if (v < best[c]) {
                  best[c] = v;
                  barg[c] = aa;
                }
              }
              if (l >= 1) {
                const V v = vmax(__ldg(sdp + c - 1), cpu);
                if (v < best[c]) {
                  best[c] = v;
                  barg[c] = ac;
                }
              }
            }
          }
        } else {
          const int lp1 = a.L + 1;
          for (int k = 0; k <= a.K; ++k) {
            for (int l = 0; l <= a.L; ++l) {
              const int c = k * lp1 + l;
              V b = s_best[c * kTileTargets + tid];
              int32_t g = s_arg[c * kTileTargets + tid];
              if (k >= 1) {
                const V v = vmax(__ldg(sdp + c - lp1), acc);
                if (v < b) {
                  b = v;
                  g = aa;
                }
              }
              if (l >= 1) {
                const V v = vmax(__ldg(sdp + c - 1), cpu);
                if (v < b) {
                  b = v;
                  g = ac;
                }
              }
              s_best[c * kTileTargets + tid] = b;
              s_arg[c * kTileTargets + tid] = g;
            }
          }
        }
      }
    }
  }

  if (active) {
    V* pv = (V*)a.part_val;
    const size_t base = (size_t)blockIdx.y * C;
    if (!kGeneric) {
#pragma unroll
      for (int c = 0; c < CMAX; ++c) {
        if (c < C) {
          pv[(base + c) * T + tl] = best[c];
          a.part_arg[(base + c) * T + tl] = barg[c];
        }
      }
    } else {
      for (int c = 0; c < C; ++c) {
        pv[(base + c) * T + tl] = s_best[c * kTileTargets + tid];
        a.part_arg[(base + c) * T + tl] = s_arg[c * kTileTargets + tid];
      }
    }
  }
  // transitions evaluated (the reference's apply_candidate count)
  for (int off = 16; off > 0; off >>= 1) nested_cnt += __shfl_xor_sync(0xffffffffu, nested_cnt, off);
  if ((tid & 31) == 0 && nested_cnt) atomicAdd(a.pair_counter, (unsigned long long)nested_cnt);
}

template <typename V>
__global__ void finalize_kernel(const LevelLaunch a) {
  constexpr V INF = VTraits<V>::INF;
  const int64_t T = a.t_hi - a.t_lo;
  const int64_t tl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tl >= T) return;
  const int64_t t = a.t_lo + tl;
  const int C = a.C, lp1 = a.L + 1;
  V* dpt = (V*)a.dp + (size_t)t * C;
  int32_t* bpt = a.bp + (size_t)t * C;
  const V* pv = (const V*)a.part_val;
  for (int c = 0; c < C; ++c) {
    V v = INF;
    int32_t g = INT_MAX;
    for (int64_t ch = 0; ch < a.n_chunks; ++ch) {
      const size_t i = ((size_t)ch * C + c) * T + tl;
      const V x = pv[i];
      const int32_t y = a.part_arg[i];
      if (x < v || (x == v && y < g)) {
        v = x;
        g = y;
      }
    }
    dpt[c] = v;
    bpt[c] = v == INF ? -1 : g;
  }
  // monotone_pass, dp_solver.cpp:180-193 (in place, k then l ascending)
  for (int k = 0; k <= a.K; ++k) {
    for (int l = 0; l <= a.L; ++l) {
      const int c = k * lp1 + l;
      if (k > 0 && dpt[c - lp1] < dpt[c]) {
        dpt[c] = dpt[c - lp1];
        bpt[c] = -3;
      }
      if (l > 0 && dpt[c - 1] < dpt[c]) {
        dpt[c] = dpt[c - 1];
        bpt[c] = -4;
      }
    }
  }
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
  int guard = K + L + 2;
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
    const int64_t prev = (int64_t)(b >> 1);
    const int cpu = b & 1;
    ords[nb] = ord;
    prevs[nb] = prev;
    cpus[nb] = cpu;
    for (int w = 0; w < W; ++w)
      block_bits[(size_t)nb * W + w] = abits[(size_t)ord * W + w] & ~abits[(size_t)prev * W + w];
    ++nb;
    if (cpu) --l;
    else --k;
    ord = prev;
  }
  out->n_blocks = nb;
  out->status = 0;
}

template <typename V, int LP1, int KP1MAX, bool TRAIN>
void launch_t(const LevelLaunch& L, dim3 grid, size_t smem, cudaStream_t st) {
  auto kern = transition_kernel<V, LP1, KP1MAX, TRAIN>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  kern<<<grid, kTileTargets, smem, st>>>(L);
}

template <typename V, bool TRAIN>
void dispatch_cells(const LevelLaunch& L, dim3 grid, size_t smem, cudaStream_t st) {
  const int lp1 = L.L + 1, kp1 = L.K + 1;
  if (lp1 == 1 && kp1 <= 9) return launch_t<V, 1, 9, TRAIN>(L, grid, smem, st);
  if (lp1 == 1 && kp1 <= 17) return launch_t<V, 1, 17, TRAIN>(L, grid, smem, st);
  if (lp1 == 2 && kp1 <= 9) return launch_t<V, 2, 9, TRAIN>(L, grid, smem, st);
  if (lp1 == 3 && kp1 <= 9) return launch_t<V, 3, 9, TRAIN>(L, grid, smem, st);
  if (lp1 == 5 && kp1 <= 9) return launch_t<V, 5, 9, TRAIN>(L, grid, smem, st);
  size_t gsmem = smem + (size_t)L.C * kTileTargets * (sizeof(V) + sizeof(int32_t));
  return launch_t<V, 0, 0, TRAIN>(L, grid, gsmem, st);
}

}  // namespace

void launch_transition(const LevelLaunch& L, cudaStream_t st) {
  const int64_t T = L.t_hi - L.t_lo;
  dim3 grid((unsigned)((T + kTileTargets - 1) / kTileTargets), (unsigned)L.n_chunks, 1);
  size_t smem = (size_t)L.W * kTileTargets * sizeof(uint64_t) * (L.training ? 2 : 1);
  if (L.value_bits == 32) {
    if (L.training) dispatch_cells<int32_t, true>(L, grid, smem, st);
    else dispatch_cells<int32_t, false>(L, grid, smem, st);
  } else {
    if (L.training) dispatch_cells<int64_t, true>(L, grid, smem, st);
    else dispatch_cells<int64_t, false>(L, grid, smem, st);
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
