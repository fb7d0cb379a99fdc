// persistent.cu — every DP level in ONE cooperative launch, as a dataflow
// wavefront (no grid barriers).
//
// The reference walks targets in ordinal order (MaxloadDp::run,
// /root/reference/proj/src/dp_solver.cpp:319-330).  dp[I] depends only on
// dp[I'] for I' ⊊ I, all in earlier levels, so:
//
//   * the work is a static, level-ordered list of items (host plan,
//     capi.cu); CTA b takes items b, b+G, b+2G, ... in order;
//   * an item scans one chunk of source ordinals for a group of targets of
//     level s and first waits (spin on per-level completion counters) only
//     until the levels its chunk covers are finished — the chunks that cover
//     old levels start long before level s-1 is done, so levels overlap;
//   * every item writes one (value, arg) partial per (target, cell); the item
//     that arrives last for a target group (atomic arrival counter) reduces
//     the partials, applies monotone_pass (dp_solver.cpp:180-193) in
//     registers, writes the dp / back-pointer rows and bumps the level's
//     completion counter (release).
//
// Two item shapes:
//   mode 0, lanes own targets (levels with >= 16 targets): item = (group of
//     32 targets, chunk); each lane owns one target and the 4 warps take
//     every 4th source of the chunk, so all lanes of a warp read the same
//     source (broadcast loads, warp-uniform frontier loop).
//   mode 1, lanes own sources (levels with few targets, e.g. the long chains
//     of C4): item = (one target, chunk); the CTA's 128 threads each take
//     sources i, i+128, ... and a warp-shuffle argmin + shared-memory merge
//     combines them.
// All CTAs are co-resident (cooperative launch) and items only wait on
// strictly earlier levels, so the spin waits cannot deadlock.
#include <climits>
#include <cstdint>

#include "scan.cuh"

namespace dsg {

namespace {

using namespace scan;

constexpr int kWarps = kTileTargets / 32;  // warps per CTA (4)
constexpr int kGroup = 32;                 // targets per mode-0 item
constexpr uint64_t kWatchdogNs = 20000000000ull;

__device__ __forceinline__ unsigned long long pack_key(int32_t v, int32_t arg) {
  return ((unsigned long long)((uint32_t)v ^ 0x80000000u) << 32) | (uint32_t)arg;
}

template <typename V>
__device__ __forceinline__ void warp_argmin(V& v, int32_t& g) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const V v2 = __shfl_xor_sync(0xffffffffu, v, off);
    const int32_t g2 = __shfl_xor_sync(0xffffffffu, g, off);
    vmin_arg(v, g, v2, g2);
  }
}

// Wait until levels [j_lo, j_hi] are complete.  Returns false on stop/err.
__device__ bool wait_levels(const PersistPlan& p, int j_lo, int j_hi) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    s_ok = 1;
    uint64_t t0 = 0;
    for (int j = j_lo; j <= j_hi && s_ok; ++j) {
      const unsigned need = (unsigned)(p.level_off[j + 1] - p.level_off[j]);
      if (ld_relaxed_sys(p.done + j) >= need) continue;
      // polite polling: back off up to ~1 us so the spinning warp does not
      // steal issue slots from the co-resident CTAs doing the real work
      unsigned ns = 32, polls = 0;
      if (!t0) t0 = globaltimer();
      while (ld_relaxed_sys(p.done + j) < need) {
        __nanosleep(ns);
        ns = ns < 1024 ? ns * 2 : 1024;
        if ((++polls & 63) != 0) continue;
        if (ld_relaxed((const unsigned*)p.stop) != 0) {
          s_ok = 0;
          break;
        }
        if (globaltimer() - t0 > kWatchdogNs) {
          atomicExch(p.err, 1);
          atomicExch(p.stop, 1);
          s_ok = 0;
          break;
        }
      }
    }
    if (p.world == 1) __threadfence();  // acquire the finished rows
    else __threadfence_system();        // ... including peers' NVLink stores
  }
  __syncthreads();
  return s_ok != 0;
}

// Mode-0 partial of (group unit, chunk): [unit][chunk][cell][lane], so a
// warp's 32 targets store one contiguous 128-byte line per cell.
template <typename V, int CMAX, bool kGeneric, int CS>
__device__ __forceinline__ void write_partial(const LevelLaunch& a, size_t pbase, int64_t unit,
                                              int64_t chunk, int64_t chunks, int lane,
                                              const V* best, const int32_t* barg, const V* colv,
                                              const int32_t* cola) {
  const int C = a.C;
  const size_t base = pbase + ((size_t)unit * chunks + chunk) * C * kGroup + lane;
  V* pv = (V*)a.part_val + base;
  int32_t* pa = a.part_arg + base;
  if (!kGeneric) {
#pragma unroll
    for (int c = 0; c < CMAX; ++c) {
      if (c < C) {
        pv[c * kGroup] = best[c];
        pa[c * kGroup] = barg[c];
      }
    }
  } else {
    for (int c = 0; c < C; ++c) {
      pv[c * kGroup] = colv[c * CS];
      pa[c * kGroup] = cola[c * CS];
    }
  }
}

template <typename V, int LP1, int KP1MAX, bool TRAIN>
__global__ void __launch_bounds__(kTileTargets) persistent_levels_kernel(const LevelLaunch a,
                                                                         const PersistPlan p) {
  constexpr V INF = VTraits<V>::INF;
  constexpr bool kGeneric = LP1 == 0;
  constexpr bool kKeys = sizeof(V) == 4;
  constexpr int CMAX = kGeneric ? 1 : LP1 * KP1MAX;
  constexpr int TS = kGroup;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_last;
  const int W = a.W, C = a.C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // shared: target group [W][32] (+ interior) — mode 1 uses column 0 —,
  // merge buffer [C][32] (value, arg), generic cells [4 warps][C][32]
  uint64_t* s_tgt = reinterpret_cast<uint64_t*>(smem);
  uint64_t* s_int = s_tgt + (size_t)W * TS;
  V* m_val = reinterpret_cast<V*>(s_int + (TRAIN ? (size_t)W * TS : 0));
  int32_t* m_arg = reinterpret_cast<int32_t*>(m_val + (size_t)C * TS);
  V* g_val = reinterpret_cast<V*>(m_arg + (size_t)C * TS);
  int32_t* g_arg = reinterpret_cast<int32_t*>(g_val + (kGeneric ? (size_t)kWarps * C * TS : 0));
  V* colv = g_val + (size_t)warp * C * TS + lane;
  int32_t* cola = g_arg + (size_t)warp * C * TS + lane;
  const V* pv = (const V*)a.part_val;
  const int32_t* pa = a.part_arg;
  unsigned nested_total = 0;
  int s = 1;  // current level (items are level ordered)
  // Which list this CTA walks: with a split, the first crit_blocks CTAs take
  // the critical items (chunks over the newest level, which gate the next
  // level) and the rest the background items (older sources, ready early),
  // so the level chain never queues behind a long background item.
  const bool split = p.crit_blocks > 0;
  const bool crit = split && (int)blockIdx.x < p.crit_blocks;
  const int64_t* base = !split ? p.item_base : (crit ? p.crit_base : p.bg_base);
  const int64_t total = !split ? p.total_items : (crit ? p.total_crit : p.total_bg);
  const int64_t first = !split ? blockIdx.x : (crit ? blockIdx.x : blockIdx.x - p.crit_blocks);
  const int64_t stride = !split ? gridDim.x : (crit ? p.crit_blocks : gridDim.x - p.crit_blocks);

  for (int64_t gi = first; gi < total; gi += stride) {
    while (s + 1 < p.n_levels && gi >= base[s + 1]) ++s;
    const int64_t t_lo = p.level_off[s], t_hi = p.level_off[s + 1];
    const int64_t T = t_hi - t_lo;
    const int64_t chunks = p.n_chunks[s];
    const int mode = p.mode[s];
    const size_t pb = (size_t)p.part_base[s];
    const int64_t it = gi - base[s];
    const int64_t units = mode == 0 ? (T + TS - 1) / TS : T;
    const int64_t unit = it % units;
    const int64_t chunk = it / units + ((split && crit) ? p.n_old[s] : 0);
    if (p.world > 1 && (int)(unit % p.world) != p.rank) continue;  // another GPU's unit
    const int64_t s0 = p.chunk_lo[p.chunk_base[s] + chunk];
    const int64_t s1 = p.chunk_lo[p.chunk_base[s] + chunk + 1];
    // sources [s0, s1) must be final
    const uint64_t tr0 = p.trace ? globaltimer() : 0;
    if (!wait_levels(p, p.level_of[s0], p.level_of[s1 - 1])) break;
    const uint64_t tr1 = p.trace ? globaltimer() : 0;
    if (blockIdx.x == 0 && tid == 0 && p.deadline_ns && globaltimer() > (uint64_t)p.deadline_ns)
      atomicExch(p.stop, 1);

    V best[CMAX];
    int32_t barg[CMAX];
    init_cells<V, LP1, KP1MAX, TS>(C, best, barg, colv, cola);
    int64_t n_act;  // targets of this unit
    if (mode == 0) {
      // ------------------------------------ lanes own targets
      const Target<V> x = load_target<V, TRAIN, TS>(a, t_lo, t_hi, unit, lane, s_tgt + lane,
                                                    s_int + lane, warp == 0);
      __syncthreads();
      nested_total += scan_sources<V, LP1, KP1MAX, TRAIN, TS, true, TS>(
          a, x, s0 + warp, s1, kWarps, s_tgt + lane, s_int + lane, best, barg, colv, cola);
      // merge the 4 warps into warp 0 through the merge buffer
      for (int src = 1; src < kWarps; ++src) {
        __syncthreads();
        if (warp == src) {
          if (!kGeneric) {
#pragma unroll
            for (int c = 0; c < CMAX; ++c) {
              if (c < C) {
                m_val[c * TS + lane] = best[c];
                m_arg[c * TS + lane] = barg[c];
              }
            }
          } else {
            for (int c = 0; c < C; ++c) {
              m_val[c * TS + lane] = colv[c * TS];
              m_arg[c * TS + lane] = cola[c * TS];
            }
          }
        }
        __syncthreads();
        if (warp == 0) {
          if (!kGeneric) {
#pragma unroll
            for (int c = 0; c < CMAX; ++c)
              if (c < C) vmin_arg(best[c], barg[c], m_val[c * TS + lane], m_arg[c * TS + lane]);
          } else {
            for (int c = 0; c < C; ++c)
              vmin_arg(colv[c * TS], cola[c * TS], m_val[c * TS + lane], m_arg[c * TS + lane]);
          }
        }
      }
      if (warp == 0) {
        if (kKeys) {
          // 32-bit values: one packed (value, arg) atomicMin per cell — the
          // L2 merges the chunks, the finalizer reads C words per target
          if (x.active) {
            unsigned long long* key = p.keys + (size_t)x.t * C;
            if (!kGeneric) {
#pragma unroll
              for (int c = 0; c < CMAX; ++c)
                if (c < C && best[c] != INF) atomicMin(key + c, pack_key((int32_t)best[c], barg[c]));
            } else {
              for (int c = 0; c < C; ++c)
                if (colv[c * TS] != INF) atomicMin(key + c, pack_key((int32_t)colv[c * TS], cola[c * TS]));
            }
          }
        } else {
          write_partial<V, CMAX, kGeneric, TS>(a, pb, unit, chunk, chunks, lane, best, barg, colv, cola);
        }
      }
      n_act = min((int64_t)TS, T - unit * TS);
    } else {
      // ------------------------------------ lanes own sources
      const int64_t t = t_lo + unit;
      for (int w = tid; w < W; w += kTileTargets) {
        s_tgt[w] = __ldg(a.abits + (size_t)t * W + w);
        if (TRAIN) s_int[w] = __ldg(a.intbits + (size_t)t * W + w);
      }
      __syncthreads();
      const Target<V> x = target_scalars<V, TRAIN>(a, t, unit, true);
      nested_total += scan_sources<V, LP1, KP1MAX, TRAIN, 1, false, TS>(
          a, x, s0 + tid, s1, kTileTargets, s_tgt, s_int, best, barg, colv, cola);
      // lanes -> warp (shuffle argmin) -> CTA (shared memory)
      if (!kGeneric) {
#pragma unroll
        for (int c = 0; c < CMAX; ++c) {
          if (c < C) {
            warp_argmin(best[c], barg[c]);
            if (lane == 0) {
              m_val[c * TS + warp] = best[c];
              m_arg[c * TS + warp] = barg[c];
            }
          }
        }
      } else {
        for (int c = 0; c < C; ++c) {
          warp_argmin(colv[c * TS], cola[c * TS]);
          if (lane == 0) {
            m_val[c * TS + warp] = colv[c * TS];
            m_arg[c * TS + warp] = cola[c * TS];
          }
        }
      }
      __syncthreads();
      V* pvw = (V*)a.part_val + pb;
      int32_t* paw = a.part_arg + pb;
      for (int c = tid; c < C; c += kTileTargets) {
        V v = m_val[c * TS];
        int32_t g = m_arg[c * TS];
        for (int w = 1; w < kWarps; ++w) vmin_arg(v, g, m_val[c * TS + w], m_arg[c * TS + w]);
        pvw[((size_t)unit * chunks + chunk) * C + c] = v;
        paw[((size_t)unit * chunks + chunk) * C + c] = g;
      }
      n_act = 1;
    }
    // arrival: the last chunk of this unit finalizes its targets
    __syncthreads();
    const uint64_t tr2 = p.trace ? globaltimer() : 0;
    if (tid == 0) {
      __threadfence();  // cumulative release of this CTA's partials
      s_last = atomicAdd(p.tile_count + p.tile_base[s] + unit, 1u) == chunks - 1;
      if (s_last) __threadfence();  // acquire the other chunks' partials
    }
    __syncthreads();
    if (s_last) {
      const int64_t tl0 = mode == 0 ? unit * TS : unit;
      if (mode == 0 && kKeys) {
        for (int r = tid; r < C * TS; r += kTileTargets) {
          const int c = r / TS, tl_local = r % TS;
          V v = INF;
          int32_t g = -1;
          if (tl_local < n_act) {
            const unsigned long long k = __ldcg(p.keys + (size_t)(t_lo + tl0 + tl_local) * C + c);
            if (k != ~0ull) {
              v = (V)(int32_t)((uint32_t)(k >> 32) ^ 0x80000000u);
              g = (int32_t)(uint32_t)(k & 0xffffffffull);
            }
          }
          m_val[r] = v;
          m_arg[r] = g;
        }
      } else if (mode == 0) {
        // lanes = the group's targets, warps over chunks (coalesced
        // [chunk][cell][lane] lines), then the 4 warps merge in shared memory
        const size_t ubase = pb + (size_t)unit * chunks * C * TS + lane;
        for (int c = 0; c < C; ++c) {
          V v = INF;
          int32_t g = INT_MAX;
          for (int64_t ch = warp; ch < chunks; ch += kWarps) {
            const size_t i = ubase + ((size_t)ch * C + c) * TS;
            vmin_arg(v, g, __ldcg(pv + i), __ldcg(pa + i));
          }
          // stash per warp in the (now idle) generic / merge area
          if (warp == 0) {
            m_val[c * TS + lane] = v;
            m_arg[c * TS + lane] = g;
          }
          for (int w = 1; w < kWarps; ++w) {
            __syncthreads();
            if (warp == w) vmin_arg(m_val[c * TS + lane], m_arg[c * TS + lane], v, g);
          }
        }
        __syncthreads();
        for (int r = tid; r < C * TS; r += kTileTargets)
          if (m_val[r] == INF) m_arg[r] = -1;
      } else {
        // one target: warps over cells, lanes over chunks, shuffle argmin
        for (int c = warp; c < C; c += kWarps) {
          const size_t base = pb + ((size_t)unit * chunks) * C + c;
          V v = INF;
          int32_t g = INT_MAX;
          for (int64_t ch = lane; ch < chunks; ch += 32)
            vmin_arg(v, g, __ldcg(pv + base + (size_t)ch * C), __ldcg(pa + base + (size_t)ch * C));
          warp_argmin(v, g);
          if (lane == 0) {
            m_val[c * TS] = v;
            m_arg[c * TS] = v == INF ? -1 : g;
          }
        }
      }
      __syncthreads();
      if (warp == 0 && lane < n_act) {
        // the finished rows go to every rank's table (this GPU's own for
        // world == 1; NVLink peer stores otherwise)
        const int64_t t = t_lo + tl0 + lane;
        if (!kGeneric) {
#pragma unroll
          for (int c = 0; c < CMAX; ++c) {
            if (c < C) {
              best[c] = m_val[c * TS + lane];
              barg[c] = m_arg[c * TS + lane];
            }
          }
          monotone_regs<V, LP1, CMAX>(best, barg, C);
          for (int r = 0; r < p.world; ++r) {
            V* dpt = (V*)p.peer_dp[r] + (size_t)t * C;
            int32_t* bpt = p.peer_bp[r] + (size_t)t * C;
#pragma unroll
            for (int c = 0; c < CMAX; ++c) {
              if (c < C) {
                dpt[c] = best[c];
                bpt[c] = barg[c];
              }
            }
          }
        } else {
          monotone_strided(m_val + lane, m_arg + lane, TS, a.K, a.L);
          for (int r = 0; r < p.world; ++r) {
            V* dpt = (V*)p.peer_dp[r] + (size_t)t * C;
            int32_t* bpt = p.peer_bp[r] + (size_t)t * C;
            for (int c = 0; c < C; ++c) {
              dpt[c] = m_val[c * TS + lane];
              bpt[c] = m_arg[c * TS + lane];
            }
          }
        }
      }
      __syncthreads();
      if (tid == 0) {
        if (p.world == 1) {
          __threadfence();  // release the rows
          atomicAdd(p.peer_done[0] + s, (unsigned)n_act);
        } else {
          __threadfence_system();  // rows reached every peer before its counter moves
          for (int r = 0; r < p.world; ++r) atomicAdd_system(p.peer_done[r] + s, (unsigned)n_act);
        }
      }
    }
    __syncthreads();
    if (p.trace && tid == 0) {
      uint64_t* tr = p.trace + (gi + ((split && !crit) ? p.total_crit : 0)) * 4;
      tr[0] = tr0;
      tr[1] = tr1;
      tr[2] = tr2;
      tr[3] = globaltimer() | (s_last ? (1ull << 63) : 0ull);
    }
  }
  for (int off = 16; off > 0; off >>= 1)
    nested_total += __shfl_xor_sync(0xffffffffu, nested_total, off);
  if (lane == 0 && nested_total) atomicAdd(a.pair_counter, (unsigned long long)nested_total);
}

size_t persist_smem(const LevelLaunch& L, bool generic, size_t vsz) {
  const int tr = L.training ? 2 : 1;
  size_t s = (size_t)L.W * kGroup * sizeof(uint64_t) * tr;   // targets
  s += (size_t)L.C * kGroup * (vsz + sizeof(int32_t));        // merge buffer
  if (generic) s += (size_t)kWarps * L.C * kGroup * (vsz + sizeof(int32_t));
  return s;
}

template <typename V, int LP1, int KP1MAX, bool TRAIN>
void run_variant(const LevelLaunch& L, const PersistPlan* P, cudaStream_t st, PersistInfo* info) {
  const size_t smem = persist_smem(L, LP1 == 0, sizeof(V));
  auto kern = persistent_levels_kernel<V, LP1, KP1MAX, TRAIN>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTileTargets, smem);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int full = per_sm * sms;
  info->per_sm = per_sm;
  if (info->query_only) {
    info->blocks = full;
    return;
  }
  int blocks = info->blocks > 0 ? info->blocks : full;
  if (blocks > full) blocks = full;
  if (blocks < 1) blocks = 1;
  LevelLaunch la = L;
  PersistPlan pa = *P;
  void* args[] = {&la, &pa};
  info->launch_error = (int)cudaLaunchCooperativeKernel((const void*)kern, dim3(blocks),
                                                        dim3(kTileTargets), args, smem, st);
  info->blocks = blocks;
}

template <typename V, bool TRAIN>
void dispatch_cells(const LevelLaunch& L, const PersistPlan* P, cudaStream_t st, PersistInfo* info) {
  const int lp1 = L.L + 1, kp1 = L.K + 1;
  if (L.repl) return run_variant<V, 0, 0, TRAIN>(L, P, st, info);  // replication: generic cells
  if (lp1 == 1 && kp1 <= 9) return run_variant<V, 1, 9, TRAIN>(L, P, st, info);
  if (lp1 == 1 && kp1 <= 17) return run_variant<V, 1, 17, TRAIN>(L, P, st, info);
  if (lp1 == 2 && kp1 <= 9) return run_variant<V, 2, 9, TRAIN>(L, P, st, info);
  if (lp1 == 3 && kp1 <= 9) return run_variant<V, 3, 9, TRAIN>(L, P, st, info);
  return run_variant<V, 0, 0, TRAIN>(L, P, st, info);
}

void dispatch(const LevelLaunch& L, const PersistPlan* P, cudaStream_t st, PersistInfo* info) {
  if (L.value_bits == 32) {
    if (L.training) dispatch_cells<int32_t, true>(L, P, st, info);
    else dispatch_cells<int32_t, false>(L, P, st, info);
  } else {
    if (L.training) dispatch_cells<int64_t, true>(L, P, st, info);
    else dispatch_cells<int64_t, false>(L, P, st, info);
  }
}

}  // namespace

void query_persistent(const LevelLaunch& L, PersistInfo* info) {
  info->query_only = 1;
  PersistPlan dummy{};
  dispatch(L, &dummy, nullptr, info);
  info->query_only = 0;
}

void launch_persistent(const LevelLaunch& L, const PersistPlan& P, cudaStream_t st,
                       PersistInfo* info) {
  dispatch(L, &P, st, info);
  count_launch();
}

}  // namespace dsg
