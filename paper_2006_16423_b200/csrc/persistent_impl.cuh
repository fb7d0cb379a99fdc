#pragma once
// persistent_impl.cuh — every DP level in ONE cooperative launch, as a dataflow
// wavefront (no grid barriers).
//
// The reference walks targets in ordinal order (MaxloadDp::run,
// /root/reference/proj/src/dp_solver.cpp:319-330).  dp[I] depends only on
// dp[I'] for I' ⊊ I, all in earlier levels, so:
//
//   * the work is a list of items (host plan, capi.cu) sorted by readiness;
//     CTAs claim the next item from one atomic counter;
//   * an item scans one chunk of source ordinals for a unit of targets of
//     level s and first waits (spin on the per-level completion counter)
//     only until the last level its chunk covers is finished — levels
//     complete in order, and the chunks that cover old levels start long
//     before level s-1 is done, so levels overlap;
//   * every item merges its per-target cell minima (value-only: the argmin
//     is recovered for the optimal path during traceback); the item that
//     arrives last for a unit (atomic arrival counter) applies monotone_pass
//     (dp_solver.cpp:180-193) in registers, writes the dp rows — into every
//     rank's table when the solve is sharded over GPUs — and bumps the
//     level's completion counter (release).
//
// Two item shapes:
//   mode 0, lanes own targets (levels with >= 16 targets): item = (group of
//     32 targets, chunk); each lane owns one target and the 4 warps take
//     every 4th source of the chunk, so all lanes of a warp read the same
//     source (broadcast loads, warp-uniform frontier loop).  The warps merge
//     in shared memory; chunks merge with a value atomicMin.
//   mode 1, lanes own sources (levels with few targets, e.g. the long chains
//     of C4): item = (one target, chunk); the CTA's 128 threads each take
//     sources i, i+128, ...; a warp-shuffle min + shared memory combine them
//     into one partial per (target, chunk, cell).
// All CTAs are co-resident (cooperative launch) and items only wait on
// strictly earlier levels, so the spin waits cannot deadlock; a watchdog
// aborts (flag) instead of hanging.
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "scan.cuh"

namespace dsg {

namespace {

using namespace scan;

constexpr int kWarps = kTileTargets / 32;  // warps per CTA (4)
constexpr int kGroup = 32;                 // targets per mode-0 item
// The exact-word/exact-cell variants (the C2 hot loop) are held to 64
// registers so 8 CTAs fit per SM (measured: 7.4 ms vs 8.0 ms at 80
// registers on C2; the few spills sit off the source loop).  The other
// variants keep their natural allocation (bounding them spills the hot loop).
#ifndef DSG_MIN_BLOCKS_EXACT
#define DSG_MIN_BLOCKS_EXACT 7  // measured: 7 (72 registers) < 8 (64) on C2 since r2
#endif
constexpr int kMinBlocksExact = DSG_MIN_BLOCKS_EXACT;
#ifndef DSG_MIN_BLOCKS_BIG
#define DSG_MIN_BLOCKS_BIG 5  // (3,7) cells: 5 (96 registers) measured best on C3 (6: +3 %, 4: +1 %)
#endif
// more register cells (e.g. C3's 3x7): a softer cap
constexpr int kMinBlocksExactBig = DSG_MIN_BLOCKS_BIG;
constexpr uint64_t kWatchdogNs = 20000000000ull;
// mode-1 old chunks of more sources take the one-source-per-thread path
// (row loads spread over all threads); fewer, and the finisher, fold with
// threads over (cell, source group)
constexpr int kCellwiseMax = 16;

template <typename V>
__device__ __forceinline__ V warp_min(V v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = min(v, (V)__shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

__device__ __forceinline__ void atomic_min_v(int32_t* p, int32_t v) { atomicMin(p, v); }
__device__ __forceinline__ void atomic_min_v(int64_t* p, int64_t v) {
  atomicMin(reinterpret_cast<long long*>(p), (long long)v);
}

// Implicit mode-0 chunk boundaries.  An item's latency under full load
// grows with its length, and an item whose last source is in level s-1-d
// has d levels of slack before it gates level s.  So the recent levels are
// chunked short, graded by that slack: level s-1-d (d = 1..grade) in chunks
// of min(len0, len1 << (d-1)); everything older (levels <= s-2-grade) in
// chunks of len0; the last chunk is the cover chunk (each target's lower
// covers, all in level s-1): s0 = s1 = -1.
__device__ __forceinline__ void mode0_chunk(const PersistPlan& p, int s, int64_t c, int64_t& s0,
                                            int64_t& s1) {
  const int G = min(p.grade, s - 1);
  const int64_t Rg = p.level_off[s - 1 - G];
  const int64_t n_old = (Rg + p.chunk_len0 - 1) / p.chunk_len0;
  if (c < n_old) {
    s0 = c * p.chunk_len0;
    s1 = min(s0 + p.chunk_len0, Rg);
    return;
  }
  c -= n_old;
  for (int d = G; d >= 1; --d) {
    const int64_t lo = p.level_off[s - 1 - d], hi = p.level_off[s - d];
    const int64_t len = min((int64_t)p.chunk_len0, (int64_t)p.chunk_len1 << (d - 1));
    const int64_t n = (hi - lo + len - 1) / len;
    if (c < n) {
      s0 = lo + c * len;
      s1 = min(s0 + len, hi);
      return;
    }
    c -= n;
  }
  s0 = s1 = -1;
}

// Mode 0 cover chunk: lane = target, warp w takes covers w, w+4, ... of it.
// Per-lane trip counts differ, so no warp collectives in here.
template <typename V, int LP1, int KP1MAX, bool TRAIN, int TS, bool CX>
__device__ __forceinline__ unsigned scan_covers(const LevelLaunch& a, const Target<V>& x, int first,
                                                int step, const uint64_t* tA, const uint64_t* tInt,
                                                V* best, V* colv, const void* dpm) {
  constexpr V INF = VTraits<V>::INF;
  constexpr bool kGeneric = LP1 == 0;
  constexpr int CMAX = kGeneric ? 1 : LP1 * KP1MAX;
  constexpr V NEG = (V)(-INF - 1);
  if (!x.active) return 0;
  const int C = CX ? CMAX : a.C;
  const int64_t c0 = __ldg(a.cov_off + x.t), c1 = __ldg(a.cov_off + x.t + 1);
  unsigned n = 0;
  for (int64_t j = c0 + first; j < c1; j += step) {
    const int64_t src = __ldg(a.cov + j);
    ++n;
    bool gated;
    V acc, cpu, mem_blk;
    const V* sdp = (const V*)dpm + (size_t)src * C;
    V row[CMAX > 1 ? CMAX - 1 : 1];
    if constexpr (!kGeneric) {
#pragma unroll
      for (int c = 0; c + 1 < CMAX; ++c) row[c] = (c + 1 < C) ? ld_row<false>(sdp + c) : INF;
      auto need = [&](V proc) {
        V thr = NEG;
#pragma unroll
        for (int c = LP1; c < CMAX; ++c)
          if (c < C) thr = vmax(thr, row[c - LP1] < best[c] ? best[c] : NEG);
        return proc < thr;
      };
      pair_cost<V, TRAIN, TS>(a, x, src, tA, tInt, gated, acc, cpu, mem_blk, need);
    } else {
      pair_cost<V, TRAIN, TS>(a, x, src, tA, tInt, gated, acc, cpu, mem_blk);
    }
    if (gated) continue;
    k4_update<V, LP1, KP1MAX, TS, CX>(a, sdp, row, acc, cpu, mem_blk, best, colv);
  }
  return n;
}

// Release-add without an L1 invalidation (atom.release: MEMBAR.ALL + ATOM;
// __threadfence() + atomicAdd would add CCTL.IVALL, which discards the L1
// of every CTA on the SM).  ATOM, not RED: a counter others spin on should
// reach L2 at once.
__device__ __forceinline__ unsigned atom_release_add(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// This CTA's rank-local tables (shared memory, set once per kernel): the
// launch's own (world == 1 or one process per GPU) or, for virtual shards,
// those of rank blockIdx.x % world (PersistPlan::vrank).
struct CtaView {
  const int4* items;
  int64_t total_items;
  unsigned long long* next;
  unsigned* tile_count;
  void* keys;
  const void* dp;  // the dp replica this CTA's sources are read from
  unsigned* done;
  int* stop;
  int rank;
  const int4* run_items;  // chain-runner items of this rank: this runner CTA takes
  int64_t run_total;      //   run_first, run_first + run_step, ... < run_total
  int run_first, run_step;
};

// Stop every rank (deadline, watchdog): a peer spinning on a level the
// stopping rank will never finish must see it instead of its watchdog.
__device__ __forceinline__ void raise_stop(const PersistPlan& p, const CtaView& v, bool err) {
  for (int r = 0; r < p.world; ++r) {
    int* ctl = reinterpret_cast<int*>(p.world > 1 ? p.peer_done[r] - 32 : v.done - 32);
    if (err) atomicExch_system(ctl + 1, 1);
    atomicExch_system(ctl, 1);
  }
}

// Wait until level j is complete (then so are all levels below it: every
// unit of level j consumes all of level j-1).  Returns false on stop/err.
__device__ bool wait_level(const PersistPlan& p, const CtaView& v, int j, bool acquire = false) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    s_ok = 1;
    const unsigned need = (unsigned)(p.level_off[j + 1] - p.level_off[j]);
    if (ld_relaxed_sys(v.done + j) < need) {
      // polite polling: back off up to ~1 us so the spinning warp does not
      // steal issue slots from the co-resident CTAs doing the real work
      unsigned ns = 32, polls = 0;
      const uint64_t t0 = globaltimer();
      while (ld_relaxed_sys(v.done + j) < need) {
        __nanosleep(ns);
        ns = ns < p.poll_ns_max ? ns * 2 : p.poll_ns_max;
        if ((++polls & 63) != 0) continue;
        if (ld_relaxed_sys((const unsigned*)v.stop) != 0) {
          s_ok = 0;
          break;
        }
        if (globaltimer() - t0 > kWatchdogNs) {
          raise_stop(p, v, true);
          s_ok = 0;
          break;
        }
      }
    }
    // world == 1: no acquire fence — every later read of data produced in
    // this kernel (dp rows, keys) goes to L2 (ld.global.cg / cp.async.cg)
    // and is control-dependent on the counter value just observed, and the
    // producers released (MEMBAR) before bumping it.  An acquire would
    // invalidate the whole L1 of the SM (CCTL.IVALL) on every item.
    // Mode-1 items (one source row per thread: the rows share L1 lines, so
    // L1-cached loads are much cheaper than per-cell L2 loads) acquire
    // instead, which invalidates the L1.
    if (p.world > 1) __threadfence_system();  // peers' NVLink stores
    else if (acquire) __threadfence();
    asm volatile("" ::: "memory");
  }
  __syncthreads();
  return s_ok != 0;
}

// Wait until this GPU's counter *c reaches need (the finisher of a mode-1
// target waits for the target's other chunks).  Returns false on stop/err.
__device__ bool wait_count(const PersistPlan& p, const CtaView& v, const unsigned* c,
                           unsigned need) {
  __shared__ int s_ok2;
  if (threadIdx.x == 0) {
    s_ok2 = 1;
    if (ld_relaxed(c) < need) {
      unsigned ns = 32, polls = 0;
      const uint64_t t0 = globaltimer();
      while (ld_relaxed(c) < need) {
        __nanosleep(ns);
        ns = ns < p.poll_ns_max ? ns * 2 : p.poll_ns_max;
        if ((++polls & 63) != 0) continue;
        if (ld_relaxed_sys((const unsigned*)v.stop) != 0) {
          s_ok2 = 0;
          break;
        }
        if (globaltimer() - t0 > kWatchdogNs) {
          raise_stop(p, v, true);
          s_ok2 = 0;
          break;
        }
      }
    }
    asm volatile("" ::: "memory");  // keys are read at L2 (see wait_level)
  }
  __syncthreads();
  return s_ok2 != 0;
}

template <typename V>
__device__ __forceinline__ V ld_relaxed_v(const V* p);
template <>
__device__ __forceinline__ int32_t ld_relaxed_v<int32_t>(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
template <>
__device__ __forceinline__ int64_t ld_relaxed_v<int64_t>(const int64_t* p) {
  int64_t v;
  asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// A dp cell read by a narrow-level item (mode 1, threads over cells): the
// row is polled cell by cell until it is no longer PENDING instead of
// waiting for the level counter — each cell is one aligned store, so a
// non-PENDING value is final, and the producer's fence + counter release
// are off the level-to-level chain.  On stop / watchdog: bail (INF).
// A poll loop's periodic check (every 64 rounds): a stop raised elsewhere,
// or this wait past the watchdog (raises the stop).  t0 starts at the first
// check.
__device__ __forceinline__ bool poll_abort(const PersistPlan& p, const CtaView& cv, uint64_t& t0) {
  if (ld_relaxed_sys((const unsigned*)cv.stop) != 0) return true;
  const uint64_t now = globaltimer();
  if (!t0) t0 = now;
  if (now - t0 > kWatchdogNs) {
    raise_stop(p, cv, true);
    return true;
  }
  return false;
}

template <typename V>
__device__ __forceinline__ V ld_final(const PersistPlan& p, const CtaView& cv, const V* q,
                                      bool& bail) {
  V v = __ldcg(q);
  if (v != VTraits<V>::PENDING) return v;
  unsigned ns = 32, polls = 0;
  const uint64_t t0 = globaltimer();
  while (true) {
    if (p.fin_poll_ns) {
      __nanosleep(ns);
      ns = ns < p.fin_poll_ns ? ns * 2 : p.fin_poll_ns;
    }
    v = ld_relaxed_v<V>(q);
    if (v != VTraits<V>::PENDING) return v;
    if ((++polls & 63) != 0) continue;
    if (ld_relaxed_sys((const unsigned*)cv.stop) != 0) break;
    if (globaltimer() - t0 > kWatchdogNs) {
      raise_stop(p, cv, true);
      break;
    }
  }
  bail = true;
  return VTraits<V>::INF;
}

// Level s gained n finished targets: release their rows, bump the level
// counter on every rank (system scope when peers read it over NVLink).
__device__ __forceinline__ void release_done(const PersistPlan& p, int s, unsigned n) {
  if (p.world == 1) {
    atom_release_add(p.peer_done[0] + s, n);  // release the rows
  } else {
    __threadfence_system();  // rows reached every peer before its counter moves
    for (int r = 0; r < p.world; ++r) atomicAdd_system(p.peer_done[r] + s, n);
  }
}

// Mode 0, one warp: this chunk of `unit` has merged its minima into the
// keys; count the arrival, and if it is the unit's last chunk apply
// monotone_pass (dp_solver.cpp:180-193) to the merged cells, store the rows
// into every rank's table and release them.  Returns whether it finalized.
template <typename V, int LP1, int CMAX>
__device__ bool arrive_finalize_unit(const LevelLaunch& a, const PersistPlan& p, const CtaView& v,
                                     int s, int64_t unit, int64_t t_lo, int64_t T, int64_t chunks,
                                     int lane, V* best, V* colv, const V* keys, int C) {
  constexpr V INF = VTraits<V>::INF;
  constexpr bool kGeneric = LP1 == 0;
  constexpr int TS = kGroup;
  unsigned last = 0;
  __syncwarp();
  if (lane == 0) {
    // release this warp's merges; the last arriver reads the others' at L2
    last = atom_release_add(v.tile_count + p.tile_base[s] + unit, 1u) == chunks - 1;
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return false;
  const int64_t n_act = min((int64_t)TS, T - unit * TS);
  if (lane < n_act) {
    const int64_t t = t_lo + unit * TS + lane;
    const V* key = keys + (size_t)t * C;
    if (!kGeneric) {
#pragma unroll
      for (int c = 0; c < CMAX; ++c)
        if (c < C) best[c] = __ldcg(key + c);
      monotone_regs<V, LP1, CMAX>(best, C);
      for (int r = 0; r < p.world; ++r) {
        V* dpt = (V*)p.peer_dp[r] + (size_t)t * C;
#pragma unroll
        for (int c = 0; c < CMAX; ++c)
          if (c < C) dpt[c] = best[c];
      }
    } else {
      for (int c = 0; c < C; ++c) colv[c * TS] = __ldcg(key + c);
      monotone_strided(colv, TS, a.K, a.L);
      for (int r = 0; r < p.world; ++r) {
        V* dpt = (V*)p.peer_dp[r] + (size_t)t * C;
        for (int c = 0; c < C; ++c) dpt[c] = colv[c * TS];
      }
    }
  }
  __syncwarp();
  if (lane == 0) release_done(p, s, (unsigned)n_act);
  return true;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

// mbarrier + bulk-copy (TMA engine, 1-D) helpers
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile(
      "{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// global -> shared bulk copy (bytes % 16 == 0, both ends 16-byte aligned),
// completing on the CTA's mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Stage a mode-0 old chunk's sources [s0, s1) — bitset rows, records and
// (16-byte aligned superset of the) dp rows, all contiguous in HBM — into
// shared memory with up to three bulk copies issued by one thread on the
// TMA engine, completing on the CTA's mbarrier (phase `ph`, flipped here);
// every thread then waits on the barrier.  The rows were produced by other
// CTAs through the generic proxy and released before the level counter the
// caller observed; the async proxy's reads are ordered after that by a proxy
// fence.
template <typename V>
__device__ __forceinline__ SrcView<V> stage_sources(const LevelLaunch& a, const void* dpm,
                                                    int64_t s0, int64_t s1, int C,
                                                    unsigned char* st, uint64_t* bar,
                                                    unsigned& ph, bool bits_only = false) {
  const int64_t n = s1 - s0;
  const size_t nb = (size_t)n * a.AW * 8, nr = (size_t)n * sizeof(SrcRec);
  const char* gb = reinterpret_cast<const char*>(a.abits + (size_t)s0 * a.AW);
  const char* gr = reinterpret_cast<const char*>(a.srec + s0);
  const size_t d0 = (size_t)s0 * C * sizeof(V), d1 = (size_t)s1 * C * sizeof(V);
  const size_t da = d0 & ~(size_t)15, de = (d1 + 15) & ~(size_t)15;
  const char* gd = reinterpret_cast<const char*>(dpm) + da;
  unsigned char* sb = st;
  unsigned char* sr = sb + nb;
  unsigned char* sd = sr + nr;
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    mbar_arrive_expect_tx(bar, (unsigned)(bits_only ? nb : nb + nr + (de - da)));
    bulk_g2s(sb, gb, (unsigned)nb, bar);
    if (!bits_only) {
      bulk_g2s(sr, gr, (unsigned)nr, bar);
      bulk_g2s(sd, gd, (unsigned)(de - da), bar);
    }
  }
  mbar_wait(bar, ph);
  ph ^= 1u;
  SrcView<V> v;
  v.bits = reinterpret_cast<const uint64_t*>(sb);
  v.rec = reinterpret_cast<const SrcRec*>(sr);
  v.dp = reinterpret_cast<const V*>(sd + (d0 - da));
  v.base = s0;
  return v;
}

// ---------------------------------------------------------------- chain blocks
// A run of single-target levels (the long chains of C4 / C1) is one runner
// CTA's: a chain block item holds up to kChainBlk consecutive levels.  The
// block's static work is done for all its levels at once — targets, the
// fold sources (covers + the F most recent levels, F set by the plan) with
// their block costs, the old chunks' arrivals and merged keys — then the
// levels run back to back, each folding its sources with the rows of the
// recent chain levels taken from a shared-memory ring (no L2 round trip on
// the level-to-level chain), applying monotone_pass (dp_solver.cpp:180-193)
// and storing its row; the block's levels are released together.  The plan
// guarantees every old chunk of a block level reads only levels before the
// block, all released before the block waits for its chunks.
constexpr int kChainBlk = 8;   // levels per chain block
constexpr int kChainSrc = kChainSrcMax;  // fold sources per chain level (covers + window)
constexpr int kChainRing = 32; // rows kept (> any level's fold window)

template <typename V>
struct ChainSmem {
  V* ring;           // [kChainRing][C]
  int64_t* ring_ord; // [kChainRing]
  int64_t* hdr;      // [kChainBlk][8]: t, chunks, tile, c0, ncov, ex0, n_src, -
  uint64_t* tgt;     // [kChainBlk][AW]
  uint64_t* tint;    // [kChainBlk][W] (training)
  V* keys;           // [kChainBlk][C]
  int32_t* src;      // [kChainBlk][kChainSrc]
  int32_t* slot;     // [kChainBlk][kChainSrc] ring row of the source, -1: global
  V* acc;            // [kChainBlk][kChainSrc]
  V* cpu;
  V* mem;
  V* part;           // [kTileTargets]
  V* row;            // [2][C] monotone scratch
};

__host__ __device__ inline size_t chain_smem_bytes(int C, int AW, int W, size_t vsz) {
  size_t b = 0;
  auto al = [&](size_t x) { b = (b + 15) & ~(size_t)15; b += x; };
  al((size_t)kChainRing * C * vsz);
  al(kChainRing * 8);
  al(kChainBlk * 8 * 8);
  al((size_t)kChainBlk * AW * 8);
  al((size_t)kChainBlk * W * 8);
  al((size_t)kChainBlk * C * vsz);
  al(kChainBlk * kChainSrc * 4);
  al(kChainBlk * kChainSrc * 4);
  al(3 * (size_t)kChainBlk * kChainSrc * vsz);
  al((size_t)kTileTargets * vsz);
  al(2 * (size_t)C * vsz);
  return b + 16;
}

template <typename V>
__device__ __forceinline__ ChainSmem<V> chain_smem(unsigned char* base, int C, int AW, int W) {
  ChainSmem<V> m;
  size_t b = 0;
  auto al = [&](size_t x) {
    b = (b + 15) & ~(size_t)15;
    unsigned char* r = base + b;
    b += x;
    return r;
  };
  m.ring = reinterpret_cast<V*>(al((size_t)kChainRing * C * sizeof(V)));
  m.ring_ord = reinterpret_cast<int64_t*>(al(kChainRing * 8));
  m.hdr = reinterpret_cast<int64_t*>(al(kChainBlk * 8 * 8));
  m.tgt = reinterpret_cast<uint64_t*>(al((size_t)kChainBlk * AW * 8));
  m.tint = reinterpret_cast<uint64_t*>(al((size_t)kChainBlk * W * 8));
  m.keys = reinterpret_cast<V*>(al((size_t)kChainBlk * C * sizeof(V)));
  m.src = reinterpret_cast<int32_t*>(al(kChainBlk * kChainSrc * 4));
  m.slot = reinterpret_cast<int32_t*>(al(kChainBlk * kChainSrc * 4));
  m.acc = reinterpret_cast<V*>(al(3 * (size_t)kChainBlk * kChainSrc * sizeof(V)));  // acc | cpu | mem
  m.cpu = m.acc + kChainBlk * kChainSrc;
  m.mem = m.cpu + kChainBlk * kChainSrc;
  m.part = reinterpret_cast<V*>(al((size_t)kTileTargets * sizeof(V)));
  m.row = reinterpret_cast<V*>(al(2 * (size_t)C * sizeof(V)));
  return m;
}

// One chain block: levels [sb, sb + nl).  Returns false when the solve
// stopped (deadline / watchdog / another rank).
template <typename V, bool TRAIN>
__device__ __forceinline__ bool chain_block(const LevelLaunch& a, const PersistPlan& p, const CtaView& cv,
                                         int sb, int nl, int run_lvl, unsigned char* area,
                                         unsigned& nested, uint64_t* tr_mid) {
  constexpr V INF = VTraits<V>::INF;
  const int tid = threadIdx.x;
  const int C = a.C, AW = a.AW, W = a.W, lp1 = a.L + 1;
  const ChainSmem<V> m = chain_smem<V>(area, C, AW, W);
  // level headers
  if (tid < nl) {
    const int s = sb + tid;
    const int64_t t = p.level_off[s];
    const int mode = p.mode[s];
    const int64_t c0 = __ldg(a.cov_off + t);
    const int64_t ncov = __ldg(a.cov_off + t + 1) - c0;
    const int64_t ex0 = p.level_off[s - mode], ex1 = p.level_off[s - 1];
    int64_t* h = m.hdr + tid * 8;
    h[0] = t;
    h[1] = p.n_chunks[s];
    h[2] = p.tile_base[s];
    h[3] = c0;
    h[4] = ncov;
    h[5] = ex0;
    h[6] = min((int64_t)kChainSrc, ncov + (ex1 - ex0));
    if (ncov + (ex1 - ex0) > kChainSrc) raise_stop(p, cv, true);  // the plan keeps it <= kChainSrc
  }
  __syncthreads();
  // target bitsets
  for (int i = tid; i < nl * AW; i += kTileTargets) {
    const int lv = i / AW, w = i % AW;
    m.tgt[i] = __ldg(a.abits + (size_t)m.hdr[lv * 8] * AW + w);
  }
  if (TRAIN)
    for (int i = tid; i < nl * W; i += kTileTargets) {
      const int lv = i / W, w = i % W;
      m.tint[i] = __ldg(a.intbits + (size_t)m.hdr[lv * 8] * W + w);
    }
  __syncthreads();
  // fold sources of every level: subset test and block costs (K2 + K3)
  const int64_t ring_lo = p.level_off[run_lvl];
  for (int i = tid; i < nl * kChainSrc; i += kTileTargets) {
    const int lv = i / kChainSrc, j = i % kChainSrc;
    const int64_t* h = m.hdr + lv * 8;
    if (j >= h[6]) continue;
    const int64_t src = j < h[4] ? (int64_t)__ldg(a.cov + h[3] + j) : h[5] + (j - h[4]);
    const Target<V> x = target_scalars<V, TRAIN>(a, h[0], 0, true);
    const PrePair<V> q = pre_pair<V, TRAIN, 1>(a, x, src, m.tgt + lv * AW, m.tint + lv * W);
    m.src[i] = q.ok ? (int32_t)src : -1;
    // rows of this run's earlier levels are in the ring (this CTA computed
    // them, in order); older rows come from the global table
    m.slot[i] = src >= ring_lo && src < h[0] ? (int32_t)(src % kChainRing) : -1;
    m.acc[i] = q.acc;
    m.cpu[i] = q.cpu;
    m.mem[i] = q.mem_blk;
    nested += q.nested ? 1u : 0u;
  }
  if (p.trace) tr_mid[0] = globaltimer();
  // the old chunks' merges (their sources all precede the block, released)
  __shared__ int s_cok;
  if (tid == 0) s_cok = 1;
  __syncthreads();
  if (tid < nl) {
    const int64_t* h = m.hdr + tid * 8;
    const unsigned need = (unsigned)(h[1] - 1);
    const unsigned* c = cv.tile_count + h[2];
    if (need > 0 && ld_relaxed(c) < need) {
      uint64_t t0 = 0;
      for (unsigned polls = 0; ld_relaxed(c) < need; ++polls) {
        __nanosleep(64);
        if ((polls & 63) == 63 && poll_abort(p, cv, t0)) {
          s_cok = 0;
          break;
        }
      }
    }
  }
  __syncthreads();
  if (!s_cok) return false;
  for (int i = tid; i < nl * C; i += kTileTargets) {
    const int lv = i / C, c = i % C;
    m.keys[i] = __ldcg(reinterpret_cast<const V*>(cv.keys) + (size_t)m.hdr[lv * 8] * C + c);
  }
  __syncthreads();
  if (p.trace) tr_mid[1] = globaltimer();
  const V* dpm = reinterpret_cast<const V*>(cv.dp);
  const int G = max(1, kTileTargets / C);
  const int my_g = tid / C, my_c = tid % C;
  const bool folder = my_g < G;  // a (cell, source group) of the fold
  const int ck = my_c / lp1, cl = my_c % lp1;
  const int offa = ck >= 1 ? my_c - lp1 : 0, offc = cl >= 1 ? my_c - 1 : 0;
  for (int lv = 0; lv < nl; ++lv) {
    const int64_t t = m.hdr[lv * 8];
    const int nsrc = (int)m.hdr[lv * 8 + 6];
    const int32_t* fs = m.src + lv * kChainSrc;
    const int32_t* fsl = m.slot + lv * kChainSrc;
    const V* fa = m.acc + lv * kChainSrc;
    const V* fc = m.cpu + lv * kChainSrc;
    bool bail = false;
    if (folder) {
      V v = INF;
      // ring rows first: 4 sources per round, every shared load of the round
      // issued before any is used (no per-source branch) ...
      for (int j0 = my_g; j0 < nsrc; j0 += 4 * G) {
        int sl[4];
        V xa[4], xc[4], ra[4], rc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + u * G;
          const bool in = j < nsrc;
          sl[u] = in ? fsl[j] : -1;
          xa[u] = in ? fa[j] : INF;
          xc[u] = in ? fc[j] : INF;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const V* row = m.ring + (size_t)(sl[u] < 0 ? 0 : sl[u]) * C;
          ra[u] = row[offa];
          rc[u] = row[offc];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (sl[u] < 0) continue;
          if (ck >= 1 && xa[u] != INF) v = min(v, vmax(ra[u], xa[u]));
          if (cl >= 1) v = min(v, vmax(rc[u], xc[u]));
        }
      }
      // ... then the rows from before the run (global, final or polled)
      for (int j = my_g; j < nsrc; j += G) {
        const int32_t src = fs[j];
        if (src < 0 || fsl[j] >= 0) continue;
        const V* row = dpm + (size_t)src * C;
        if (ck >= 1 && fa[j] != INF) v = min(v, vmax(ld_final(p, cv, row + offa, bail), fa[j]));
        if (cl >= 1) v = min(v, vmax(ld_final(p, cv, row + offc, bail), fc[j]));
      }
      m.part[tid] = v;
    }
    if (__syncthreads_or(bail)) return false;
    // merge the groups with the keys, then monotone_pass: row pass (over l),
    // column pass (over k); thread c < C keeps cell c
    V* r0 = m.row;
    V* r1 = m.row + C;
    if (tid < C) {
      V v = m.keys[lv * C + tid];
      for (int g = 0; g < G; ++g) v = min(v, m.part[g * C + tid]);
      r0[tid] = v;
    }
    __syncthreads();
    if (tid < C) {
      V v = r0[tid];
      for (int ll = 1; ll <= cl; ++ll) v = min(v, r0[tid - ll]);
      r1[tid] = v;
    }
    __syncthreads();
    if (tid < C) {
      V v = r1[tid];
      for (int kk = 1; kk <= ck; ++kk) v = min(v, r1[tid - kk * lp1]);
      m.ring[(size_t)(t % kChainRing) * C + tid] = v;
      if (p.world == 1) const_cast<V*>(dpm)[(size_t)t * C + tid] = v;
      else
        for (int r = 0; r < p.world; ++r) ((V*)p.peer_dp[r])[(size_t)t * C + tid] = v;
    }
    __syncthreads();
  }
  // release the block's levels (one fence for all)
  if (tid == 0) {
    if (p.world == 1) {
      __threadfence();
      for (int lv = 0; lv < nl; ++lv) atomicAdd(p.peer_done[0] + sb + lv, 1u);
    } else {
      __threadfence_system();
      for (int lv = 0; lv < nl; ++lv)
        for (int r = 0; r < p.world; ++r) atomicAdd_system(p.peer_done[r] + sb + lv, 1u);
    }
  }
  return true;
}

template <typename V, int LP1, int KP1MAX, bool TRAIN, int WT, bool CX>
__device__ __forceinline__ void persistent_body(const LevelLaunch& a, const PersistPlan& p) {
  constexpr V INF = VTraits<V>::INF;
  constexpr bool kGeneric = LP1 == 0;
  constexpr int CMAX = kGeneric ? 1 : LP1 * KP1MAX;
  constexpr int TS = kGroup;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_last, s_any_last;
  const int W = a.W, C = CX ? CMAX : a.C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // shared: target columns [AW][32] (padded, pad word 0) + interior
  // [W][32] (mode 1 uses column 0), merge column [C][32], generic cells
  // [4 warps][C][32]
  uint64_t* s_tgt = reinterpret_cast<uint64_t*>(smem);
  uint64_t* s_int = s_tgt + (size_t)a.AW * TS;
  V* m_val = reinterpret_cast<V*>(s_int + (TRAIN ? (size_t)W * TS : 0));
  V* g_val = m_val + (size_t)C * TS;
  V* colv = g_val + (size_t)warp * C * TS + lane;
  // staging area for one old chunk's sources (16-byte aligned)
  // (offset arithmetic on the shared array itself: a round trip through an
  // integer would turn every staged load into a generic LD instead of LDS)
  unsigned char* st_area =
      smem + ((reinterpret_cast<unsigned char*>(g_val + (kGeneric ? (size_t)kWarps * C * TS : 0)) -
               smem + 15) & ~(ptrdiff_t)15);
  unsigned nested_total = 0;
  // the staging area's mbarrier (one arrival: the issuing thread's expect_tx)
  __shared__ __align__(8) uint64_t s_stage_bar;
  unsigned stage_ph = 0;
  if (tid == 0) {
    mbar_init(&s_stage_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // this CTA's rank-local tables (virtual shards: rank blockIdx.x % world)
  __shared__ CtaView cv;
  if (tid == 0) {
    if (p.virt) {
      const int r = (int)(blockIdx.x % (unsigned)p.world);
      const VRank vr = p.vrank[r];
      cv.items = vr.items;
      cv.total_items = vr.total_items;
      cv.next = reinterpret_cast<unsigned long long*>(vr.ctl + 2);
      cv.tile_count = vr.tile_count;
      cv.keys = vr.keys;
      cv.dp = vr.dp;
      cv.done = vr.ctl + 32;
      cv.stop = reinterpret_cast<int*>(vr.ctl);
      cv.rank = r;
      cv.run_items = vr.run_items;
      // CTAs r, r + world, ... (the first `runners`) run rank r's runner
      // segments (header: run_items[i].y = start of segment i)
      const int ri = (int)(blockIdx.x / (unsigned)p.world);
      cv.run_first = ri < p.runners && vr.run_total > 0 ? __ldg(vr.run_items + ri).y : 0;
      cv.run_total = ri < p.runners && vr.run_total > 0 ? __ldg(vr.run_items + ri + 1).y : 0;
      cv.run_step = 1;
    } else {
      cv.items = p.items;
      cv.total_items = p.total_items;
      cv.next = p.next;
      cv.tile_count = p.tile_count;
      cv.keys = p.keys;
      cv.dp = a.dp;
      cv.done = p.done;
      cv.stop = p.stop;
      cv.rank = p.rank;
      cv.run_items = p.run_items;
      const int ri = (int)blockIdx.x;
      cv.run_first = ri < p.runners && p.run_total > 0 ? __ldg(p.run_items + ri).y : 0;
      cv.run_total = ri < p.runners && p.run_total > 0 ? __ldg(p.run_items + ri + 1).y : 0;
      cv.run_step = 1;
    }
  }
  __syncthreads();
  // chain blocks: an empty row ring (shared memory is not cleared at launch)
  if (p.chain && cv.run_total > cv.run_first) {
    int64_t* ro = chain_smem<V>(st_area, a.C, a.AW, W).ring_ord;  // chain_block's layout (a.C)
    for (int i = tid; i < kChainRing; i += kTileTargets) ro[i] = -1;
    __syncthreads();
  }
  // Roles: with crit_ctas > 0 the list starts with the cover items (they gate
  // the levels) and the first crit_ctas CTAs claim only those, so a level's
  // critical work never queues behind ready background work; the other CTAs
  // claim the rest.  Every item still waits only for items listed before it
  // in its own queue or for cover items, which the critical CTAs run in level
  // order, so neither queue can deadlock.  (Virtual shards: one queue.)
  const bool crit_role = (int)blockIdx.x < p.crit_ctas;
  const int64_t n_crit = p.crit_ctas > 0 ? (int64_t)*p.crit_end : 0;
  unsigned long long* ctr = crit_role ? p.crit_next : cv.next;
  const int64_t q_lo = crit_role ? 0 : n_crit, q_hi = crit_role ? n_crit : cv.total_items;
  __shared__ long long s_gi;
  // the chain runner first takes its own items (gi < 0: run item -gi-1)
  // next run item of this CTA (gi = -(index + 1)); in shared memory, not a
  // register live across the scan loop
  __shared__ long long s_run_pos;
  if (tid == 0) {
    const long long rp = cv.run_first;
    s_gi = rp < cv.run_total ? -(1 + rp) : q_lo + (long long)atomicAdd(ctr, 1ull);
    s_run_pos = rp + cv.run_step;
    s_any_last = 0;
  }
  __syncthreads();

  while (true) {
    const int64_t gi = s_gi;
    if (gi >= q_hi) break;
    const int4 item = gi < 0 ? __ldg(cv.run_items + (-gi - 1)) : __ldg(cv.items + gi);
    // claim the next item now; its latency hides behind this one (the
    // runner's own items need no claim)
    // — but the runner claims its first shared item only after its last own
    // item: holding a claimed item while blocked on the chain could hold
    // exactly the chunk that chain waits for
    // (kept in shared memory: no registers live across the scan)
    __shared__ long long s_next_gi;
    if (tid == 0) {
      const long long rp = s_run_pos;
      s_next_gi = rp < cv.run_total ? -(1 + rp)
                  : gi < 0         ? LLONG_MIN
                                   : (long long)(q_lo + atomicAdd(ctr, 1ull));
      if (rp < cv.run_total) s_run_pos = rp + cv.run_step;
    }
    if (item.y < 0) {
      // a chain block (runner lists only)
      const uint64_t tc0 = p.trace ? globaltimer() : 0;
      uint64_t tmid[2] = {0, 0};
      if (!chain_block<V, TRAIN>(a, p, cv, item.x, -item.y, item.w, st_area, nested_total, tmid)) break;
      __syncthreads();
      if (p.trace && tid == 0) {
        // start, static part done, chunk merges read, end
        uint64_t* tr = p.trace + (cv.total_items + (-gi - 1)) * 4;
        tr[0] = tc0;
        tr[1] = tmid[0];
        tr[2] = tmid[1];
        tr[3] = globaltimer() | (1ull << 63);
      }
      if (tid == 0) {
        const long long ng = s_next_gi;
        s_gi = ng == LLONG_MIN ? (long long)(q_lo + atomicAdd(ctr, 1ull)) : ng;
      }
      __syncthreads();
      continue;
    }
    const int s = item.x;
    const int64_t unit = item.y;
    const int64_t chunk = item.z;
    const int64_t t_lo = p.level_off[s], t_hi = p.level_off[s + 1];
    const int64_t T = t_hi - t_lo;
    const int64_t chunks = p.n_chunks[s];
    const int mode = p.mode[s];
    int64_t s0, s1;
    if (mode == 0) {
      mode0_chunk(p, s, chunk, s0, s1);
    } else if (chunk < chunks - 1) {
      s0 = p.chunk_lo[p.chunk_base[s] + chunk];
      s1 = p.chunk_lo[p.chunk_base[s] + chunk + 1];
    } else {
      s0 = s1 = -1;  // the cover chunk
    }
    const uint64_t tr0 = p.trace ? globaltimer() : 0;
    uint64_t tr1 = 0;
    if (blockIdx.x == 0 && tid == 0 && p.deadline_ns && globaltimer() > (uint64_t)p.deadline_ns)
      raise_stop(p, cv, false);
    V best[CMAX];
    uint64_t tr_fold = 0;   // trace: a finisher's fold done (its rows final)
    bool any_last = false;  // trace: some unit of this item finalized
    if (mode == 0) {
      // ------------------------------------ lanes own targets
      // the four warps share one unit and split the chunk's sources
      init_cells<V, LP1, KP1MAX, TS>(C, best, colv);
      if (!kGeneric && warp == 0) {  // the merge column (read back after the scan)
#pragma unroll
        for (int c = 0; c < CMAX; ++c)
          if (c < C) m_val[c * TS + lane] = INF;
      }
      const Target<V> x = load_target<V, TRAIN, TS>(a, t_lo, t_hi, unit, lane, s_tgt + lane,
                                                    s_int + lane, warp == 0);
      // start from the unit's merged minimum so far (other chunks' atomicMin
      // merges): a valid upper bound that lets the scan prune early
      if constexpr (!kGeneric) {
        if (x.active) {
          const V* key = reinterpret_cast<const V*>(cv.keys) + (size_t)x.t * C;
#pragma unroll
          for (int c = 0; c < CMAX; ++c)
            if (c < C) best[c] = __ldcg(key + c);
        }
      }
      // a chunk none of whose pairs can change a cell of any of the unit's
      // targets (chunk_live over the block maxima) only counts its nested
      // pairs; CTA-uniform (the warps' seeds may differ by a late merge)
      bool dead = false;
      if constexpr (!kGeneric) {
        if (s0 >= 0 && p.dead_skip)
          dead = !__syncthreads_or(chunk_live<V, LP1, CMAX>(a, x, best, s0, s1, C));
      }
      // sources [s0, s1) must be final; the target data and the key seeds
      // above do not depend on them, so their latency hides behind the wait
      if (!wait_level(p, cv, item.w)) break;
      tr1 = p.trace ? globaltimer() : 0;
      if (dead) {
        if (p.stage) {
          const SrcView<V> sv = stage_sources<V>(a, cv.dp, s0, s1, C, st_area, &s_stage_bar, stage_ph, true);
          nested_total += count_nested<TS, WT, CX, true>(a, x.active, s0 + warp, s1, kWarps,
                                                         s_tgt + lane, sv.bits, sv.base);
        } else {
          nested_total += count_nested<TS, WT, CX, false>(a, x.active, s0 + warp, s1, kWarps,
                                                          s_tgt + lane, nullptr, 0);
        }
        // the cells are unchanged: no warp merge, no key merge, only the
        // chunk's arrival
        if (warp == 0)
          any_last = arrive_finalize_unit<V, LP1, CMAX>(a, p, cv, s, unit, t_lo, T, chunks, lane,
                                                        best, colv,
                                                        reinterpret_cast<const V*>(cv.keys), C);
      } else {
        if (s0 < 0) {
          nested_total += scan_covers<V, LP1, KP1MAX, TRAIN, TS, CX>(a, x, warp, kWarps, s_tgt + lane,
                                                                     s_int + lane, best, colv, cv.dp);
        } else if (p.stage) {
          nested_total += scan_sources<V, LP1, KP1MAX, TRAIN, TS, true, TS, WT, CX, 0, true>(
              a, x, s0 + warp, s1, kWarps, s_tgt + lane, s_int + lane, best, colv,
              stage_sources<V>(a, cv.dp, s0, s1, C, st_area, &s_stage_bar, stage_ph));
        } else {
          nested_total += scan_sources<V, LP1, KP1MAX, TRAIN, TS, true, TS, WT, CX>(
              a, x, s0 + warp, s1, kWarps, s_tgt + lane, s_int + lane, best, colv, SrcView<V>{},
              cv.dp);
        }
        // merge the 4 warps into warp 0: one barrier (shared-memory atomicMin
        // into the merge column warp 0 reset at the item's start; generic
        // cells are already per-warp columns in shared memory)
        if (!kGeneric && warp != 0) {
#pragma unroll
          for (int c = 0; c < CMAX; ++c)
            if (c < C && best[c] != INF) atomic_min_v(m_val + c * TS + lane, best[c]);
        }
        __syncthreads();
        if (warp == 0) {
          if (!kGeneric) {
#pragma unroll
            for (int c = 0; c < CMAX; ++c)
              if (c < C) best[c] = min(best[c], m_val[c * TS + lane]);
          } else {
            for (int w = 1; w < kWarps; ++w)
              for (int c = 0; c < C; ++c)
                colv[c * TS] = min(colv[c * TS], g_val[((size_t)w * C + c) * TS + lane]);
          }
          // chunks of a unit merge in L2 with a value atomicMin; the last
          // arriving chunk finalizes the unit (this warp alone)
          if (x.active) {
            V* key = reinterpret_cast<V*>(cv.keys) + (size_t)x.t * C;
            if (!kGeneric) {
#pragma unroll
              for (int c = 0; c < CMAX; ++c)
                if (c < C && best[c] != INF) atomic_min_v(key + c, best[c]);
            } else {
              for (int c = 0; c < C; ++c)
                if (colv[c * TS] != INF) atomic_min_v(key + c, colv[c * TS]);
            }
          }
          any_last = arrive_finalize_unit<V, LP1, CMAX>(a, p, cv, s, unit, t_lo, T, chunks, lane,
                                                        best, colv,
                                                        reinterpret_cast<const V*>(cv.keys), C);
        }
      }
      if (any_last) s_any_last = 1;
    } else {
      // ------------------------------------ lanes own sources
      // Every mode-1 chunk has <= 128 sources (capi.cu).  The newest chunk
      // (c = chunks-1, the one that gates the level) is the target's
      // finisher: it waits for the other chunks' key merges and finalizes —
      // no atomic merge or arrival round trip on the critical path.  The
      // item list puts it after the target's other chunks, so its wait
      // cannot deadlock.
      const int64_t t = t_lo + unit;
      const bool fin = chunk == chunks - 1;
      for (int w = tid; w < a.AW; w += kTileTargets) {
        s_tgt[w] = __ldg(a.abits + (size_t)t * a.AW + w);
        if (TRAIN && w < W) s_int[w] = __ldg(a.intbits + (size_t)t * W + w);
      }
      const Target<V> x = target_scalars<V, TRAIN>(a, t, unit, true);
      V* key = reinterpret_cast<V*>(cv.keys) + (size_t)t * C;
      __syncthreads();
      // One source per thread for the static part: thread j evaluates
      // source j's subset test and block cost (K2+K3) before any wait.  Once
      // the sources are final, threads over (cell, source group) fold the
      // candidates (one L2 round trip for the rows), and the groups merge per
      // cell.  The finisher starts from the other chunks' merged minima and
      // ends with monotone_pass (dp_solver.cpp:180-193: in place, k then l
      // ascending = the 2-D prefix minimum over the (k, l) grid, a row pass
      // then a column pass); an old chunk merges into the keys and arrives.
      if (!fin && s1 - s0 > kCellwiseMax) {
        // an old chunk: thread tid takes source s0 + tid
        init_cells<V, LP1, KP1MAX, TS>(C, best, colv);
        const int64_t my = s0 + tid;
        const bool has = my < s1;
        PrePair<V> q{};
        if (has) q = pre_pair<V, TRAIN, 1>(a, x, my, s_tgt, s_int);
        if (!wait_level(p, cv, item.w, true)) break;  // acquire (ends with __syncthreads)
        tr1 = p.trace ? globaltimer() : 0;
        if (has) post_pair<V, LP1, KP1MAX, TS, CX>(a, q, my, best, colv, cv.dp);
        nested_total += q.nested ? 1u : 0u;
        // lanes -> warp (shuffle min) -> CTA (shared memory) -> keys
        if (!kGeneric) {
#pragma unroll
          for (int c = 0; c < CMAX; ++c) {
            if (c < C) {
              const V v = warp_min(best[c]);
              if (lane == 0) m_val[c * TS + warp] = v;
            }
          }
        } else {
          for (int c = 0; c < C; ++c) {
            const V v = warp_min(colv[c * TS]);
            if (lane == 0) m_val[c * TS + warp] = v;
          }
        }
        __syncthreads();
        for (int c = tid; c < C; c += kTileTargets) {
          V v = m_val[c * TS];
#pragma unroll
          for (int w = 1; w < kWarps; ++w) v = min(v, m_val[c * TS + w]);
          if (v != INF) atomic_min_v(key + c, v);
        }
        __syncthreads();
        if (tid == 0) {
          __threadfence();  // cumulative release of this CTA's merges
          atomicAdd(cv.tile_count + p.tile_base[s] + unit, 1u);
        }
      } else {
        const int64_t c0 = fin ? __ldg(a.cov_off + t) : s0;
        const int64_t ncov = fin ? __ldg(a.cov_off + t + 1) - c0 : 0;
        // mode 1 + F: the finisher also folds the F levels s-2 .. s-1-F
        // (one short ordinal range)
        const int64_t ex0 = (fin && mode > 1) ? p.level_off[s - mode] : 0;
        const int64_t ex1 = (fin && mode > 1) ? p.level_off[s - 1] : 0;
        const int64_t c1 = fin ? c0 + ncov + (ex1 - ex0) : s1;
        __shared__ int32_t f_src[kTileTargets];
        __shared__ V f_acc[kTileTargets], f_cpu[kTileTargets], f_mem[kTileTargets];
        __shared__ V f_part[kTileTargets];
        const int lp1 = a.L + 1;
        const V* dpm = reinterpret_cast<const V*>(cv.dp);
        bool ok = true;
        for (int64_t b0 = c0; b0 < c1 || b0 == c0; b0 += kTileTargets) {
          const int nb = (int)min((int64_t)kTileTargets, c1 - b0);
          // (cell, group) layout: G <= nb groups of C threads when C <= 128
          const int G = C <= kTileTargets ? max(1, min(nb, kTileTargets / C)) : 1;
          const int my_g = C <= kTileTargets ? tid / C : 0, my_c = C <= kTileTargets ? tid % C : tid;
          if (tid < nb) {
            const int64_t j = b0 + tid;
            const int64_t src = !fin ? j : (j - c0 < ncov ? (int64_t)__ldg(a.cov + j) : ex0 + (j - c0 - ncov));
            const PrePair<V> q = pre_pair<V, TRAIN, 1>(a, x, src, s_tgt, s_int);
            f_src[tid] = q.ok ? (int32_t)src : -1;
            f_acc[tid] = q.acc;
            f_cpu[tid] = q.cpu;
            f_mem[tid] = q.mem_blk;
            nested_total += q.nested ? 1u : 0u;  // every lower cover is nested
          }
          if (b0 == c0) {
            // the finisher: the other chunks' merges first (listed before it)
            if (fin && chunks > 1 &&
                !wait_count(p, cv, cv.tile_count + p.tile_base[s] + unit, (unsigned)(chunks - 1))) {
              ok = false;
              break;
            }
            for (int c = tid; c < C; c += kTileTargets) m_val[c] = fin ? __ldcg(key + c) : INF;
            // no level wait: the fold polls the source cells it reads
            __syncthreads();
            tr1 = p.trace ? globaltimer() : 0;
          } else {
            __syncthreads();
          }
          bool bail = false;
          for (int c = my_c; c < C && my_g < G; c += kTileTargets) {
            const int k = c / lp1, l = c % lp1;
            V v = INF;
            if (kGeneric && a.repl) {
              for (int j = my_g; j < nb; j += G) {
                const int32_t src = f_src[j];
                if (src < 0) continue;
                const V* row = dpm + (size_t)src * C;
                const V acc = f_acc[j];
                if (k >= 1 && acc != INF) {
                  for (int rr = 1; rr <= k; ++rr) {
                    const V load = rr == 1 ? acc : replicated<V>(a, acc, f_mem[j], rr);
                    v = min(v, vmax(ld_final(p, cv, row + c - rr * lp1, bail), load));
                  }
                }
                if (l >= 1) v = min(v, vmax(ld_final(p, cv, row + c - 1, bail), f_cpu[j]));
              }
            } else {
              // batches of up to 8 sources: every cell load of the batch is in
              // flight at once (one L2 round trip), PENDING cells polled after
              constexpr int kB = 8;
              for (int j0 = my_g; j0 < nb; j0 += kB * G) {
                V ra[kB], rc[kB];
#pragma unroll
                for (int u = 0; u < kB; ++u) {
                  const int j = j0 + u * G;
                  const int32_t src = j < nb ? f_src[j] : -1;
                  const V* row = dpm + (size_t)(src < 0 ? 0 : src) * C;
                  ra[u] = (src >= 0 && k >= 1 && f_acc[j] != INF) ? __ldcg(row + c - lp1) : INF;
                  rc[u] = (src >= 0 && l >= 1) ? __ldcg(row + c - 1) : INF;
                }
#pragma unroll
                for (int u = 0; u < kB; ++u) {
                  const int j = j0 + u * G;
                  if (j >= nb) break;
                  const int32_t src = f_src[j];
                  if (src < 0) continue;
                  const V* row = dpm + (size_t)src * C;
                  if (ra[u] == VTraits<V>::PENDING) ra[u] = ld_final(p, cv, row + c - lp1, bail);
                  if (rc[u] == VTraits<V>::PENDING) rc[u] = ld_final(p, cv, row + c - 1, bail);
                  if (k >= 1 && f_acc[j] != INF) v = min(v, vmax(ra[u], f_acc[j]));
                  if (l >= 1) v = min(v, vmax(rc[u], f_cpu[j]));
                }
              }
            }
            if (G > 1) f_part[tid] = v;
            else m_val[c] = min(m_val[c], v);
          }
          if (__syncthreads_or(bail)) {
            ok = false;
            break;
          }
          if (G > 1) {
            for (int c = tid; c < C; c += kTileTargets) {
              V v = m_val[c];
              for (int g = 0; g < G; ++g) v = min(v, f_part[g * C + c]);
              m_val[c] = v;
            }
            __syncthreads();
          }
          if (b0 + kTileTargets >= c1) break;
        }
        if (!ok) break;
        if (fin) {
          V* tmp = m_val + C;  // row pass (over l), then column pass (over k)
          for (int c = tid; c < C; c += kTileTargets) {
            const int l = c % lp1;
            V v = m_val[c];
            for (int ll = 1; ll <= l; ++ll) v = min(v, m_val[c - ll]);
            tmp[c] = v;
          }
          __syncthreads();
          for (int c = tid; c < C; c += kTileTargets) {
            const int k = c / lp1;
            V v = tmp[c];
            for (int kk = 1; kk <= k; ++kk) v = min(v, tmp[c - kk * lp1]);
            // one GPU: the local table (no dependent load of the peer list
            // on the level-to-level chain)
            if (p.world == 1) const_cast<V*>(reinterpret_cast<const V*>(cv.dp))[(size_t)t * C + c] = v;
            else
              for (int r = 0; r < p.world; ++r) ((V*)p.peer_dp[r])[(size_t)t * C + c] = v;
          }
          if (p.trace) tr_fold = globaltimer();
          __syncthreads();  // every cell stored before the (cumulative) release
          if (tid == 0) {
            release_done(p, s, 1u);
            s_any_last = 1;
          }
        } else {
          for (int c = tid; c < C; c += kTileTargets)
            if (m_val[c] != INF) atomic_min_v(key + c, m_val[c]);
          __syncthreads();
          if (tid == 0) {
            __threadfence();  // cumulative release of this CTA's merges
            atomicAdd(cv.tile_count + p.tile_base[s] + unit, 1u);
          }
        }
      }
    }
    __syncthreads();
    const uint64_t tr2 = p.trace ? (tr_fold ? tr_fold : globaltimer()) : 0;
    if (p.trace && tid == 0) {  // runner items after the list's
      const long long g = s_gi;
      uint64_t* tr = p.trace + (g >= 0 ? g : cv.total_items + (-g - 1)) * 4;
      tr[0] = tr0;
      tr[1] = tr1;
      tr[2] = tr2;
      tr[3] = globaltimer() | (s_any_last ? (1ull << 63) : 0ull);
    }
    if (tid == 0) s_any_last = 0;
    if (tid == 0) {
      const long long ng = s_next_gi;
      s_gi = ng == LLONG_MIN ? (long long)(q_lo + atomicAdd(ctr, 1ull)) : ng;
    }
    __syncthreads();
  }
  for (int off = 16; off > 0; off >>= 1)
    nested_total += __shfl_xor_sync(0xffffffffu, nested_total, off);
  if (lane == 0 && nested_total) atomicAdd(a.pair_counter, (unsigned long long)nested_total);
}

template <typename V, int LP1, int KP1MAX, bool TRAIN, int WT, bool CX>
__global__ void __launch_bounds__(kTileTargets) persistent_levels_kernel(const LevelLaunch a,
                                                                         const PersistPlan p) {
  persistent_body<V, LP1, KP1MAX, TRAIN, WT, CX>(a, p);
}

// exact variants: register budget for kMinBlocksExact resident CTAs per SM
template <typename V, int LP1, int KP1MAX, bool TRAIN, int WT, bool CX>
__global__ void __launch_bounds__(kTileTargets,
                                  LP1 * KP1MAX <= 9 && sizeof(V) == 4 ? kMinBlocksExact
                                                                      : kMinBlocksExactBig)
    persistent_levels_kernel_x(const LevelLaunch a, const PersistPlan p) {
  persistent_body<V, LP1, KP1MAX, TRAIN, WT, CX>(a, p);
}

size_t persist_smem(const LevelLaunch& L, const PersistPlan* P, bool generic, size_t vsz) {
  size_t s = kGroup * sizeof(uint64_t) * (L.AW + (L.training ? L.W : 0));  // targets
  s += (size_t)L.C * kGroup * vsz;                                          // merge column
  if (generic) s += (size_t)kWarps * L.C * kGroup * vsz;
  if (P && P->stage) {
    // one old chunk: bitset rows, records, dp rows (+ alignment slack)
    const size_t n = (size_t)max(P->chunk_len0, P->chunk_len1);
    s += 16 + n * L.AW * 8 + n * sizeof(SrcRec) + n * L.C * vsz + 32;
  }
  return s;
}

template <typename V, int LP1, int KP1MAX, bool TRAIN, int WT = 0, bool CX = false>
void run_variant(const LevelLaunch& L, const PersistPlan* P, cudaStream_t st, PersistInfo* info) {
  const size_t smem = persist_smem(L, P, LP1 == 0, sizeof(V));
  void (*kern)(const LevelLaunch, const PersistPlan);
  if constexpr (CX) kern = persistent_levels_kernel_x<V, LP1, KP1MAX, TRAIN, WT, CX>;
  else kern = persistent_levels_kernel<V, LP1, KP1MAX, TRAIN, WT, CX>;
  // the attribute is per device context: set it on every call (cheap), and
  // report 0 resident CTAs when the shared memory cannot fit at all (the
  // host then falls back to the per-level driver)
  int dev = 0, sms = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  int per_sm = 0;
  if (smem <= (size_t)optin &&
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
          cudaSuccess &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTileTargets, smem) !=
          cudaSuccess)
    per_sm = 0;
  cudaGetLastError();  // a failed query must not poison the next launch check
  const int full = per_sm * sms;
  info->per_sm = per_sm;
  if (info->query_only) {
    info->blocks = full;
    return;
  }
  if (full < 1) {
    info->blocks = 0;
    info->launch_error = (int)cudaErrorInvalidConfiguration;
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

}  // namespace

// Kernel variants, compiled in separate translation units (persistent_v*.cu)
// so nvcc builds them in parallel.  dispatch_exact_*: the int32 exact-word /
// exact-cell and small-W register variants (false: none applies);
// dispatch_general_*: register cells by (L+1, K+1) bound, else generic.
#define DSG_PV_DECL(V, T)                                                                     \
  bool dispatch_exact_##V##_##T(const LevelLaunch& L, const PersistPlan* P, cudaStream_t st,  \
                                PersistInfo* info);                                           \
  void dispatch_general_##V##_##T(const LevelLaunch& L, const PersistPlan* P, cudaStream_t st, \
                                  PersistInfo* info);
DSG_PV_DECL(i32, inf)
DSG_PV_DECL(i32, train)
DSG_PV_DECL(i64, inf)
DSG_PV_DECL(i64, train)
#undef DSG_PV_DECL

}  // namespace dsg
