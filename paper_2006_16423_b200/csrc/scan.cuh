// scan.cuh — the fused K2+K3+K4 pair scan shared by both level drivers.
//
// Replaces the reference's per-target DFS over sub-ideals
// (walk_subideals + apply_candidate, /root/reference/proj/src/dp_solver.cpp:
// 197-317) with a dense scan that needs no hash lookups and no allocation:
//
//   * K2 (pair enumeration): I' ⊆ I is a W-word AND-NOT test of the source
//     bitset against the target bitset held in shared memory;
//   * K3 (block cost): prefix differences from the 64-byte source record +
//     the source-frontier walk of describe.cu (two 64-bit masks per chunk
//     of <= 64 producers), see acc_block_cost;
//   * K4 (min-max): per cell max(dp[I'][k-1][l], acc) and
//     max(dp[I'][k][l-1], cpu) with a strict-< update; the argmin is
//     2*I' + (cpu block), so "smallest (value, arg)" is a total order and the
//     result does not depend on how sources are split across lanes, warps,
//     CTAs or GPUs.
//
// Template knobs: V = int32_t/int64_t fixed point; LP1 = L+1 and KP1MAX =
// max K+1 for register-resident cells (LP1 == 0: generic shared-memory
// cells); TS = stride of the target column in shared memory (32/128 when
// lanes own targets, 1 when all lanes share one target); UNIFORM = all lanes
// walk the same sources (enables the warp-wide early skip).
#pragma once

#include <climits>
#include <cstdint>

#include "dsg_device.cuh"
#include "dsg_internal.h"

namespace dsg {
namespace scan {

// DSG_PAIR_STATS (a separate diagnostic build): where the nested pairs go
#ifdef DSG_PAIR_STATS
#define DSG_STAT(a, k, n) atomicAdd((a).stats + (k), (unsigned long long)(n))
#else
#define DSG_STAT(a, k, n) ((void)0)
#endif

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// A source dp row cell: rows finished by other CTAs inside the persistent
// kernel are read at L2 (ld.global.cg: never a stale L1 line, so the
// dependency wait needs no L1 invalidation); staged rows come from shared
// memory.
template <bool SMEM, typename V>
__device__ __forceinline__ V ld_row(const V* p) {
  if constexpr (SMEM) return *p;
  else return __ldcg(p);
}

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

__device__ __forceinline__ SrcRec load_rec(const SrcRec* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  int4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2), d = __ldg(q + 3);
  SrcRec r;
  r.cpu = (int64_t)(((uint64_t)(uint32_t)a.y << 32) | (uint32_t)a.x);
  r.acc = (int64_t)(((uint64_t)(uint32_t)a.w << 32) | (uint32_t)a.z);
  r.mem = (int64_t)(((uint64_t)(uint32_t)b.y << 32) | (uint32_t)b.x);
  r.unsup = b.z;
  r.n_chunks = b.w;
  r.chunk0 = c.x;
  r.n_f = c.y;
  r.n_n = c.z;
  r.off_f = c.w;
  r.off_n = d.x;
  r.pad = d.y;
  r.infmask = ((uint64_t)(uint32_t)d.w << 32) | (uint32_t)d.z;
  return r;
}

// The same record from shared memory (staged chunks, plain loads).
__device__ __forceinline__ SrcRec load_rec_s(const SrcRec* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  const int4 a = q[0], b = q[1], c = q[2], d = q[3];
  SrcRec r;
  r.cpu = (int64_t)(((uint64_t)(uint32_t)a.y << 32) | (uint32_t)a.x);
  r.acc = (int64_t)(((uint64_t)(uint32_t)a.w << 32) | (uint32_t)a.z);
  r.mem = (int64_t)(((uint64_t)(uint32_t)b.y << 32) | (uint32_t)b.x);
  r.unsup = b.z;
  r.n_chunks = b.w;
  r.chunk0 = c.x;
  r.n_f = c.y;
  r.n_n = c.z;
  r.off_f = c.w;
  r.off_n = d.x;
  r.pad = d.y;
  r.infmask = ((uint64_t)(uint32_t)d.w << 32) | (uint32_t)d.z;
  return r;
}

// A chunk's source rows staged in shared memory (mode-0 old chunks): bitset
// rows (pitch AW), records and dp rows of ordinals [base, base + n).
template <typename V>
struct SrcView {
  const uint64_t* bits;
  const SrcRec* rec;
  const V* dp;
  int64_t base;
};

// General backward-contiguity gate (is_contiguous over reachability_within
// of the backward part, graph.cpp:349-363), used when the fast up-set test
// does not apply.  tA: the target column (stride TS).
template <int TS>
__device__ bool bw_contiguous(const LevelLaunch& a, const uint64_t* tA,
                              const uint64_t* __restrict__ sA) {
  const int W = a.W;
  uint64_t rf[kMaxWords], rt[kMaxWords], B[kMaxWords];
  bool any = false;
  for (int w = 0; w < W; ++w) {
    B[w] = tA[w * TS] & ~sA[w] & a.bwset[w];
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

// One frontier chunk: hit = producers with an upper neighbour inside the
// target, miss = producers with an upper neighbour outside it.
template <typename V, int TS>
__device__ __forceinline__ void frontier_chunk(const LevelLaunch& a, int n_f, int n_n, int off_f,
                                               int off_n, uint64_t infm, const uint64_t* tA,
                                               V& cin, V& csub, bool& cin_inf, int& cout_inf) {
  const NItem* __restrict__ nitems = a.nitems;
  const V* __restrict__ fpool = (const V*)a.fpool;
  uint64_t hit = 0, miss = 0;
  for (int i = 0; i < n_n; ++i) {
    const uint4 it = __ldg(reinterpret_cast<const uint4*>(nitems + off_n + i));
    const uint64_t pm = ((uint64_t)it.w << 32) | it.z;
    const bool in = (tA[it.x * TS] >> it.y) & 1ull;
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

template <typename V>
struct Target {
  V cpu, acc, mem, fw;
  int un, fwi;
  bool up, active;
  int64_t t, tl, l_lo, l_hi;
};

// Scalars of target t (tl = index within its level).
template <typename V, bool TRAIN>
__device__ __forceinline__ Target<V> target_scalars(const LevelLaunch& a, int64_t t, int64_t tl,
                                                    bool active) {
  Target<V> x;
  x.tl = tl;
  x.active = active;
  x.t = t;
  x.cpu = __ldg((const V*)a.pfx_cpu + t);
  x.acc = __ldg((const V*)a.pfx_acc + t);
  x.mem = __ldg((const V*)a.pfx_mem + t);
  x.fw = __ldg((const V*)a.fw + t);
  x.un = __ldg(a.unsup + t);
  x.fwi = __ldg(a.fwinf + t);
  x.up = TRAIN ? (__ldg(a.upset + t) != 0) : true;
  x.l_lo = TRAIN ? __ldg(a.l_off + t) : 0;
  x.l_hi = TRAIN ? __ldg(a.l_off + t + 1) : 0;
  return x;
}

// Thread `lane` of a group of TS targets of [t_lo, t_hi): scalars, and (if
// stage) its target / interior bitsets into its shared-memory column.
template <typename V, bool TRAIN, int TS>
__device__ __forceinline__ Target<V> load_target(const LevelLaunch& a, int64_t t_lo, int64_t t_hi,
                                                 int64_t grp, int lane, uint64_t* colA,
                                                 uint64_t* colInt, bool stage = true) {
  const int W = a.W;
  const int64_t tl = grp * TS + lane;
  const bool active = t_lo + tl < t_hi;
  const int64_t t = active ? t_lo + tl : t_lo;
  if (stage) {
    for (int w = 0; w < a.AW; ++w) colA[w * TS] = active ? __ldg(a.abits + (size_t)t * a.AW + w) : 0ull;
    for (int w = 0; w < W; ++w) {
      if (TRAIN) colInt[w * TS] = active ? __ldg(a.intbits + (size_t)t * W + w) : 0ull;
    }
  }
  return target_scalars<V, TRAIN>(a, t, tl, active);
}

// Block cost of B = A(t) \ A(s) on an accelerator (BlockTracker::acc_load,
// dp_solver.cpp:90-97), given the prefix difference proc; INF if infeasible.
//   comm_out(B) = W(F(A)) - W({u in F(A') : succ(u)\A' ⊄ A})
//                 + W(P'(A') ∩ Int(A))                         [training]
//   comm_in(B)  = W({u in F(A') : (succ(u)\A') ∩ A ≠ ∅})
//                 + W({u in L(A) : succ(u) ∩ A ⊄ A'})          [training]
template <typename V, bool TRAIN, int TS>
__device__ __forceinline__ V acc_block_cost(const LevelLaunch& a, int64_t s, const SrcRec& r,
                                            V proc, const Target<V>& x, const uint64_t* tA,
                                            const uint64_t* tInt, const uint64_t* sAs = nullptr) {
  constexpr V INF = VTraits<V>::INF;
  V cin = 0, csub = 0;
  bool cin_inf = false;
  int cout_inf = x.fwi;
  if (r.n_chunks > 0)
    frontier_chunk<V, TS>(a, r.n_f, r.n_n, r.off_f, r.off_n, r.infmask, tA, cin, csub, cin_inf,
                          cout_inf);
  for (int c = 1; c < r.n_chunks; ++c) {
    const FChunk* ch = a.chunks + r.chunk0 + c;
    frontier_chunk<V, TS>(a, __ldg(&ch->n_f), __ldg(&ch->n_n), __ldg(&ch->off_f),
                          __ldg(&ch->off_n), __ldg(&ch->infmask), tA, cin, csub, cin_inf, cout_inf);
  }
  V cout = x.fw - csub;
  if (TRAIN) {
    const int64_t p0 = __ldg(a.p_off + s), p1 = __ldg(a.p_off + s + 1);
    for (int64_t p = p0; p < p1; ++p) {
      const PItem* pi = a.pitems + p;
      const uint32_t word = __ldg(&pi->word), bit = __ldg(&pi->bit);
      const bool in = (tInt[word * TS] >> bit) & 1ull;
      cout += in ? (V)__ldg(&pi->weight) : (V)0;
      cout_inf += (in && __ldg(&pi->inf)) ? 1 : 0;
    }
    // the source's bitset row: staged in shared memory when the chunk is
    const uint64_t* sA = sAs ? sAs : a.abits + (size_t)s * a.AW;
    for (int64_t e = x.l_lo; e < x.l_hi; ++e) {
      const LEntry le = a.lentries[e];
      bool charged = false;
      for (int i = 0; i < le.n_items; ++i) {
        const MaskItem mi = a.litems[le.off_items + i];
        charged |= (mi.mask & ~(sAs ? sA[mi.word] : __ldg(sA + mi.word))) != 0ull;
      }
      cin += charged ? (V)le.weight : (V)0;
      cin_inf |= charged && le.inf;
    }
  }
  if (cin_inf || cout_inf > 0) return INF;
  return combine<V>(cin, proc, cout, a.interleave);
}

struct AlwaysNeeded {
  template <typename V>
  __device__ __forceinline__ bool operator()(V) const {
    return true;
  }
};

// K2+K3 for one (target, source) pair: false when I' ⊄ I (not a
// transition) — *counted* is set when it is a transition at all (the
// reference counts gated training pairs too) and *gated* when the training
// backward gate rejects the block.  On success: accelerator load (INF if
// infeasible), CPU load, block memory.
//
// need(proc): whether an accelerator load >= proc could still improve a
// cell.  acc(B) >= proc(B) in every interleaving mode (the comm terms are
// non-negative, graph.cpp:457-467), so when it cannot the frontier walk is
// skipped (by the whole warp when no lane needs it) and acc = INF — the
// cell minima are unchanged.
template <typename V, bool TRAIN, int TS, class Need = AlwaysNeeded, bool STAGED = false>
__device__ __forceinline__ bool pair_cost(const LevelLaunch& a, const Target<V>& x, int64_t s,
                                          const uint64_t* tA, const uint64_t* tInt, bool& gated,
                                          V& acc, V& cpu, V& mem_blk, Need need = Need(),
                                          const SrcRec* rs = nullptr,
                                          const uint64_t* sAs = nullptr) {
  constexpr V INF = VTraits<V>::INF;
  const SrcRec r = STAGED ? load_rec_s(rs) : load_rec(a.srec + s);
  gated = false;
  if (TRAIN && a.has_bw) {
    const uint64_t* sA = sAs ? sAs : a.abits + (size_t)s * a.AW;
    if (!(a.fastgate && x.up && __ldg(a.upset + s)) && !bw_contiguous<TS>(a, tA, sA)) {
      gated = true;
      return true;
    }
  }
  cpu = x.cpu - (V)r.cpu;
  mem_blk = (V)(x.mem - (V)r.mem);
  acc = INF;
  bool acc_ok = a.K > 0 && (x.un - r.unsup) == 0;
  if (acc_ok && a.memcheck) acc_ok = !(mem_blk > (V)a.mlim);
  const V proc = (V)(x.acc - (V)r.acc);
  if (acc_ok && need(proc)) {
    acc = acc_block_cost<V, TRAIN, TS>(a, s, r, proc, x, tA, tInt, sAs);
    DSG_STAT(a, 2, 1);
  }
  return true;
}

// replicated_load (dp_solver.cpp:100-108) for r >= 2 on exactly scaled values
// Every value carries the factor S = lcm(1..K)·|b_num| (capi.cu prepare), so
// mem_blk / |b_num| and then / rr are exact; dividing before multiplying keeps
// every intermediate <= the final sync term, which the host's value-width
// bound covers (multiplying by (rr-1)·b_den first can wrap the 32-bit path).
template <typename V>
__device__ __forceinline__ V replicated(const LevelLaunch& a, V acc, V mem_blk, int rr) {
  const V divided = acc / (V)rr;
  const V sync = (V)a.repl_sign * (((mem_blk / (V)a.repl_bn) / (V)rr) * (V)(rr - 1) * (V)a.repl_bd);
  return a.repl_combine == 0 ? (V)(divided + sync) : vmax(divided, sync);
}

// K4 for one nested, ungated pair: cell = min(cell, max(dp[I'][k-1][l],
// acc)) and min(cell, max(dp[I'][k][l-1], cpu)).  row: the source row's
// cells 0..CMAX-2 in registers (register cells); sdp: the row in memory
// (generic cells, replication).
template <typename V, int LP1, int KP1MAX, int CS, bool CX, bool SMEM = false>
__device__ __forceinline__ void k4_update(const LevelLaunch& a, const V* sdp, const V* row, V acc,
                                          V cpu, V mem_blk, V* best, V* colv) {
  constexpr V INF = VTraits<V>::INF;
  constexpr bool kGeneric = LP1 == 0;
  constexpr int CMAX = kGeneric ? 1 : LP1 * KP1MAX;
  const int C = CX ? CMAX : a.C;
  if (kGeneric && a.repl && acc != INF) {
    const int lp1 = a.L + 1;
    for (int rr = 1; rr <= a.K; ++rr) {
      const V load = rr == 1 ? acc : replicated<V>(a, acc, mem_blk, rr);
      for (int k = rr; k <= a.K; ++k)
        for (int l = 0; l <= a.L; ++l) {
          const int c = k * lp1 + l;
          colv[c * CS] = min(colv[c * CS], vmax(ld_row<SMEM>(sdp + c - rr * lp1), load));
        }
    }
    acc = INF;  // accelerator candidates done; the CPU ones below
  }
  if (!kGeneric) {
#pragma unroll
    for (int c = 0; c < CMAX; ++c) {
      const int k = c / (LP1 ? LP1 : 1);
      const int l = c % (LP1 ? LP1 : 1);
      if (c < C) {
        V b = best[c];
        if (k >= 1) b = min(b, vmax(row[c - LP1], acc));
        if (l >= 1) b = min(b, vmax(row[c - 1], cpu));
        best[c] = b;
      }
    }
  } else {
    // generic cells: batches of 8 so the source-row loads are all in
    // flight before the shared-memory read-modify-writes
    const int lp1 = a.L + 1;
    constexpr int B = 8;
    for (int c0 = 0; c0 < C; c0 += B) {
      V va[B], vc[B];
#pragma unroll
      for (int i = 0; i < B; ++i) {
        const int c = c0 + i;
        va[i] = (c < C && c >= lp1) ? ld_row<SMEM>(sdp + c - lp1) : INF;
        vc[i] = (c < C && (c % lp1) != 0) ? ld_row<SMEM>(sdp + c - 1) : INF;
      }
#pragma unroll
      for (int i = 0; i < B; ++i) {
        const int c = c0 + i;
        if (c < C) colv[c * CS] = min(colv[c * CS], min(vmax(va[i], acc), vmax(vc[i], cpu)));
      }
    }
  }
}

// Scan sources s0, s0+step, ... < s1 for target x: the fused K2+K3+K4 loop.
// The K4 update is value-only — cell = min(cell, max(dp[I'][k-1][l], acc))
// and min(cell, max(dp[I'][k][l-1], cpu)), two IMNMX per candidate; the
// argmin is recovered exactly for the ≤ K+L cells of the optimal path during
// traceback (traceback_search).  Cells live in registers (LP1 > 0) or in a
// shared-memory column colv with stride CS (LP1 == 0: large (K+1)(L+1),
// replication).  Source dp rows are plain (coherent) loads: inside the
// persistent kernel other CTAs wrote them after this kernel started.
//
// WT > 0: W <= WT: the subset test is fully unrolled (WT/2 predicated
// 16-byte source loads, one LOP3 per word against the shared target column).
// CX: C == LP1 * KP1MAX exactly (no per-cell predicates); with CX, the
// padded row length a.AW == WT exactly as well (no per-word predicates).
// PF > 0: prefetch (L1) the rows of the source PF steps ahead — pays off
// when each thread walks its own sources (lanes own sources), not when the
// warp shares them.
template <typename V, int LP1, int KP1MAX, bool TRAIN, int TS, bool UNIFORM, int CS, int WT = 0,
          bool CX = false, int PF = 0, bool STAGED = false>
__device__ __forceinline__ unsigned scan_sources(const LevelLaunch& a, const Target<V>& x,
                                                 int64_t s0, int64_t s1, int step,
                                                 const uint64_t* tA, const uint64_t* tInt, V* best,
                                                 V* colv, SrcView<V> sv = SrcView<V>{},
                                                 const void* dpo = nullptr) {
  constexpr V INF = VTraits<V>::INF;
  constexpr bool kGeneric = LP1 == 0;
  constexpr int CMAX = kGeneric ? 1 : LP1 * KP1MAX;
  constexpr V NEG = (V)(-INF - 1);
  const int W = (CX && WT > 0) ? WT : a.W;  // exact: W rounded up, pad word 0
  const int AWp = (CX && WT > 0) ? WT : a.AW;  // row pitch (a compile-time constant when exact)
  const int C = CX ? CMAX : a.C;
  // dpo: the dp replica this CTA reads (a virtual shard's own table)
  const V* dp = (const V*)(dpo ? dpo : a.dp);
  unsigned nested_cnt = 0;
  // L == 0 (accelerator cells only): a pair can change a cell only through
  // max(dp[I'][k-1], acc) < best[k], and acc >= proc, so it is a candidate
  // only if the block is supported, fits in memory and proc < max_k best[k].
  // Everything else — most nested pairs of a memory-bound DP — skips the row
  // loads, the pruning test and the min-max update (the minima are unchanged,
  // so results stay bit-identical).  maxbest only shrinks; it is refreshed
  // after every update.
  constexpr bool kAccOnly = LP1 == 1;
  V maxbest = NEG;
  if constexpr (kAccOnly) {
#pragma unroll
    for (int c = 1; c < CMAX; ++c)
      if (c < C) maxbest = vmax(maxbest, best[c]);
  }
  for (int64_t s = s0; s < s1; s += step) {
    if (PF > 0 && s + PF * step < s1) {
      // pull a later source's rows into L1 while this one is evaluated
      const int64_t sn = s + PF * step;
      prefetch_l1(a.abits + (size_t)sn * AWp);
      prefetch_l1(a.srec + sn);
      prefetch_l1((const V*)a.dp + (size_t)sn * C);
    }
    // K2: I' ⊆ I
    // 16-byte source words (rows padded to even length, pad word 0); the
    // target's pad column is never read past W
    const ulonglong2* __restrict__ sA2 = reinterpret_cast<const ulonglong2*>(
        STAGED ? sv.bits + (size_t)(s - sv.base) * AWp : a.abits + (size_t)s * AWp);
    uint64_t stray = 0;
    if constexpr (WT > 0) {
#pragma unroll
      for (int j = 0; j < WT / 2; ++j) {
        if (2 * j < W) {
          const ulonglong2 v = STAGED ? sA2[j] : __ldg(sA2 + j);
          stray |= v.x & ~tA[2 * j * TS];
          if (2 * j + 1 < W) stray |= v.y & ~tA[(2 * j + 1) * TS];
        }
      }
    } else {
#pragma unroll 4
      for (int w = 0; w < W; w += 2) {
        const ulonglong2 v = STAGED ? sA2[w >> 1] : __ldg(sA2 + (w >> 1));
        stray |= v.x & ~tA[w * TS];
        if (w + 1 < W) stray |= v.y & ~tA[(w + 1) * TS];
      }
    }
    const bool nested = x.active && stray == 0ull;
    if (UNIFORM && !__any_sync(0xffffffffu, nested)) continue;
    bool cand = true;
    if constexpr (kAccOnly) {
      // the first 32 bytes of the source record: cpu, acc, mem, unsup
      // (every lane evaluates it, so the vote below is warp-uniform)
      const int4* q = reinterpret_cast<const int4*>(STAGED ? sv.rec + (s - sv.base) : a.srec + s);
      const int4 r0 = STAGED ? q[0] : __ldg(q), r1 = STAGED ? q[1] : __ldg(q + 1);
      const V racc = (V)(int64_t)(((uint64_t)(uint32_t)r0.w << 32) | (uint32_t)r0.z);
      const V rmem = (V)(int64_t)(((uint64_t)(uint32_t)r1.y << 32) | (uint32_t)r1.x);
      cand = nested && a.K > 0 && (x.un - r1.z) == 0 && (V)(x.acc - racc) < maxbest;
      if (a.memcheck) cand = cand && !((V)(x.mem - rmem) > (V)a.mlim);
      if (UNIFORM && !__any_sync(0xffffffffu, cand)) {
        nested_cnt += nested ? 1u : 0u;
        if (nested) DSG_STAT(a, 1, 1);
        continue;
      }
    }
    if (!nested) continue;
    ++nested_cnt;
    if (!cand) {
      DSG_STAT(a, 1, 1);
      continue;
    }
    bool gated;
    V acc, cpu, mem_blk;
    const V* sdp = STAGED ? sv.dp + (size_t)(s - sv.base) * C : dp + (size_t)s * C;
    // the source row cells the update reads (indices <= C-2), loaded once
    V row[CMAX > 1 ? CMAX - 1 : 1];
    if constexpr (!kGeneric) {
#pragma unroll
      for (int c = 0; c + 1 < CMAX; ++c) row[c] = (c + 1 < C) ? ld_row<STAGED>(sdp + c) : INF;
      // prune: the accelerator cost matters only if max(dp[I'][k-1][l], proc)
      // beats the running minimum of some cell, i.e. proc < thr
      auto need = [&](V proc) {
        V thr = NEG;
#pragma unroll
        for (int c = LP1; c < CMAX; ++c)
          if (c < C) thr = vmax(thr, row[c - LP1] < best[c] ? best[c] : NEG);
        return proc < thr;
      };
      pair_cost<V, TRAIN, TS, decltype(need), STAGED>(
          a, x, s, tA, tInt, gated, acc, cpu, mem_blk, need, sv.rec + (s - sv.base),
          STAGED && TRAIN ? sv.bits + (size_t)(s - sv.base) * AWp : nullptr);
    } else {
      pair_cost<V, TRAIN, TS, AlwaysNeeded, STAGED>(
          a, x, s, tA, tInt, gated, acc, cpu, mem_blk, AlwaysNeeded(), sv.rec + (s - sv.base),
          STAGED && TRAIN ? sv.bits + (size_t)(s - sv.base) * AWp : nullptr);
    }
    if (gated) continue;
    DSG_STAT(a, 3, 1);
    k4_update<V, LP1, KP1MAX, CS, CX, STAGED>(a, sdp, row, acc, cpu, mem_blk, best, colv);
    if constexpr (kAccOnly) {
      maxbest = NEG;
#pragma unroll
      for (int c = 1; c < CMAX; ++c)
        if (c < C) maxbest = vmax(maxbest, best[c]);
    }
  }
  return nested_cnt;
}

// Chunk-level liveness of one lane's target against the sources [s0, s1):
// with the block maxima of the source prefix sums (describe.cu
// chunk_max_kernel), the smallest block any source of the chunk can give is
// proc >= x.acc - max acc, mem >= x.mem - max mem, cpu >= x.cpu - max cpu.
// If even those cannot pass the per-pair tests of scan_sources — memory over
// the limit or proc above every accelerator cell's running minimum, and cpu
// above every CPU cell's — no pair of the chunk can change a cell of this
// target (acc(B) >= proc(B), as for the per-pair pruning).
template <typename V, int LP1, int CMAX>
__device__ __forceinline__ bool chunk_live(const LevelLaunch& a, const Target<V>& x, const V* best,
                                           int64_t s0, int64_t s1, int C) {
  constexpr V INF = VTraits<V>::INF;
  constexpr V NEG = (V)(-INF - 1);
  if (!x.active) return false;
  int64_t ma = LLONG_MIN, mm = LLONG_MIN, mc = LLONG_MIN;
  for (int64_t b = s0 / kChunkMaxLen; b <= (s1 - 1) / kChunkMaxLen; ++b) {
    const longlong2 m0 = __ldg(reinterpret_cast<const longlong2*>(a.cmax) + 2 * b);
    const long long m2 = __ldg(reinterpret_cast<const long long*>(a.cmax) + 4 * b + 2);
    ma = max(ma, (int64_t)m0.x);
    mm = max(mm, (int64_t)m0.y);
    mc = max(mc, (int64_t)m2);
  }
  V mb_acc = NEG, mb_cpu = NEG;
#pragma unroll
  for (int c = 0; c < CMAX; ++c) {
    if (c < C) {
      if (c >= LP1) mb_acc = vmax(mb_acc, best[c]);
      if (LP1 > 1 && (c % LP1) != 0) mb_cpu = vmax(mb_cpu, best[c]);
    }
  }
  bool acc_live = a.K > 0 && (V)(x.acc - (V)ma) < mb_acc;
  if (a.memcheck) acc_live = acc_live && !((V)(x.mem - (V)mm) > (V)a.mlim);
  const bool cpu_live = LP1 > 1 && (V)(x.cpu - (V)mc) < mb_cpu;
  return acc_live || cpu_live;
}

// Count-only scan for a chunk no pair of which can change a cell: the K2
// subset test alone (the pairs still count as transitions, dp_solver.cpp:
// 256-317 visits them).  Target words in registers when W is exact.
template <int TS, int WT, bool CX, bool STAGED>
__device__ __forceinline__ unsigned count_nested(const LevelLaunch& a, bool active, int64_t s0,
                                                 int64_t s1, int step, const uint64_t* tA,
                                                 const uint64_t* sbits, int64_t sbase) {
  unsigned n = 0;
  if (!active) return 0;
  if constexpr (CX && WT > 0) {
    uint64_t tw[WT];
#pragma unroll
    for (int j = 0; j < WT; ++j) tw[j] = tA[j * TS];
    for (int64_t s = s0; s < s1; s += step) {
      const ulonglong2* sA2 = reinterpret_cast<const ulonglong2*>(
          STAGED ? sbits + (size_t)(s - sbase) * WT : a.abits + (size_t)s * WT);
      uint64_t stray = 0;
#pragma unroll
      for (int j = 0; j < WT / 2; ++j) {
        const ulonglong2 v = STAGED ? sA2[j] : __ldg(sA2 + j);
        stray |= (v.x & ~tw[2 * j]) | (v.y & ~tw[2 * j + 1]);
      }
      n += stray == 0ull ? 1u : 0u;
    }
  } else {
    const int W = a.W, AW = a.AW;
    for (int64_t s = s0; s < s1; s += step) {
      const uint64_t* sA = STAGED ? sbits + (size_t)(s - sbase) * AW : a.abits + (size_t)s * AW;
      uint64_t stray = 0;
      for (int w = 0; w < W; ++w) stray |= (STAGED ? sA[w] : __ldg(sA + w)) & ~tA[w * TS];
      n += stray == 0ull ? 1u : 0u;
    }
  }
  DSG_STAT(a, 0, n);
  return n;
}

// Split K2+K3 / K4 for items whose sources may not be final yet (mode 1,
// one source per thread): everything but the source's dp row is static, so
// the subset test and the block cost run BEFORE the dependency wait and only
// the row loads + the min-max update remain after it.  No pruning (it needs
// the row).
template <typename V>
struct PrePair {
  bool ok;  // nested and not gated
  bool nested;
  V acc, cpu, mem_blk;
};

template <typename V, bool TRAIN, int TS>
__device__ __forceinline__ PrePair<V> pre_pair(const LevelLaunch& a, const Target<V>& x, int64_t s,
                                               const uint64_t* tA, const uint64_t* tInt) {
  PrePair<V> q;
  q.ok = false;
  q.nested = false;
  q.acc = q.cpu = q.mem_blk = (V)0;
  const ulonglong2* __restrict__ sA2 =
      reinterpret_cast<const ulonglong2*>(a.abits + (size_t)s * a.AW);
  uint64_t stray = 0;
  for (int w = 0; w < a.W; w += 2) {
    const ulonglong2 v = __ldg(sA2 + (w >> 1));
    stray |= v.x & ~tA[w * TS];
    if (w + 1 < a.W) stray |= v.y & ~tA[(w + 1) * TS];
  }
  if (!x.active || stray != 0ull) return q;
  q.nested = true;
  bool gated;
  pair_cost<V, TRAIN, TS>(a, x, s, tA, tInt, gated, q.acc, q.cpu, q.mem_blk);
  q.ok = !gated;
  return q;
}

template <typename V, int LP1, int KP1MAX, int CS, bool CX, bool L1 = true>
__device__ __forceinline__ void post_pair(const LevelLaunch& a, const PrePair<V>& q, int64_t s,
                                          V* best, V* colv, const void* dpo) {
  constexpr V INF = VTraits<V>::INF;
  constexpr int CMAX = LP1 == 0 ? 1 : LP1 * KP1MAX;
  if (!q.ok) return;
  const int C = CX ? CMAX : a.C;
  const V* sdp = (const V*)dpo + (size_t)s * C;
  V row[CMAX > 1 ? CMAX - 1 : 1];
  if constexpr (LP1 != 0) {
#pragma unroll
    for (int c = 0; c + 1 < CMAX; ++c) row[c] = (c + 1 < C) ? ld_row<L1>(sdp + c) : INF;
  }
  // L1: plain loads, the caller's dependency wait acquired (L1 invalidated);
  // else L2 loads (ld.global.cg) after a wait without an acquire
  k4_update<V, LP1, KP1MAX, CS, CX, L1>(a, sdp, row, q.acc, q.cpu, q.mem_blk, best, colv);
}

template <typename V, int LP1, int KP1MAX, int CS>
__device__ __forceinline__ void init_cells(int C, V* best, V* colv) {
  constexpr V INF = VTraits<V>::INF;
  constexpr int CMAX = LP1 == 0 ? 1 : LP1 * KP1MAX;
#pragma unroll
  for (int c = 0; c < CMAX; ++c) best[c] = INF;
  if (LP1 == 0)
    for (int c = 0; c < C; ++c) colv[c * CS] = INF;
}

// lexicographic (value, arg) minimum
template <typename V>
__device__ __forceinline__ void vmin_arg(V& v, int32_t& g, V v2, int32_t g2) {
  if (v2 < v || (v2 == v && g2 < g)) {
    v = v2;
    g = g2;
  }
}

// monotone_pass, dp_solver.cpp:180-193 (in place, k then l ascending), on
// register cells with compile-time indices
template <typename V, int LP1, int CMAX>
__device__ __forceinline__ void monotone_regs(V* v, int C) {
#pragma unroll
  for (int c = 0; c < CMAX; ++c) {
    const int k = c / (LP1 ? LP1 : 1), l = c % (LP1 ? LP1 : 1);
    if (c < C) {
      if (k > 0) v[c] = min(v[c], v[c - (LP1 ? LP1 : 1)]);
      if (l > 0) v[c] = min(v[c], v[c - 1]);
    }
  }
}

// ... and on a strided shared-memory / global column
template <typename V>
__device__ __forceinline__ void monotone_strided(V* v, int stride, int K, int L) {
  const int lp1 = L + 1;
  for (int k = 0; k <= K; ++k) {
    for (int l = 0; l <= L; ++l) {
      const int c = k * lp1 + l;
      V cur = v[c * stride];
      if (k > 0) cur = min(cur, v[(c - lp1) * stride]);
      if (l > 0) cur = min(cur, v[(c - 1) * stride]);
      v[c * stride] = cur;
    }
  }
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// system scope: counters that peer GPUs bump over NVLink
__device__ __forceinline__ unsigned ld_relaxed_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

}  // namespace scan
}  // namespace dsg
