// enumerate.cu — K1: ideal-lattice enumeration on the device.
//
// Replaces enumerate_impl (/root/reference/proj/src/ideals.cpp:14-75): a
// breadth-first walk of the lattice by cardinality from the empty ideal,
// adding one eligible node (all in_all-predecessors inside, restricted to
// the universe, ideals.cpp:38-48) at a time, followed by the reference's
// ordering: size-major, lexicographic within a level (NodeSet::lex_less,
// graph.cpp:62-72).
//
// Two deduplication strategies produce the same level sets:
//   * canonical parent (default): J ∪ {v} is emitted only by the parent
//     whose removed node v is the largest-index maximal element of J ∪ {v},
//     so every ideal has exactly one parent and no dedup is needed;
//   * GPU hash set (DSG_FLAG_HASH_ENUM): every parent emits every child
//     into a candidate buffer; candidates are inserted into an
//     open-addressing table keyed by the bitset (FNV-1a, as NodeSet::hash,
//     graph.cpp:81-88) and only first-inserted copies survive.
// Both keep per-ideal "maximal" and "addable" masks so that a child is
// derived from its parent in O(W + deg) instead of a rescan.
//
// Levels are tiny compared with the DP (< 1 % of the work),
// so the level loop runs inside ONE persistent CTA with __syncthreads()
// between levels: no host round trip and no grid barrier per level.
#include <cooperative_groups.h>
#include <cooperative_groups/reduce.h>
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "dsg_device.cuh"
#include "dsg_internal.h"

namespace dsg {

namespace {

namespace cg = cooperative_groups;

// measured on C2 / C4 / C5 (tools/build_variant.py): 1024 beats 512 and 256
#ifndef DSG_ENUM_THREADS
#define DSG_ENUM_THREADS 1024
#endif
constexpr int kEnumThreads = DSG_ENUM_THREADS;

__device__ __forceinline__ uint64_t above_mask(int v, int w) {
  // bits with index > v inside word w
  int vw = v >> 6;
  if (w < vw) return 0ull;
  if (w > vw) return ~0ull;
  int b = v & 63;
  return b == 63 ? 0ull : (~0ull << (b + 1));
}

// Child J ∪ {v} of parent p: bits, maximal mask, addable mask.
__device__ void write_child(int W, int v, const uint64_t* __restrict__ pj,
                            const uint64_t* __restrict__ pm, const uint64_t* __restrict__ pa,
                            const uint64_t* __restrict__ pred_u,
                            const uint64_t* __restrict__ succ_u, uint64_t* cj, uint64_t* cm,
                            uint64_t* ca) {
  const uint64_t* pv = pred_u + (size_t)v * W;
  const uint64_t* sv = succ_u + (size_t)v * W;
  for (int w = 0; w < W; ++w) {
    uint64_t vb = (w == (v >> 6)) ? (1ull << (v & 63)) : 0ull;
    cj[w] = pj[w] | vb;
    cm[w] = (pm[w] & ~pv[w]) | vb;
    ca[w] = pa[w] & ~vb;
  }
  // successors of v that become addable: all their preds inside J ∪ {v}
  for (int w = 0; w < W; ++w) {
    uint64_t s = sv[w];
    while (s) {
      int b = __ffsll((long long)s) - 1;
      s &= s - 1;
      int x = (w << 6) | b;
      const uint64_t* px = pred_u + (size_t)x * W;
      bool ok = true;
      for (int k = 0; k < W && ok; ++k) ok = (px[k] & ~cj[k]) == 0ull;
      if (ok) ca[w] |= 1ull << b;
    }
  }
}

__device__ uint64_t fnv_hash(const uint64_t* s, int W) {
  uint64_t h = 1469598103934665603ull;
  for (int i = 0; i < W; ++i) {
    h ^= s[i];
    h *= 1099511628211ull;
  }
  return h;
}

struct EnumArgs {
  int W;
  int n;
  const uint64_t* pred_u;
  const uint64_t* succ_u;
  const uint8_t* in_universe;
  const int32_t* pu_off;
  const int32_t* pu_adj;
  const int32_t* su_off;
  const int32_t* su_adj;
  int n_pu, n_su;      // adjacency list lengths
  int32_t* spill_par;  // [cap] warp mode: accepted pairs beyond kAccCap
  int32_t* spill_v;
  int csr_in_smem;     // stage the adjacency in shared memory
  int warp_items;      // warp mode while parents x words <= this
  uint64_t* bits;      // [cap][W]
  uint64_t* maxm;      // [cap][W]
  uint64_t* addm;      // [cap][W]
  int32_t* level_of;   // [cap]
  int64_t cap;
  int64_t budget;
  int64_t* level_off;  // [n + 2]
  EnumStatus* status;
  // hash-set mode
  int hash_mode;
  uint64_t* cand_bits; // [cand_cap][W]  (also cand max/add follow)
  uint64_t* cand_maxm;
  uint64_t* cand_addm;
  int64_t cand_cap;
  int64_t* table;      // [table_cap] candidate index or -1
  int64_t table_cap;
  int cluster_ok;      // stop at the first level wider than wide_min (code 4)
  int64_t wide_min;    // levels above this go to the cluster (<= cta_cap(W))
  int resume;          // cluster kernel: continue from status->resume_*
};

// Resident modes: the frontier (parents and children, bits / maximal /
// addable words each) lives in shared memory — up to small_cap(W) ideals
// per level when warp 0 runs alone (tiny levels), up to cta_cap(W) when the
// whole CTA runs; accepted (parent, node) pairs beyond kAccCap spill to
// global scratch.
constexpr int kAccCap = 2048;

__host__ __device__ __forceinline__ int cta_cap(int W) {
  const int c = (144 * 1024) / (2 * 3 * W * (int)sizeof(uint64_t));
  return c < 4096 ? c : 4096;
}

__host__ __device__ __forceinline__ int small_cap(int W) {
  const int c = cta_cap(W);
  return c < 64 ? c : 64;
}

// frontier buffers [2][cta_cap][3W] u64, accepted pairs [2][kAccCap] i32,
// top maximal element [2][cta_cap] i32
__host__ __device__ __forceinline__ size_t enum_warp_bytes(int W) {
  return (size_t)2 * cta_cap(W) * 3 * W * sizeof(uint64_t) +
         (size_t)(kAccCap * 2 + 2 * cta_cap(W)) * sizeof(int32_t);
}

__host__ __device__ __forceinline__ size_t enum_csr_bytes(int n, int n_pu, int n_su) {
  return (size_t)(2 * (n + 1) + n_pu + n_su) * sizeof(int32_t);
}

// Universe adjacency (unique entries); staged in shared memory when it fits.
struct Adj {
  const int32_t* pu_off;
  const int32_t* pu_adj;
  const int32_t* su_off;
  const int32_t* su_adj;
};

__device__ __forceinline__ bool bit_of(const uint64_t* s, int u) {
  return (s[u >> 6] >> (u & 63)) & 1ull;
}

// Canonical-parent expansion of one level [lo, hi) (ideals.cpp:38-48
// restated as set algebra on the parent's masks):
//   canonical  ⇔ #(maximal ∩ above(v)) == #(pred(v) ∩ maximal ∩ above(v))
//   max(J∪v)   = (max(J) \ pred(v)) ∪ {v}
//   add(J∪v)   = (add(J) \ {v}) ∪ {y ∈ succ(v) : pred(y) ⊆ J ∪ {v}}
//
// Wide levels, the whole CTA in two phases (a barrier between): phase A,
// threads over (parent, word) pairs test the candidates of that word and
// record each canonical child (parent, node) at its slot; phase B, threads
// over (child, word) pairs build the child rows.  Parent rows are read
// from global memory (L1 after the first touch).
__device__ void expand_cta(const EnumArgs& a, const Adj& g, int64_t lo, int64_t hi, int level,
                           unsigned long long* s_next) {
  const int W = a.W;
  const int nt = blockDim.x;
  const int i0 = threadIdx.x / W, x0 = threadIdx.x % W, di = nt / W, dx = nt % W;
  const int64_t nP = hi - lo;
  // phase A
  for (int64_t i = i0, x = x0; i < nP;) {
    const size_t row = (size_t)(lo + i) * W;
    uint64_t cand = a.addm[row + x];
    if (cand) {
      const uint64_t* M = a.maxm + row;
      int upper = 0;  // maximal elements in the words above x
      for (int y = (int)x + 1; y < W; ++y) upper += __popcll(M[y]);
      const uint64_t mx = M[x];
      do {
        const int b = __ffsll((long long)cand) - 1;
        cand &= cand - 1;
        const int v = ((int)x << 6) | b;
        const int above = upper + __popcll(mx & above_mask(v, (int)x));
        if (above) {
          int covered = 0;
          const int p1 = g.pu_off[v + 1];
          for (int e = g.pu_off[v]; e < p1; ++e) {
            const int u = g.pu_adj[e];
            covered += (u > v && bit_of(M, u)) ? 1 : 0;
          }
          if (covered != above) continue;
        }
        const unsigned long long slot = atomicAdd(s_next, 1ull);
        if ((int64_t)slot >= a.cap) continue;
        a.spill_par[slot] = (int32_t)(lo + i);
        a.spill_v[slot] = v;
      } while (cand);
    }
    x += dx;
    i += di;
    if (x >= W) {
      x -= W;
      ++i;
    }
  }
  __syncthreads();
  const int64_t end = min((int64_t)*s_next, a.cap);
  // phase B
  for (int64_t k = i0, x = x0; hi + k < end;) {
    const int64_t slot = hi + k;
    const int64_t par = a.spill_par[slot];
    const int v = a.spill_v[slot];
    const uint64_t* J = a.bits + (size_t)par * W;
    const uint64_t bx = (v >> 6) == x ? 1ull << (v & 63) : 0ull;
    uint64_t m = a.maxm[(size_t)par * W + x];
    const int p1 = g.pu_off[v + 1];
    for (int e = g.pu_off[v]; e < p1; ++e) {
      const int u = g.pu_adj[e];
      if ((u >> 6) == x) m &= ~(1ull << (u & 63));
    }
    m |= bx;
    uint64_t ad = a.addm[(size_t)par * W + x] & ~bx;
    const int s1 = g.su_off[v + 1];
    for (int e = g.su_off[v]; e < s1; ++e) {
      const int y = g.su_adj[e];
      if ((y >> 6) != x) continue;
      bool ok = true;
      const int f1 = g.pu_off[y + 1];
      for (int f = g.pu_off[y]; f < f1 && ok; ++f) {
        const int u = g.pu_adj[f];
        ok = u == v || bit_of(J, u);
      }
      if (ok) ad |= 1ull << (y & 63);
    }
    a.bits[slot * W + x] = J[x] | bx;
    a.maxm[slot * W + x] = m;
    a.addm[slot * W + x] = ad;
    if (x == 0) a.level_of[slot] = level + 1;
    x += dx;
    k += di;
    if (x >= W) {
      x -= W;
      ++k;
    }
  }
}

// Wide levels (alternative): one thread per parent, masks in local memory.
__device__ void expand_thread(const EnumArgs& a, const Adj& g, int64_t lo, int64_t hi, int level,
                              unsigned long long* s_next) {
  const int W = a.W;
  for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
    uint64_t J[kMaxWords], M[kMaxWords], A[kMaxWords], T[kMaxWords];
    for (int w = 0; w < W; ++w) {
      J[w] = a.bits[(size_t)p * W + w];
      M[w] = a.maxm[(size_t)p * W + w];
      A[w] = a.addm[(size_t)p * W + w];
    }
    for (int w = 0; w < W; ++w) {
      uint64_t cand = A[w];
      while (cand) {
        const int b = __ffsll((long long)cand) - 1;
        cand &= cand - 1;
        const int v = (w << 6) | b;
        const int p0 = g.pu_off[v], p1 = g.pu_off[v + 1];
        int above = 0;
        for (int x = w; x < W; ++x) above += __popcll(M[x] & above_mask(v, x));
        if (above) {
          int covered = 0;
          for (int e = p0; e < p1; ++e) {
            const int u = g.pu_adj[e];
            covered += (u > v && bit_of(M, u)) ? 1 : 0;
          }
          if (covered != above) continue;
        }
        const unsigned long long slot = atomicAdd(s_next, 1ull);
        if ((int64_t)slot >= a.cap) continue;
        const uint64_t vb = 1ull << b;
        for (int x = 0; x < W; ++x) T[x] = M[x];
        for (int e = p0; e < p1; ++e) {
          const int u = g.pu_adj[e];
          T[u >> 6] &= ~(1ull << (u & 63));
        }
        T[w] |= vb;
        for (int x = 0; x < W; ++x) {
          a.bits[slot * W + x] = J[x] | (x == w ? vb : 0ull);
          a.maxm[slot * W + x] = T[x];
        }
        for (int x = 0; x < W; ++x) T[x] = A[x];
        T[w] &= ~vb;
        const int s1 = g.su_off[v + 1];
        for (int e = g.su_off[v]; e < s1; ++e) {
          const int y = g.su_adj[e];
          bool ok = true;
          const int f1 = g.pu_off[y + 1];
          for (int f = g.pu_off[y]; f < f1 && ok; ++f) {
            const int u = g.pu_adj[f];
            ok = u == v || bit_of(J, u);
          }
          if (ok) T[y >> 6] |= 1ull << (y & 63);
        }
        for (int x = 0; x < W; ++x) a.addm[slot * W + x] = T[x];
        a.level_of[slot] = level + 1;
      }
    }
  }
}

// Resident levels, run by a team — warp 0 alone (TEAM = 32, tiny levels,
// no CTA barrier) or the whole CTA (TEAM = kEnumThreads) — level after level
// while the frontier stays in shared memory, without an L2 round trip on the
// dependency chain.  Phase A: threads over (parent, word) find the canonical
// candidates; phase B: threads over (child, word) build the child rows into
// global memory and into the next shared frontier.  The canonical test walks
// the parent's maximal elements above v from the top (kept per cached ideal)
// while they are predecessors of v.  Returns after expanding a level whose
// successor does not qualify for this team; *s_next then holds the new end
// and (lo, hi, level) describe the level just expanded, exactly as after one
// CTA-wide step.  The adjacency lists must be staged in shared memory.
template <int TEAM>
__device__ __forceinline__ void team_sync() {
  if (TEAM == 32) __syncwarp();
  else __syncthreads();
}

template <int TEAM>
__device__ void expand_resident(const EnumArgs& a, int64_t* lo_io, int64_t* hi_io, int* level_io,
                                unsigned long long* s_next, uint64_t* smem, int* s_nc) {
  const int W = a.W;
  const int r = TEAM == 32 ? (threadIdx.x & 31) : threadIdx.x;
  const int cap_buf = cta_cap(W);
  const int cap = TEAM == 32 ? small_cap(W) : cap_buf;
  const int R = 3 * W;  // words per cached ideal: J | M | A
  uint64_t* par = smem;
  uint64_t* chi = smem + (size_t)cap_buf * R;
  int32_t* acc_i = reinterpret_cast<int32_t*>(smem + (size_t)2 * cap_buf * R);
  int32_t* acc_v = acc_i + kAccCap;
  int32_t* top_p = acc_v + kAccCap;
  int32_t* top_c = top_p + cap_buf;
  const int32_t* pu_off = reinterpret_cast<const int32_t*>(smem + enum_warp_bytes(W) / sizeof(uint64_t));
  const int32_t* su_off = pu_off + (a.n + 1);
  const int32_t* pu_adj = su_off + (a.n + 1);
  const int32_t* su_adj = pu_adj + a.n_pu;
  // thread items (i, x) over a [count][W] grid: start (r / W, r % W), step
  // TEAM = (di, dx)
  const int i0 = r / W, x0 = r % W, di = TEAM / W, dx = TEAM % W;
  int64_t lo = *lo_io, hi = *hi_io;
  int level = *level_io;
  // child counters, double-buffered by level parity: the next level's is
  // reset during this level's phase B, so a level costs two team barriers
  int par_nc = 0;
  {
    const int nP0 = (int)(hi - lo);
    if (r == 0) s_nc[0] = s_nc[1] = 0;
    for (int j = r; j < nP0; j += TEAM) top_p[j] = -1;
    team_sync<TEAM>();
    for (int i = i0, x = x0; i < nP0;) {
      const size_t src = (size_t)(lo + i) * W + x;
      const uint64_t m = a.maxm[src];
      par[(size_t)i * R + x] = a.bits[src];
      par[(size_t)i * R + W + x] = m;
      par[(size_t)i * R + 2 * W + x] = a.addm[src];
      if (m) atomicMax(&top_p[i], (x << 6) | (63 - __clzll((long long)m)));
      x += dx;
      i += di;
      if (x >= W) {
        x -= W;
        ++i;
      }
    }
    team_sync<TEAM>();
  }
  while (true) {
    if (TEAM == 32 && hi - lo == 1 && W <= 32) {
      // A level holding ONE ideal: each of its children is canonical (the
      // child's canonical parent has this level's size, so it is this
      // ideal).  While the ideal has exactly one addable node the next level
      // is that single child: walk such chains with one lane per bitset word
      // (registers, no phase barriers), then continue generically.
      const int w = r;
      uint64_t J = 0, M = 0, A = 0;
      if (w < W) {
        J = par[w];
        M = par[W + w];
        A = par[2 * W + w];
      }
      bool moved = false;
      while (true) {
        const unsigned cnt = __reduce_add_sync(0xffffffffu, (unsigned)__popcll(A));
        if (cnt != 1u || hi + 1 > a.budget || hi + 1 > a.cap) break;
        const unsigned has = __ballot_sync(0xffffffffu, A != 0ull);
        const int lw = __ffs((int)has) - 1;
        const uint64_t aw = __shfl_sync(0xffffffffu, A, lw);
        const int v = (lw << 6) | (__ffsll((long long)aw) - 1);
        const uint64_t bx = w == (v >> 6) ? 1ull << (v & 63) : 0ull;
        // max(J ∪ v) = (max(J) \ pred(v)) ∪ {v}; add = (add(J) \ {v}) ∪
        // {y ∈ succ(v) : pred(y) ⊆ J ∪ {v}}
        J |= bx;
        for (int e = pu_off[v], e1 = pu_off[v + 1]; e < e1; ++e) {
          const int u = pu_adj[e];
          if ((u >> 6) == w) M &= ~(1ull << (u & 63));
        }
        M |= bx;
        A &= ~bx;
        for (int e = su_off[v], e1 = su_off[v + 1]; e < e1; ++e) {
          const int y = su_adj[e];
          bool miss = false;
          for (int f = pu_off[y], f1 = pu_off[y + 1]; f < f1; ++f) {
            const int u = pu_adj[f];
            miss |= (u >> 6) == w && !((J >> (u & 63)) & 1ull);
          }
          if (!__any_sync(0xffffffffu, miss) && (y >> 6) == w) A |= 1ull << (y & 63);
        }
        const int64_t slot = hi;
        if (w < W) {
          a.bits[slot * W + w] = J;
          a.maxm[slot * W + w] = M;
          a.addm[slot * W + w] = A;
        }
        if (w == 0) {
          a.level_of[slot] = level + 1;
          a.level_off[level + 2] = hi + 1;
        }
        lo = hi;
        hi = hi + 1;
        ++level;
        moved = true;
      }
      if (moved) {
        // the generic step continues from this single ideal
        if (w < W) {
          par[w] = J;
          par[W + w] = M;
          par[2 * W + w] = A;
        }
        const int tb = M ? (w << 6) | (63 - __clzll((long long)M)) : -1;
        const int top = __reduce_max_sync(0xffffffffu, tb);
        if (w == 0) top_p[0] = top;
        __syncwarp();
      }
    }
    const int nP = (int)(hi - lo);
    int* nc = s_nc + par_nc;
    // phase A: canonical candidates
    for (int i = i0, x = x0; i < nP;) {
      uint64_t cand = par[(size_t)i * R + 2 * W + x];
      if (cand) {
        const uint64_t* M = par + (size_t)i * R + W;
        const int top = top_p[i];
        do {
          const int b = __ffsll((long long)cand) - 1;
          cand &= cand - 1;
          const int v = (x << 6) | b;
          // canonical <=> every maximal element of J above v is a
          // predecessor of v: (max(J) ∩ above(v)) \ pred(v) = ∅, word by
          // word up to the top maximal element's word
          bool canon = true;
          if (top > v) {
            const uint64_t* pv = a.pred_u + (size_t)v * W;
            for (int w = v >> 6; w <= (top >> 6); ++w) {
              if (M[w] & above_mask(v, w) & ~__ldg(pv + w)) {
                canon = false;
                break;
              }
            }
          }
          if (!canon) continue;
          const int k = atomicAdd(nc, 1);
          const int64_t slot = hi + k;
          if (k < kAccCap) {
            acc_i[k] = i;
            acc_v[k] = v;
          } else if (slot < a.cap) {
            a.spill_par[slot] = i;
            a.spill_v[slot] = v;
          }
        } while (cand);
      }
      x += dx;
      i += di;
      if (x >= W) {
        x -= W;
        ++i;
      }
    }
    for (int j = r; j < cap; j += TEAM) top_c[j] = -1;
    if (TEAM != 32) __threadfence_block();  // spills visible to the CTA
    team_sync<TEAM>();
    const int nC = *nc;
    if (r == 0) s_nc[par_nc ^ 1] = 0;  // read by everyone before the last barrier
    // phase B: child rows
    for (int k = i0, x = x0; k < nC;) {
      const int64_t slot = hi + k;
      if (slot >= a.cap) break;
      const int i = k < kAccCap ? acc_i[k] : a.spill_par[slot];
      const int v = k < kAccCap ? acc_v[k] : a.spill_v[slot];
      const uint64_t* J = par + (size_t)i * R;
      const uint64_t bx = (v >> 6) == x ? 1ull << (v & 63) : 0ull;
      uint64_t m = J[W + x];
      const int p1 = pu_off[v + 1];
      for (int e = pu_off[v]; e < p1; ++e) {
        const int u = pu_adj[e];
        if ((u >> 6) == x) m &= ~(1ull << (u & 63));
      }
      m |= bx;
      uint64_t ad = J[2 * W + x] & ~bx;
      const int s1 = su_off[v + 1];
      for (int e = su_off[v]; e < s1; ++e) {
        const int y = su_adj[e];
        if ((y >> 6) != x) continue;
        bool ok = true;
        const int f1 = pu_off[y + 1];
        for (int f = pu_off[y]; f < f1 && ok; ++f) {
          const int u = pu_adj[f];
          ok = u == v || bit_of(J, u);
        }
        if (ok) ad |= 1ull << (y & 63);
      }
      const uint64_t jb = J[x] | bx;
      a.bits[slot * W + x] = jb;
      a.maxm[slot * W + x] = m;
      a.addm[slot * W + x] = ad;
      if (k < cap) {
        chi[(size_t)k * R + x] = jb;
        chi[(size_t)k * R + W + x] = m;
        chi[(size_t)k * R + 2 * W + x] = ad;
        if (m) atomicMax(&top_c[k], (x << 6) | (63 - __clzll((long long)m)));
      }
      if (x == 0) a.level_of[slot] = level + 1;
      x += dx;
      k += di;
      if (x >= W) {
        x -= W;
        ++k;
      }
    }
    team_sync<TEAM>();  // child rows, top_c, the reset counter
    const int64_t new_hi = hi + nC;
    if (r == 0) *s_next = (unsigned long long)new_hi;  // read by the caller after its barrier
    par_nc ^= 1;
    // stay while the next level fits this team: warp mode for tiny levels,
    // CTA mode for the rest up to the shared-memory cap
    const bool tiny = (int64_t)nC * W <= a.warp_items && nC <= small_cap(W);
    // (the CTA stays on while the level fits its frontier — and, when the
    // cluster walk may take over, is not wider than wide_min)
    const bool fits = TEAM == 32 ? tiny
                                 : (nC <= cap && !tiny && (!a.cluster_ok || nC <= a.wide_min));
    if (nC == 0 || !fits || new_hi > a.budget || new_hi > a.cap) break;
    // advance without leaving the team (the CTA step's bookkeeping)
    lo = hi;
    hi = new_hi;
    ++level;
    if (r == 0) a.level_off[level + 1] = hi;
    uint64_t* t = par;
    par = chi;
    chi = t;
    int32_t* tt = top_p;
    top_p = top_c;
    top_c = tt;
  }
  *lo_io = lo;
  *hi_io = hi;
  *level_io = level;
}

__global__ void __launch_bounds__(kEnumThreads) enumerate_levels_kernel(EnumArgs a) {
  const int W = a.W;
  extern __shared__ uint64_t s_dyn[];
  __shared__ unsigned long long s_next;
  __shared__ unsigned long long s_cand;
  __shared__ int s_stop;
  __shared__ int s_nc[2];
  __shared__ int64_t s_lo, s_hi;
  __shared__ int s_level;
  const int tid = threadIdx.x;

  // adjacency: shared-memory copy behind the group staging when it fits
  Adj adj{a.pu_off, a.pu_adj, a.su_off, a.su_adj};
  if (a.csr_in_smem && !a.hash_mode) {
    int32_t* c = reinterpret_cast<int32_t*>(s_dyn + enum_warp_bytes(W) / sizeof(uint64_t));
    int32_t* pu_off = c;
    int32_t* su_off = pu_off + (a.n + 1);
    int32_t* pu_adj = su_off + (a.n + 1);
    int32_t* su_adj = pu_adj + a.n_pu;
    for (int i = tid; i <= a.n; i += blockDim.x) {
      pu_off[i] = a.pu_off[i];
      su_off[i] = a.su_off[i];
    }
    for (int i = tid; i < a.n_pu; i += blockDim.x) pu_adj[i] = a.pu_adj[i];
    for (int i = tid; i < a.n_su; i += blockDim.x) su_adj[i] = a.su_adj[i];
    adj = Adj{pu_off, pu_adj, su_off, su_adj};
  }

  // the empty ideal, ideals.cpp:23-24
  for (int w = tid; w < W; w += blockDim.x) {
    a.bits[w] = 0;
    a.maxm[w] = 0;
    a.addm[w] = 0;
  }
  __syncthreads();
  for (int v = tid; v < a.n; v += blockDim.x) {
    if (!a.in_universe[v]) continue;
    bool root = true;
    for (int w = 0; w < W; ++w) root &= a.pred_u[(size_t)v * W + w] == 0ull;
    if (root) atomicOr((unsigned long long*)&a.addm[v >> 6], 1ull << (v & 63));
  }
  if (tid == 0) {
    a.level_of[0] = 0;
    a.level_off[0] = 0;
    a.level_off[1] = 1;
    s_stop = 0;
  }
  __syncthreads();

  int64_t lo = 0, hi = 1;
  int level = 0;
  while (hi > lo) {
    if (tid == 0) {
      s_next = (unsigned long long)hi;
      s_cand = 0;
    }
    __syncthreads();
    if (!a.hash_mode) {
      const int64_t nP = hi - lo;
      if (a.csr_in_smem && nP <= small_cap(W) && nP * W <= a.warp_items) {
        if (tid < 32) {
          expand_resident<32>(a, &lo, &hi, &level, &s_next, s_dyn, s_nc);
          if (tid == 0) {
            s_lo = lo;
            s_hi = hi;
            s_level = level;
          }
        }
        __syncthreads();
        lo = s_lo;
        hi = s_hi;
        level = s_level;
      } else if (a.cluster_ok && nP > a.wide_min) {
        // a level wider than the shared frontier: the cluster kernel takes
        // over from here (launch_enumerate / capi.cu enumerate_device)
        if (tid == 0) {
          a.status->code = 4;
          a.status->resume_lo = lo;
          a.status->resume_hi = hi;
          a.status->resume_level = level;
          s_stop = 1;
        }
        __syncthreads();
        break;
      } else if (a.csr_in_smem && nP <= cta_cap(W)) {
        // every thread runs the same control flow on shared counters, so
        // (lo, hi, level) stay identical across the CTA
        expand_resident<kEnumThreads>(a, &lo, &hi, &level, &s_next, s_dyn, s_nc);
      } else {
        expand_cta(a, adj, lo, hi, level, &s_next);
      }
    } else {
      // phase 1: every parent writes every child into the candidate buffer
      for (int64_t p = lo + tid; p < hi; p += blockDim.x) {
        const uint64_t* pj = a.bits + (size_t)p * W;
        const uint64_t* pm = a.maxm + (size_t)p * W;
        const uint64_t* pa = a.addm + (size_t)p * W;
        for (int w = 0; w < W; ++w) {
          uint64_t s = pa[w];
          while (s) {
            int b = __ffsll((long long)s) - 1;
            s &= s - 1;
            int v = (w << 6) | b;
            unsigned long long c = atomicAdd(&s_cand, 1ull);
            if ((int64_t)c >= a.cand_cap) continue;
            write_child(W, v, pj, pm, pa, a.pred_u, a.succ_u, a.cand_bits + c * W,
                        a.cand_maxm + c * W, a.cand_addm + c * W);
          }
        }
      }
      __syncthreads();
      int64_t n_cand = (int64_t)s_cand;
      if (n_cand > a.cand_cap || 2 * n_cand > a.table_cap) {
        if (tid == 0) {
          a.status->code = 3;  // candidate capacity
          a.status->needed = n_cand;
          s_stop = 1;
        }
        __syncthreads();
        break;
      }
      for (int64_t i = tid; i < a.table_cap; i += blockDim.x) a.table[i] = -1;
      __syncthreads();
      // phase 2: insert into the hash set; the first inserted copy wins
      const int64_t tmask = a.table_cap - 1;
      for (int64_t c = tid; c < n_cand; c += blockDim.x) {
        const uint64_t* cj = a.cand_bits + c * W;
        int64_t pos = (int64_t)(fnv_hash(cj, W) & (uint64_t)tmask);
        bool fresh = false;
        while (true) {
          unsigned long long prev = atomicCAS((unsigned long long*)&a.table[pos],
                                              (unsigned long long)(-1LL), (unsigned long long)c);
          if (prev == (unsigned long long)(-1LL)) {
            fresh = true;
            break;
          }
          const uint64_t* oj = a.cand_bits + (int64_t)prev * W;
          bool same = true;
          for (int k = 0; k < W && same; ++k) same = oj[k] == cj[k];
          if (same) break;
          pos = (pos + 1) & tmask;
        }
        if (!fresh) continue;
        unsigned long long slot = atomicAdd(&s_next, 1ull);
        if ((int64_t)slot >= a.cap) continue;
        for (int k = 0; k < W; ++k) {
          a.bits[slot * W + k] = cj[k];
          a.maxm[slot * W + k] = a.cand_maxm[c * W + k];
          a.addm[slot * W + k] = a.cand_addm[c * W + k];
        }
        a.level_of[slot] = level + 1;
      }
    }
    __syncthreads();
    int64_t new_hi = (int64_t)s_next;
    if (new_hi > a.budget || new_hi > a.cap) {
      if (tid == 0) {
        a.status->code = new_hi > a.budget ? 1 : 2;  // budget / capacity
        a.status->needed = new_hi;
      }
      __syncthreads();
      break;
    }
    lo = hi;
    hi = new_hi;
    ++level;
    if (tid == 0 && hi > lo) a.level_off[level + 1] = hi;
    __syncthreads();
  }
  if (tid == 0 && a.status->code == 0 && !s_stop) {
    a.status->total = hi;
    a.status->n_levels = level;  // levels 0..level-1 are non-empty
  }
}

// ---- the level walk spread over a thread-block cluster -----------------
//
// Wide levels are where the single-CTA walk is issue-bound (C2: ~3.5 us per
// level at IPC 1.9 on one SM).  Here a cluster of kClusterCTAs CTAs walks the
// levels together: CTA r expands parents [lo + r*len, lo + (r+1)*len) of the
// level, each canonical child is built in full by the thread that found it
// (no intra-level barrier), the children take contiguous slots after a
// per-CTA count + block scan + one DSMEM atomicAdd on CTA 0's counter, and
// ONE cluster barrier (release / acquire: the new rows, written through
// global memory, are then visible to every CTA) ends the level.  Tiny levels
// stay with warp 0 of CTA 0 (expand_resident<32>, frontier in its shared
// memory) while the other CTAs wait at the barrier.
constexpr int kClusterCTAs = 8;

__device__ __forceinline__ bool canonical_child(const EnumArgs& a, const Adj& g,
                                                const uint64_t* M, int x, uint64_t mx, int upper,
                                                int v) {
  const int above = upper + __popcll(mx & above_mask(v, x));
  if (!above) return true;
  int covered = 0;
  const int p1 = g.pu_off[v + 1];
  for (int e = g.pu_off[v]; e < p1; ++e) {
    const int u = g.pu_adj[e];
    covered += (u > v && bit_of(M, u)) ? 1 : 0;
  }
  return covered == above;
}

// Child J ∪ {v} of parent `par` (all rows in global memory), written to slot.
__device__ __forceinline__ void build_child(const EnumArgs& a, const Adj& g, int64_t par, int v,
                                            int64_t slot, int level) {
  const int W = a.W;
  const uint64_t* J = a.bits + (size_t)par * W;
  const uint64_t* PM = a.maxm + (size_t)par * W;
  const uint64_t* PA = a.addm + (size_t)par * W;
  const uint64_t* pv = a.pred_u + (size_t)v * W;
  const int vw = v >> 6;
  const uint64_t vb = 1ull << (v & 63);
  for (int x = 0; x < W; ++x) {
    const uint64_t bx = x == vw ? vb : 0ull;
    a.bits[(size_t)slot * W + x] = J[x] | bx;
    a.maxm[(size_t)slot * W + x] = (PM[x] & ~__ldg(pv + x)) | bx;
  }
  uint64_t* CA = a.addm + (size_t)slot * W;
  for (int x = 0; x < W; ++x) CA[x] = PA[x] & ~(x == vw ? vb : 0ull);
  // successors of v that become addable: all their preds inside J ∪ {v}
  const int s1 = g.su_off[v + 1];
  for (int e = g.su_off[v]; e < s1; ++e) {
    const int y = g.su_adj[e];
    bool ok = true;
    const int f1 = g.pu_off[y + 1];
    for (int f = g.pu_off[y]; f < f1 && ok; ++f) {
      const int u = g.pu_adj[f];
      ok = u == v || bit_of(J, u);
    }
    if (ok) CA[y >> 6] |= 1ull << (y & 63);
  }
  a.level_of[slot] = level + 1;
}

// One level [lo, hi) across the cluster: returns this CTA's children count
// base slot (after the DSMEM claim); children are written at base + k.
__device__ __forceinline__ void expand_slice(const EnumArgs& a, const Adj& g, int64_t plo,
                                             int64_t phi, int level, int64_t level_end,
                                             unsigned long long* ctr0, int* s_scan,
                                             unsigned long long* s_base) {
  const int W = a.W;
  const int nt = blockDim.x, tid = threadIdx.x;
  const int64_t nP = phi - plo;
  // pass 1: count this thread's canonical children over (parent, word) items
  int mine = 0;
  for (int64_t it = tid; it < nP * W; it += nt) {
    const int64_t i = it / W;
    const int x = (int)(it % W);
    const size_t row = (size_t)(plo + i) * W;
    uint64_t cand = a.addm[row + x];
    if (!cand) continue;
    const uint64_t* M = a.maxm + row;
    int upper = 0;
    for (int y = x + 1; y < W; ++y) upper += __popcll(M[y]);
    const uint64_t mx = M[x];
    for (; cand; cand &= cand - 1) {
      const int v = (x << 6) | (__ffsll((long long)cand) - 1);
      mine += canonical_child(a, g, M, x, mx, upper, v) ? 1 : 0;
    }
  }
  // block exclusive scan of the counts, one DSMEM claim for the CTA
  const int lane = tid & 31, warp = tid >> 5;
  int incl = mine;
  for (int off = 1; off < 32; off <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += t;
  }
  if (lane == 31) s_scan[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = lane < (nt >> 5) ? s_scan[lane] : 0;
    int wi = w;
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += t;
    }
    s_scan[lane] = wi - w;  // exclusive over warps
    if (lane == 31) *s_base = atomicAdd(ctr0, (unsigned long long)wi);  // CTA total
  }
  __syncthreads();
  int64_t slot = level_end + (int64_t)*s_base + s_scan[warp] + (incl - mine);
  // pass 2: the same candidates, now written
  for (int64_t it = tid; it < nP * W; it += nt) {
    const int64_t i = it / W;
    const int x = (int)(it % W);
    const size_t row = (size_t)(plo + i) * W;
    uint64_t cand = a.addm[row + x];
    if (!cand) continue;
    const uint64_t* M = a.maxm + row;
    int upper = 0;
    for (int y = x + 1; y < W; ++y) upper += __popcll(M[y]);
    const uint64_t mx = M[x];
    for (; cand; cand &= cand - 1) {
      const int v = (x << 6) | (__ffsll((long long)cand) - 1);
      if (!canonical_child(a, g, M, x, mx, upper, v)) continue;
      if (slot < a.cap) build_child(a, g, plo + i, v, slot, level);
      ++slot;
    }
  }
}

__global__ void __launch_bounds__(kEnumThreads) enumerate_cluster_kernel(EnumArgs a) {
  namespace cgc = cooperative_groups;
  cgc::cluster_group cluster = cgc::this_cluster();
  const unsigned crank = cluster.block_rank();
  const int W = a.W;
  extern __shared__ uint64_t s_dyn[];
  __shared__ unsigned long long s_ctr[3];  // CTA 0's: children of level L in s_ctr[L % 3]
  __shared__ unsigned long long s_next;
  __shared__ int s_nc[2];
  __shared__ int s_scan[32];
  __shared__ unsigned long long s_base;
  __shared__ long long s_state[4];  // CTA 0 after a warp-mode run: lo, hi, level, status
  const int tid = threadIdx.x;

  // adjacency lists in shared memory (each CTA its own copy)
  int32_t* c = reinterpret_cast<int32_t*>(s_dyn + enum_warp_bytes(W) / sizeof(uint64_t));
  int32_t* pu_off = c;
  int32_t* su_off = pu_off + (a.n + 1);
  int32_t* pu_adj = su_off + (a.n + 1);
  int32_t* su_adj = pu_adj + a.n_pu;
  for (int i = tid; i <= a.n; i += blockDim.x) {
    pu_off[i] = a.pu_off[i];
    su_off[i] = a.su_off[i];
  }
  for (int i = tid; i < a.n_pu; i += blockDim.x) pu_adj[i] = a.pu_adj[i];
  for (int i = tid; i < a.n_su; i += blockDim.x) su_adj[i] = a.su_adj[i];
  const Adj adj{pu_off, pu_adj, su_off, su_adj};
  if (tid < 3) s_ctr[tid] = 0;
  if (crank == 0 && !a.resume) {
    // the empty ideal, ideals.cpp:23-24
    for (int w = tid; w < W; w += blockDim.x) {
      a.bits[w] = 0;
      a.maxm[w] = 0;
      a.addm[w] = 0;
    }
    __syncthreads();
    for (int v = tid; v < a.n; v += blockDim.x) {
      if (!a.in_universe[v]) continue;
      bool root = true;
      for (int w = 0; w < W; ++w) root &= a.pred_u[(size_t)v * W + w] == 0ull;
      if (root) atomicOr((unsigned long long*)&a.addm[v >> 6], 1ull << (v & 63));
    }
    if (tid == 0) {
      a.level_of[0] = 0;
      a.level_off[0] = 0;
      a.level_off[1] = 1;
    }
  }
  cluster.sync();
  unsigned long long* ctr0 = cluster.map_shared_rank(s_ctr, 0);
  long long* state0 = cluster.map_shared_rank(s_state, 0);

  int64_t lo = a.resume ? a.status->resume_lo : 0, hi = a.resume ? a.status->resume_hi : 1;
  int level = a.resume ? (int)a.status->resume_level : 0;
  int status = 0;  // 1 budget, 2 capacity
  while (hi > lo) {
    const int64_t nP = hi - lo;
    if (nP <= a.wide_min) {
      // CTA 0 alone walks levels up to its shared frontier capacity — tiny
      // ones with warp 0, the others with the whole CTA — level after level
      // with the frontier in its shared memory, until a wide level (or the
      // end); the other CTAs wait at the barrier
      if (crank == 0) {
        while (hi > lo && hi - lo <= a.wide_min) {
          const int64_t np = hi - lo;
          if (tid == 0) s_next = (unsigned long long)hi;
          __syncthreads();
          if (np <= small_cap(W) && np * W <= a.warp_items) {
            if (tid < 32) {
              expand_resident<32>(a, &lo, &hi, &level, &s_next, s_dyn, s_nc);
              if (tid == 0) {
                s_state[0] = lo;
                s_state[1] = hi;
                s_state[2] = level;
              }
            }
            __syncthreads();
            lo = s_state[0];
            hi = s_state[1];
            level = (int)s_state[2];
          } else {
            expand_resident<kEnumThreads>(a, &lo, &hi, &level, &s_next, s_dyn, s_nc);
          }
          __syncthreads();
          const int64_t new_hi = (int64_t)s_next;
          if (new_hi > a.budget || new_hi > a.cap) {
            if (tid == 0) {
              a.status->code = new_hi > a.budget ? 1 : 2;
              a.status->needed = new_hi;
            }
            status = 1;
            break;
          }
          lo = hi;
          hi = new_hi;
          ++level;
          if (tid == 0 && hi > lo) a.level_off[level + 1] = hi;
          __syncthreads();
        }
        if (tid == 0) {
          s_state[0] = lo;
          s_state[1] = hi;
          s_state[2] = level;
          s_state[3] = status;
          s_ctr[level % 3] = 0;  // the counter of the next (wide) level starts at 0
        }
      }
      cluster.sync();
      lo = state0[0];
      hi = state0[1];
      level = (int)state0[2];
      status = (int)state0[3];
      cluster.sync();  // everyone has read CTA 0's state before it is rewritten
      if (status) break;
      continue;
    }
    // a wide level across the cluster
    if (crank == 0 && tid == 0) s_ctr[(level + 1) % 3] = 0;  // the next level's counter
    const int64_t len = (nP + kClusterCTAs - 1) / kClusterCTAs;
    const int64_t plo = min(hi, lo + (int64_t)crank * len), phi = min(hi, plo + len);
    expand_slice(a, adj, plo, phi, level, hi, ctr0 + (level % 3), s_scan, &s_base);
    cluster.sync();
    const int64_t new_hi = hi + (int64_t)ctr0[level % 3];
    if (new_hi > a.budget || new_hi > a.cap) {
      if (crank == 0 && tid == 0) {
        a.status->code = new_hi > a.budget ? 1 : 2;
        a.status->needed = new_hi;
      }
      status = 1;
      break;
    }
    lo = hi;
    hi = new_hi;
    ++level;
    if (crank == 0 && tid == 0 && hi > lo) a.level_off[level + 1] = hi;
  }
  cluster.sync();  // no CTA exits while its shared memory may still be read
  if (crank == 0 && tid == 0 && a.status->code == 0 && !status) {
    a.status->total = hi;
    a.status->n_levels = level;
  }
}

// Lexicographic rank within a level (graph.cpp:62-72): the set holding the
// smallest differing index comes first.  rank(i) = #{j in level : j < i}.
__device__ __forceinline__ bool lex_less(const uint64_t* a, const uint64_t* b, int w0, int W) {
  for (int w = w0; w < W; ++w) {
    uint64_t d = a[w] ^ b[w];
    if (d) return (a[w] & (d & (~d + 1))) != 0ull;
  }
  return false;
}

constexpr int kRankRows = 64;   // ideals ranked per CTA
constexpr int kRankParts = 4;   // threads per ideal (each takes every 4th row)

// Levels above kRankDirect ideals are ordered by chunk-local ranks (the
// all-pairs count inside aligned chunks of kRankDirect) followed by
// merge-path passes (each element's position in the merged run = its
// position in its own run + a binary search in the partner run): O(T log T)
// comparisons instead of the direct rank's O(T^2) (a 12,870-ideal level of
// the 3 %-dense sweep point cost 2.4 ms that way).
constexpr int64_t kRankDirect = 1024;
constexpr int64_t kRankChunk = 256;  // chunk-local ranks, then merges from this width

// a before b in the level order (NodeSet::lex_less, graph.cpp:62-72): the
// set holding the smallest differing index comes first = the larger
// bit-reversed word at the first difference
__device__ __forceinline__ bool lex_before(const uint64_t* a, const uint64_t* b, int w0, int W) {
  for (int w = w0; w < W; ++w) {
    const uint64_t x = __brevll(__ldg(a + w)), y = __brevll(__ldg(b + w));
    if (x != y) return x > y;
  }
  return false;
}

__global__ void fill_i32_kernel(int* p, int n, int v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// The words every ideal of a level shares with the level's first ideal
// (lvl_d[s] = the first word where any differs): comparisons inside the level
// start there.  A long common stem leaves a wide lattice's ideals equal in
// all but their last words (a 2,000-node sweep point: 30 of 32).
__global__ void level_prefix_kernel(int W, int64_t total, const uint64_t* __restrict__ bits,
                                    const int32_t* __restrict__ level_of,
                                    const int64_t* __restrict__ level_off, int* __restrict__ lvl_d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int s = level_of[i];
  const int64_t lo = level_off[s];
  if (i == lo) return;
  int w = 0;
  while (w < W && bits[(size_t)i * W + w] == bits[(size_t)lo * W + w]) ++w;
  atomicMin(lvl_d + s, w);
}

__global__ void rank_chunk_kernel(int W, int64_t total, const uint64_t* __restrict__ bits,
                                  const int32_t* __restrict__ level_of,
                                  const int64_t* __restrict__ level_off, const int* __restrict__ lvl_d,
                                  int64_t* __restrict__ perm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int s = level_of[i];
  const int64_t lo = level_off[s], hi = level_off[s + 1];
  if (hi - lo <= kRankDirect) return;
  const int64_t c0 = lo + (i - lo) / kRankChunk * kRankChunk, c1 = min(hi, c0 + kRankChunk);
  const uint64_t* bi = bits + (size_t)i * W;
  int64_t r = 0;
  const int d0 = lvl_d[s];
  for (int64_t j = c0; j < c1; ++j) r += lex_before(bits + (size_t)j * W, bi, d0, W) ? 1 : 0;
  perm[c0 + r] = i;
}

__global__ void merge_pass_kernel(int W, int64_t total, int64_t width,
                                  const uint64_t* __restrict__ bits,
                                  const int32_t* __restrict__ level_of,
                                  const int64_t* __restrict__ level_off, const int* __restrict__ lvl_d,
                                  const int64_t* __restrict__ in, int64_t* __restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= total) return;
  const int s = level_of[p];  // positions keep their level
  const int64_t lo = level_off[s], hi = level_off[s + 1];
  if (hi - lo <= kRankDirect) return;
  const int64_t run = (p - lo) / width, r0 = lo + run * width;
  const int64_t q0 = lo + (run ^ 1) * width, q1 = min(hi, q0 + width);
  const int64_t e = in[p];
  if (q0 >= hi) {  // no partner run (the odd last one): stays in place
    out[p] = e;
    return;
  }
  const uint64_t* be = bits + (size_t)e * W;
  const int d0 = lvl_d[s];
  int64_t a = q0, b = q1;  // partner elements before e
  while (a < b) {
    const int64_t m = (a + b) >> 1;
    if (lex_before(bits + (size_t)in[m] * W, be, d0, W)) a = m + 1;
    else b = m;
  }
  out[min(r0, q0) + (p - r0) + (a - q0)] = e;
}

__global__ void scatter_perm_kernel(int W, int64_t total, const uint64_t* __restrict__ bits,
                                    const uint64_t* __restrict__ maxm,
                                    const int32_t* __restrict__ level_of,
                                    const int64_t* __restrict__ level_off,
                                    const int64_t* __restrict__ perm, uint64_t* __restrict__ out_bits,
                                    uint64_t* __restrict__ out_maxm) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= total) return;
  const int s = level_of[p];
  if (level_off[s + 1] - level_off[s] <= kRankDirect) return;
  const int64_t e = perm[p];
  for (int w = 0; w < W; ++w) {
    out_bits[(size_t)p * W + w] = bits[(size_t)e * W + w];
    out_maxm[(size_t)p * W + w] = maxm[(size_t)e * W + w];
  }
}

__global__ void __launch_bounds__(kRankRows* kRankParts)
    lex_rank_scatter_kernel(int W, int64_t total, const uint64_t* __restrict__ bits,
                            const uint64_t* __restrict__ maxm, const int32_t* __restrict__ level_of,
                            const int64_t* __restrict__ level_off, const int* __restrict__ lvl_d,
                            uint64_t* __restrict__ out_bits, uint64_t* __restrict__ out_maxm) {
  extern __shared__ uint64_t s_tile[];  // [tile rows][W], bit-reversed
  __shared__ int s_part[kRankParts][kRankRows];
  const int row = threadIdx.x % kRankRows, part = threadIdx.x / kRankRows;
  const int64_t i0 = (int64_t)blockIdx.x * kRankRows;
  const int64_t i = i0 + row;
  const int64_t il = min(i, total - 1);
  const int s = level_of[il];
  const int64_t lo = level_off[s], hi = level_off[s + 1];
  // levels above kRankDirect: rank_chunk + merge passes instead
  const bool act = i < total && hi - lo <= kRankDirect;
  const uint64_t* bi = bits + (size_t)il * W;
  int rank = 0;
  if (W <= 8) {
    // bit-reversed words: lex_less(a, b) <=> rev(a) > rev(b) as a big-endian
    // multi-word integer (the smallest differing index becomes the most
    // significant differing bit), so a comparison is a plain word compare.
    // The CTA tiles the union of its rows' levels through shared memory.
    uint64_t key[8];
    for (int w = 0; w < W; ++w) key[w] = __brevll(bi[w]);
    // the union of the (direct-ranked) levels of this CTA's rows
    __shared__ unsigned long long s_ulo, s_uhi;
    if (threadIdx.x == 0) {
      s_ulo = ~0ull;
      s_uhi = 0;
    }
    __syncthreads();
    if (part == 0 && act) {
      atomicMin(&s_ulo, (unsigned long long)lo);
      atomicMax(&s_uhi, (unsigned long long)hi);
    }
    __syncthreads();
    const int64_t uhi = (int64_t)s_uhi, ulo = uhi ? (int64_t)s_ulo : 0;  // none: empty range
    const int tile = kRankRows * kRankParts;
    for (int64_t t0 = ulo; t0 < uhi; t0 += tile) {
      const int n = (int)min((int64_t)tile, uhi - t0);
      __syncthreads();
      for (int k = threadIdx.x; k < n * W; k += blockDim.x)
        s_tile[k] = __brevll(bits[(size_t)t0 * W + k]);
      __syncthreads();
      const int j0 = (int)max((int64_t)0, lo - t0), j1 = (int)min((int64_t)n, hi - t0);
      for (int j = j0 + part; j < j1; j += kRankParts) {
        const uint64_t* bj = s_tile + (size_t)j * W;
        int w = 0;
        while (w < W - 1 && bj[w] == key[w]) ++w;
        rank += bj[w] > key[w] ? 1 : 0;
      }
    }
  } else if (act) {
    const int d0 = lvl_d[s];
    for (int64_t j = lo + part; j < hi; j += kRankParts)
      rank += lex_less(bits + (size_t)j * W, bi, d0, W) ? 1 : 0;
  }
  s_part[part][row] = rank;
  __syncthreads();
  if (part != 0 || !act) return;
  for (int q = 1; q < kRankParts; ++q) rank += s_part[q][row];
  uint64_t* o = out_bits + (size_t)(lo + rank) * W;
  uint64_t* om = out_maxm + (size_t)(lo + rank) * W;
  const uint64_t* mi = maxm + (size_t)i * W;
  for (int w = 0; w < W; ++w) {
    o[w] = bi[w];
    om[w] = mi[w];
  }
}

// Lower covers: the sub-ideals I' ⊂ I one level down are
// exactly I \ {v} for the maximal elements v of I (in the universe order),
// so the DP's newest-level pairs need no subset scan.  Their ordinals are
// found by binary search in level s-1, which is sorted by lex_less.
__global__ void cover_count_kernel(int W, int64_t I, const uint64_t* __restrict__ smax,
                                   int64_t* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > I) return;
  int64_t c = 0;
  if (i < I)
    for (int w = 0; w < W; ++w) c += __popcll(smax[(size_t)i * W + w]);
  cnt[i] = i < I ? c : 0;
}

__global__ void cover_fill_kernel(int W, int64_t I, const uint64_t* __restrict__ sbits,
                                  const uint64_t* __restrict__ smax,
                                  const int32_t* __restrict__ level_of,
                                  const int64_t* __restrict__ level_off,
                                  const int64_t* __restrict__ cov_off, int32_t* __restrict__ cov,
                                  const int* __restrict__ lvl_pre, int* __restrict__ err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= I) return;
  const int s = level_of[i];
  if (s == 0) return;
  const int64_t lo0 = level_off[s - 1], hi0 = level_off[s];
  // I \ {v} is an ideal of level s-1: it shares that level's common prefix
  const int w0 = lvl_pre ? lvl_pre[s - 1] : 0;
  const uint64_t* bi = sbits + (size_t)i * W;
  int64_t out = cov_off[i];
  uint64_t key[kMaxWords];
  for (int w = 0; w < W; ++w) key[w] = bi[w];
  for (int w = 0; w < W; ++w) {
    uint64_t m = smax[(size_t)i * W + w];
    while (m) {
      const uint64_t bit = m & (~m + 1);
      m ^= bit;
      key[w] &= ~bit;  // I \ {v}
      int64_t lo = lo0, hi = hi0;  // first j with !(bits_j < key)
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (lex_less(sbits + (size_t)mid * W, key, w0, W)) lo = mid + 1;
        else hi = mid;
      }
      bool eq = lo < hi0;
      for (int x = 0; eq && x < W; ++x) eq = sbits[(size_t)lo * W + x] == key[x];
      if (!eq) atomicExch(err, 1);  // cannot happen for a lattice from K1
      cov[out++] = eq ? (int32_t)lo : 0;
      key[w] |= bit;
    }
  }
}

}  // namespace

void launch_enumerate(const EnumLaunch& L, cudaStream_t st) {
  EnumArgs a;
  a.W = L.W;
  a.n = L.n;
  a.pred_u = L.pred_u;
  a.succ_u = L.succ_u;
  a.in_universe = L.in_universe;
  a.pu_off = L.pu_off;
  a.pu_adj = L.pu_adj;
  a.su_off = L.su_off;
  a.su_adj = L.su_adj;
  a.bits = L.bits;
  a.maxm = L.maxm;
  a.addm = L.addm;
  a.level_of = L.level_of;
  a.cap = L.cap;
  a.budget = L.budget;
  a.level_off = L.level_off;
  a.status = L.status;
  a.hash_mode = L.hash_mode;
  a.cand_bits = L.cand_bits;
  a.cand_maxm = L.cand_maxm;
  a.cand_addm = L.cand_addm;
  a.cand_cap = L.cand_cap;
  a.table = L.table;
  a.table_cap = L.table_cap;
  a.n_pu = L.n_pu;
  a.n_su = L.n_su;
  a.spill_par = L.spill_par;
  a.warp_items = 48;  // measured: C2 / C4 best at 32-64
  if (const char* e = std::getenv("DSG_ENUM_WARP_ITEMS")) a.warp_items = std::atoi(e);
  a.spill_v = L.spill_v;
  size_t smem = enum_warp_bytes(a.W);
  const size_t csr = enum_csr_bytes(a.n, a.n_pu, a.n_su);
  a.csr_in_smem = (!a.hash_mode && smem + csr <= 200 * 1024) ? 1 : 0;
  if (a.csr_in_smem) smem += csr;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(enumerate_levels_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  // canonical dedup: the cluster walk (env DSG_ENUM_CLUSTER=0: one CTA)
  static const bool cluster_off = [] {
    const char* e = std::getenv("DSG_ENUM_CLUSTER");
    return e && std::atoi(e) == 0;
  }();
  a.cluster_ok = !a.hash_mode && a.csr_in_smem && !cluster_off;
  a.wide_min = cta_cap(a.W);
  if (const char* e = std::getenv("DSG_ENUM_WIDE"))
    a.wide_min = std::max<int64_t>(1, std::min<int64_t>(a.wide_min, std::atoll(e)));
  a.resume = L.resume;
  if (L.resume) {
    cudaFuncSetAttribute(enumerate_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kClusterCTAs);
    cfg.blockDim = dim3(kEnumThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kClusterCTAs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, enumerate_cluster_kernel, a);
    count_launch();
    return;
  }
  enumerate_levels_kernel<<<1, kEnumThreads, smem, st>>>(a);
  count_launch();
}

bool launch_lex_rank(int W, int64_t total, const uint64_t* bits, const uint64_t* maxm,
                     const int32_t* level_of, const int64_t* level_off, uint64_t* out_bits,
                     uint64_t* out_maxm, int64_t max_level, int64_t* perm_a, int64_t* perm_b,
                     int* lvl_d, int n_levels, cudaStream_t st) {
  const bool prefix = W > 8 || max_level > kRankDirect;
  const int64_t blocks = (total + kRankRows - 1) / kRankRows;
  const size_t smem = W <= 8 ? (size_t)kRankRows * kRankParts * W * sizeof(uint64_t) : 0;
  if (prefix) {
    // the per-level common prefix (the word-by-word comparisons start there)
    fill_i32_kernel<<<(unsigned)((n_levels + 255) / 256), 256, 0, st>>>(lvl_d, n_levels, W);
    count_launch();
    level_prefix_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(W, total, bits, level_of,
                                                                          level_off, lvl_d);
    count_launch();
  }
  lex_rank_scatter_kernel<<<(unsigned)blocks, kRankRows * kRankParts, smem, st>>>(
      W, total, bits, maxm, level_of, level_off, lvl_d, out_bits, out_maxm);
  count_launch();
  if (max_level <= kRankDirect) return prefix;
  const unsigned g = (unsigned)((total + 255) / 256);
  rank_chunk_kernel<<<g, 256, 0, st>>>(W, total, bits, level_of, level_off, lvl_d, perm_a);
  count_launch();
  for (int64_t width = kRankChunk; width < max_level; width *= 2) {
    merge_pass_kernel<<<g, 256, 0, st>>>(W, total, width, bits, level_of, level_off, lvl_d, perm_a,
                                         perm_b);
    count_launch();
    std::swap(perm_a, perm_b);
  }
  scatter_perm_kernel<<<g, 256, 0, st>>>(W, total, bits, maxm, level_of, level_off, perm_a,
                                         out_bits, out_maxm);
  count_launch();
  return prefix;
}

namespace {
__global__ void adj_bits_kernel(int n, int W, const int32_t* __restrict__ pu_off,
                                const int32_t* __restrict__ pu_adj, const int32_t* __restrict__ su_off,
                                const int32_t* __restrict__ su_adj, const int32_t* __restrict__ out_off,
                                const int32_t* __restrict__ out_adj, uint64_t* __restrict__ pred_u,
                                uint64_t* __restrict__ succ_u, uint64_t* __restrict__ succ_real) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;  // row v is this thread's alone
  uint64_t* p = pred_u + (size_t)v * W;
  uint64_t* q = succ_u + (size_t)v * W;
  uint64_t* r = succ_real + (size_t)v * W;
  for (int e = pu_off[v]; e < pu_off[v + 1]; ++e) p[pu_adj[e] >> 6] |= 1ull << (pu_adj[e] & 63);
  for (int e = su_off[v]; e < su_off[v + 1]; ++e) q[su_adj[e] >> 6] |= 1ull << (su_adj[e] & 63);
  for (int e = out_off[v]; e < out_off[v + 1]; ++e) r[out_adj[e] >> 6] |= 1ull << (out_adj[e] & 63);
}
}  // namespace

void launch_adj_bits(int n, int W, const int32_t* pu_off, const int32_t* pu_adj, const int32_t* su_off,
                     const int32_t* su_adj, const int32_t* out_off, const int32_t* out_adj,
                     uint64_t* pred_u, uint64_t* succ_u, uint64_t* succ_real, cudaStream_t st) {
  if (n <= 0) return;
  adj_bits_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(n, W, pu_off, pu_adj, su_off, su_adj,
                                                               out_off, out_adj, pred_u, succ_u,
                                                               succ_real);
  count_launch();
}

void launch_cover_count(int W, int64_t I, const uint64_t* smax, int64_t* cnt, cudaStream_t st) {
  const int threads = 256;
  cover_count_kernel<<<(unsigned)((I + 1 + threads - 1) / threads), threads, 0, st>>>(W, I, smax,
                                                                                       cnt);
  count_launch();
}

void launch_cover_fill(int W, int64_t I, const uint64_t* sbits, const uint64_t* smax,
                       const int32_t* level_of, const int64_t* level_off, const int64_t* cov_off,
                       int32_t* cov, const int* lvl_pre, int* err, cudaStream_t st) {
  const int threads = 128;
  cover_fill_kernel<<<(unsigned)((I + threads - 1) / threads), threads, 0, st>>>(
      W, I, sbits, smax, level_of, level_off, cov_off, cov, lvl_pre, err);
  count_launch();
}

}  // namespace dsg
