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
#include <cstdint>

#include "dsg_device.cuh"
#include "dsg_internal.h"

namespace dsg {

namespace {

constexpr int kEnumThreads = 1024;

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
};

__global__ void __launch_bounds__(kEnumThreads) enumerate_levels_kernel(EnumArgs a) {
  const int W = a.W;
  __shared__ unsigned long long s_next;
  __shared__ unsigned long long s_cand;
  __shared__ int s_stop;
  const int tid = threadIdx.x;

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
            // canonical parent: no maximal element above v survives
            const uint64_t* pv = a.pred_u + (size_t)v * W;
            bool canon = true;
            for (int k = 0; k < W && canon; ++k) canon = (pm[k] & ~pv[k] & above_mask(v, k)) == 0ull;
            if (!canon) continue;
            unsigned long long slot = atomicAdd(&s_next, 1ull);
            if ((int64_t)slot >= a.cap) continue;
            write_child(W, v, pj, pm, pa, a.pred_u, a.succ_u, a.bits + slot * W,
                        a.maxm + slot * W, a.addm + slot * W);
            a.level_of[slot] = level + 1;
          }
        }
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

// Lexicographic rank within a level (graph.cpp:62-72): the set holding the
// smallest differing index comes first.  rank(i) = #{j in level : j < i}.
__device__ __forceinline__ bool lex_less(const uint64_t* a, const uint64_t* b, int W) {
  for (int w = 0; w < W; ++w) {
    uint64_t d = a[w] ^ b[w];
    if (d) return (a[w] & (d & (~d + 1))) != 0ull;
  }
  return false;
}

__global__ void lex_rank_scatter_kernel(int W, int64_t total, const uint64_t* __restrict__ bits,
                                        const int32_t* __restrict__ level_of,
                                        const int64_t* __restrict__ level_off,
                                        uint64_t* __restrict__ out_bits) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  int s = level_of[i];
  int64_t lo = level_off[s], hi = level_off[s + 1];
  const uint64_t* bi = bits + (size_t)i * W;
  int64_t rank = 0;
  for (int64_t j = lo; j < hi; ++j) rank += lex_less(bits + (size_t)j * W, bi, W) ? 1 : 0;
  uint64_t* o = out_bits + (size_t)(lo + rank) * W;
  for (int w = 0; w < W; ++w) o[w] = bi[w];
}

}  // namespace

void launch_enumerate(const EnumLaunch& L, cudaStream_t st) {
  EnumArgs a;
  a.W = L.W;
  a.n = L.n;
  a.pred_u = L.pred_u;
  a.succ_u = L.succ_u;
  a.in_universe = L.in_universe;
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
  enumerate_levels_kernel<<<1, kEnumThreads, 0, st>>>(a);
  count_launch();
}

void launch_lex_rank(int W, int64_t total, const uint64_t* bits, const int32_t* level_of,
                     const int64_t* level_off, uint64_t* out_bits, cudaStream_t st) {
  int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  lex_rank_scatter_kernel<<<(unsigned)blocks, threads, 0, st>>>(W, total, bits, level_of, level_off,
                                                                 out_bits);
  count_launch();
}

}  // namespace dsg
