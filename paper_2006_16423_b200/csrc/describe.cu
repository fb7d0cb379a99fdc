// describe.cu — K1b: per-ideal descriptors for the fused transition kernel.
//
// The reference recomputes block costs incrementally along its DFS
// (BlockTracker, /root/reference/proj/src/dp_solver.cpp:33-98).  On the
// device every (target I, source I') pair is independent, so the cost of
// the block B = A(I) \ A(I') must come from O(1)-size per-ideal data plus a
// walk over the SOURCE's small frontier.  With A = A(I), A' = A(I') and
// real edges only (acc_cost_parts, graph.cpp:397-428):
//
//   cpu/proc/mem/unsupported(B)  = prefix(A) - prefix(A')
//   comm_out(B) = W(F(A)) - W({u in F(A') : succ(u)\A' ⊄ A})
//                 + W(P'(A') ∩ Int(A))                        [training]
//   comm_in(B)  = W({u in F(A') : (succ(u)\A') ∩ A ≠ ∅})
//                 + W({u in L(A) : succ(u) ∩ A ⊄ A'})         [training]
//
// with F(X) = {v in X : a real successor outside X}, Int(X) = X \ F(X),
// P'(X) = L(X) = Pred(X) \ X.  For inference graphs A is an ideal, so
// P' and L are empty and only the frontier walk remains.  The frontier
// walk tests each upper neighbour n in N(A') = succ(F(A')) \ A' once
// against the target bitset and ORs in a bitmask of the producers that
// feed n, so both comm terms come from two 64-bit masks.
//
// Pass 1 counts table sizes per ideal, a scan turns them into offsets,
// pass 2 fills the pools.
#include <climits>
#include <cstdint>

#include "dsg_device.cuh"
#include "dsg_internal.h"

namespace dsg {

namespace {

template <typename F>
__device__ __forceinline__ void for_bits(const uint64_t* s, int W, F&& f) {
  for (int w = 0; w < W; ++w) {
    uint64_t x = s[w];
    while (x) {
      int b = __ffsll((long long)x) - 1;
      x &= x - 1;
      f((w << 6) | b);
    }
  }
}

template <typename T>
__device__ __forceinline__ T group_sum(T v, int G, unsigned gm) {
  for (int off = G >> 1; off > 0; off >>= 1) v += __shfl_xor_sync(gm, v, off);
  return v;
}

__device__ __forceinline__ uint64_t group_or(uint64_t v, int G, unsigned gm) {
  for (int off = G >> 1; off > 0; off >>= 1) v |= __shfl_xor_sync(gm, v, off);
  return v;
}

constexpr int kDescThreads = 128;

// Lanes per ideal: enough to cover the bitset words (a power of two <= 32),
// so an ideal of n members costs O(n / G) dependent steps instead of O(n)
// (one thread per ideal was 0.5 ms on C1's 242 ideals of ~350 members) —
// but no more lanes than about one full wave of threads needs: large
// lattices keep all lanes busy with fewer lanes per ideal.
__host__ __device__ __forceinline__ size_t desc_group_bytes(int W) {
  return 4 * W * sizeof(uint64_t) + 2 * (W + 1) * sizeof(int32_t);
}

// G lanes per ideal: about one wave of threads in flight, and the groups'
// shared rows within kDescSmemMax (wide bitsets on large lattices: W = 24 at
// 47K ideals needs 62 KB at G = 2)
constexpr size_t kDescSmemMax = 96 * 1024;
__host__ __device__ __forceinline__ int desc_group(int W, int64_t I) {
  int G = 32;  // the member loops stride over bit positions, so any W uses G lanes
  // (wider bitsets give each lane more words per member loop: a larger budget)
  const int64_t budget = (int64_t)148 * 8 * kDescThreads * (W > 8 ? W / 8 : 1);
  while (G > 1 && I * G > budget) G >>= 1;
  while (G < 32 && (size_t)(kDescThreads / G) * desc_group_bytes(W) > kDescSmemMax) G <<= 1;
  return G;
}

// shared words per group: A, F, T (chunk neighbours), P; then two rank arrays
__host__ __device__ __forceinline__ size_t desc_smem(int W, int64_t I) {
  const int groups = kDescThreads / desc_group(W, I);
  return (size_t)groups * desc_group_bytes(W);
}

template <typename V, bool FILL>
__global__ void __launch_bounds__(kDescThreads) describe_kernel(DescribeLaunch a) {
  extern __shared__ uint64_t d_sh[];
  const DevGraph& g = a.g;
  const int W = g.W;
  // a group of G lanes per ideal (the lanes split the bitset words); the
  // ranked outputs (frontier producers in index order, 64 per chunk; the
  // training lists in index order) come from per-word popcount prefixes
  const int G = desc_group(W, a.I), groups = kDescThreads / G;
  const int gid = threadIdx.x / G, lane = threadIdx.x % G;
  const unsigned gm = G == 32 ? 0xffffffffu : ((1u << G) - 1) << ((threadIdx.x & 31) & ~(G - 1));
  const int64_t o = (int64_t)blockIdx.x * groups + gid;
  if (o >= a.I) return;  // group-uniform
  // member loops: this lane takes the bit positions ≡ lane (mod G) of every word
  uint64_t lm = 0;
  for (int b = lane; b < 64; b += G) lm |= 1ull << b;
  uint64_t* A = d_sh + (size_t)gid * 4 * W;
  uint64_t* F = A + W;
  uint64_t* T = F + W;
  uint64_t* P = T + W;
  int32_t* rF = reinterpret_cast<int32_t*>(d_sh + (size_t)groups * 4 * W) + (size_t)gid * 2 * (W + 1);
  int32_t* rT = rF + W + 1;
  const uint64_t* J = a.sbits + (size_t)o * W;
  for (int w = lane; w < W; w += G) {
    A[w] = J[w];
    F[w] = 0;
    T[w] = 0;
    P[w] = 0;
  }
  __syncwarp(gm);
  if (a.training) {  // A = J ∪ paired backward nodes (dp_solver.cpp:235-250)
    for (int w = 0; w < W; ++w) {
      for (uint64_t x = J[w] & lm; x; x &= x - 1) {
        const int v = (w << 6) | (__ffsll((long long)x) - 1);
        const uint64_t* tw = g.twins + (size_t)v * W;
        for (int y = 0; y < W; ++y) {
          const uint64_t t = tw[y];
          if (t) atomicOr((unsigned long long*)&A[y], (unsigned long long)t);
        }
      }
    }
    __syncwarp(gm);
  }
  // prefix sums and the frontier F(A) (members with a real successor outside)
  int64_t cpu = 0, acc = 0, mem = 0, fwv = 0;
  int32_t un = 0, fwi = 0, nF = 0;
  for (int w = 0; w < W; ++w) {
    uint64_t fw = 0;
    for (uint64_t x = A[w] & lm; x; x &= x - 1) {
      const int b = __ffsll((long long)x) - 1, v = (w << 6) | b;
      cpu += g.cpu[v];
      acc += g.acc[v];
      mem += g.mem[v];
      un += g.unsup[v];
      bool leaves = false;
      for (int e = g.out_real_off[v]; e < g.out_real_off[v + 1] && !leaves; ++e)
        leaves = !bit_of(A, g.out_real_adj[e]);
      if (leaves) {
        fw |= 1ull << b;
        fwv += g.comm[v];
        fwi += g.comminf[v];
        ++nF;
      }
    }
    if (fw) atomicOr((unsigned long long*)&F[w], (unsigned long long)fw);
  }
  cpu = group_sum(cpu, G, gm);
  acc = group_sum(acc, G, gm);
  mem = group_sum(mem, G, gm);
  fwv = group_sum(fwv, G, gm);
  un = group_sum(un, G, gm);
  fwi = group_sum(fwi, G, gm);
  nF = group_sum(nF, G, gm);
  __syncwarp(gm);
  if (lane == 0) {
    int r = 0;
    for (int w = 0; w < W; ++w) {
      rF[w] = r;
      r += __popcll(F[w]);
    }
  }
  __syncwarp(gm);
  const int n_chunks = (nF + 63) / 64;
  int64_t* cnt = a.counts;
  const int64_t stride = a.I + 1;
  int64_t n_items = 0;
  // frontier chunks: producers ranked in index order, 64 per chunk
  const int64_t chunk_base = FILL ? cnt[kCntChunks * stride + o] : 0;
  const int64_t f_base = FILL ? cnt[kCntF * stride + o] : 0;
  const int64_t n_base = FILL ? cnt[kCntN * stride + o] : 0;
  FChunk first{};
  for (int c = 0; c < n_chunks; ++c) {
    const int lo = c * 64, hi = min(nF, lo + 64);
    // the chunk's upper neighbours T (successors outside A), weights, ∞ mask
    uint64_t infm = 0;
    for (int w = 0; w < W; ++w) {
      if (rF[w] >= hi || rF[w] + __popcll(F[w]) <= lo) continue;
      for (uint64_t x = F[w] & lm; x; x &= x - 1) {
        const int b = __ffsll((long long)x) - 1;
        const int r = rF[w] + __popcll(F[w] & ((1ull << b) - 1));
        if (r < lo || r >= hi) continue;
        const int u = (w << 6) | b;
        for (int e = g.out_real_off[u]; e < g.out_real_off[u + 1]; ++e) {
          const int y = g.out_real_adj[e];
          if (!bit_of(A, y)) atomicOr((unsigned long long*)&T[y >> 6], 1ull << (y & 63));
        }
        if (FILL) {
          ((V*)a.fpool)[f_base + r] = (V)g.comm[u];
          if (g.comminf[u]) infm |= 1ull << (r - lo);
        }
      }
    }
    infm = group_or(infm, G, gm);
    __syncwarp(gm);
    int nN = 0;
    for (int w = lane; w < W; w += G) nN += __popcll(T[w]);
    nN = group_sum(nN, G, gm);
    if (FILL) {
      if (lane == 0) {
        int r = 0;
        for (int w = 0; w < W; ++w) {
          rT[w] = r;
          r += __popcll(T[w]);
        }
      }
      __syncwarp(gm);
      // NItem per upper neighbour y: which chunk producers feed it
      for (int w = 0; w < W; ++w) {
        for (uint64_t x = T[w] & lm; x; x &= x - 1) {
          const int b = __ffsll((long long)x) - 1;
          const int r = rT[w] + __popcll(T[w] & ((1ull << b) - 1));
          const int y = (w << 6) | b;
          uint64_t pm = 0;
          for (int fw = 0; fw < W; ++fw) {
            int q = rF[fw];
            if (q >= hi || q + __popcll(F[fw]) <= lo) continue;
            for (uint64_t z = F[fw]; z; z &= z - 1, ++q) {
              if (q < lo || q >= hi) continue;
              const int u = (fw << 6) | (__ffsll((long long)z) - 1);
              if (bit_of(g.succ_real + (size_t)u * W, y)) pm |= 1ull << (q - lo);
            }
          }
          NItem it;
          it.word = (uint32_t)(y >> 6);
          it.bit = (uint32_t)(y & 63);
          it.predmask = pm;
          a.nitems[n_base + n_items + r] = it;
        }
      }
      FChunk ch;
      ch.n_f = hi - lo;
      ch.n_n = nN;
      ch.off_f = (int32_t)(f_base + lo);
      ch.off_n = (int32_t)(n_base + n_items);
      ch.infmask = infm;
      if (lane == 0) a.chunks[chunk_base + c] = ch;
      if (c == 0) first = ch;
    }
    n_items += nN;
    __syncwarp(gm);
    for (int w = lane; w < W; w += G) T[w] = 0;
    __syncwarp(gm);
  }
  int64_t nP = 0, nLI = 0;
  int up = 1;
  if (a.training) {
    // P'(A) = L(A) = real predecessors of A outside A
    for (int w = 0; w < W; ++w) {
      for (uint64_t x = A[w] & lm; x; x &= x - 1) {
        const int v = (w << 6) | (__ffsll((long long)x) - 1);
        for (int e = g.in_real_off[v]; e < g.in_real_off[v + 1]; ++e) {
          const int u = g.in_real_adj[e];
          if (!bit_of(A, u)) atomicOr((unsigned long long*)&P[u >> 6], 1ull << (u & 63));
        }
      }
    }
    __syncwarp(gm);
    // per u: one MaskItem per word where succ(u) meets A
    for (int w = 0; w < W; ++w) {
      for (uint64_t x = P[w] & lm; x; x &= x - 1) {
        const int u = (w << 6) | (__ffsll((long long)x) - 1);
        const uint64_t* su = g.succ_real + (size_t)u * W;
        for (int y = 0; y < W; ++y) nLI += (su[y] & A[y]) ? 1 : 0;
        ++nP;
      }
    }
    nP = group_sum(nP, G, gm);
    nLI = group_sum(nLI, G, gm);
    if (FILL && lane == 0) {  // ranked outputs, in index order (|P'| is small)
      const int64_t p_base = cnt[kCntP * stride + o];
      const int64_t l_base = cnt[kCntL * stride + o];
      const int64_t li_base = cnt[kCntLItems * stride + o];
      int64_t np = 0, nli = 0;
      for (int w = 0; w < W; ++w) {
        for (uint64_t x = P[w]; x; x &= x - 1) {
          const int u = (w << 6) | (__ffsll((long long)x) - 1);
          const uint64_t* su = g.succ_real + (size_t)u * W;
          int items = 0;
          for (int y = 0; y < W; ++y) {
            const uint64_t m = su[y] & A[y];
            if (m) {
              MaskItem mi;
              mi.word = (uint32_t)y;
              mi.pad = 0;
              mi.mask = m;
              a.litems[li_base + nli + items] = mi;
              ++items;
            }
          }
          PItem pi;
          pi.word = (uint32_t)(u >> 6);
          pi.bit = (uint32_t)(u & 63);
          pi.inf = g.comminf[u];
          pi.pad = 0;
          pi.weight = g.comm[u];
          a.pitems[p_base + np] = pi;
          LEntry le;
          le.n_items = items;
          le.off_items = (int32_t)(li_base + nli);
          le.inf = g.comminf[u];
          le.pad = 0;
          le.weight = g.comm[u];
          a.lentries[l_base + np] = le;
          nli += items;
          ++np;
        }
      }
    }
    // Φ(J) = A ∩ backward: an up-set of the backward part?
    if (a.has_bw) {
      for (int w = 0; w < W; ++w) {
        for (uint64_t x = A[w] & g.bwset[w] & lm; x; x &= x - 1) {
          const int b = (w << 6) | (__ffsll((long long)x) - 1);
          const uint64_t* bs = g.bw_succ + (size_t)b * W;
          for (int y = 0; y < W; ++y)
            if (bs[y] & ~A[y]) up = 0;
        }
      }
      up = __all_sync(gm, up) ? 1 : 0;
    }
  }
  if (!FILL) {
    if (lane == 0) {
      cnt[kCntChunks * stride + o] = n_chunks;
      cnt[kCntF * stride + o] = nF;
      cnt[kCntN * stride + o] = n_items;
      cnt[kCntP * stride + o] = nP;
      cnt[kCntL * stride + o] = nP;
      cnt[kCntLItems * stride + o] = nLI;
    }
    return;
  }
  for (int w = lane; w < a.AW; w += G) a.abits[(size_t)o * a.AW + w] = w < W ? A[w] : 0ull;
  if (a.training)
    for (int w = lane; w < W; w += G) a.intbits[(size_t)o * W + w] = A[w] & ~F[w];
  if (lane != 0) return;
  if (a.training) a.upset[o] = (uint8_t)up;
  ((V*)a.pfx_cpu)[o] = (V)cpu;
  ((V*)a.pfx_acc)[o] = (V)acc;
  ((V*)a.pfx_mem)[o] = (V)mem;
  a.unsup[o] = un;
  ((V*)a.fw)[o] = (V)fwv;
  a.fwinf[o] = fwi;
  SrcRec r;
  r.cpu = cpu;
  r.acc = acc;
  r.mem = mem;
  r.unsup = un;
  r.n_chunks = n_chunks;
  r.chunk0 = (int32_t)chunk_base;
  r.n_f = first.n_f;
  r.n_n = first.n_n;
  r.off_f = first.off_f;
  r.off_n = first.off_n;
  r.pad = 0;
  r.infmask = first.infmask;
  a.srec[o] = r;
}

// In-place exclusive scan of one [n + 1] int64 array per block
// (element n is 0 on entry and receives the total).
// Exclusive scan of one [n + 1] count array per CTA (the entry n becomes the
// total).  Tiles of 1024 x 8 entries: each thread scans 8 consecutive
// entries (coalesced 16-byte loads), warp shuffles and one shared pass over
// the 32 warp sums give the tile's offsets, and the tile total carries over.
__global__ void __launch_bounds__(1024) scan_counts_kernel(int64_t* counts, int64_t n) {
  constexpr int kPer = 8;
  int64_t* x = counts + (size_t)blockIdx.x * (n + 1);
  const int64_t total_n = n + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int64_t wsum[32];
  __shared__ int64_t carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  // the array base is 8-byte aligned only: vector loads when 16-aligned
  const bool vec = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  for (int64_t base = 0; base < total_n; base += (int64_t)blockDim.x * kPer) {
    const int64_t lo = base + (int64_t)threadIdx.x * kPer;
    int64_t v[kPer];
    if (vec && lo + kPer <= total_n) {
#pragma unroll
      for (int j = 0; j < kPer; j += 2) {
        const longlong2 q = *reinterpret_cast<const longlong2*>(x + lo + j);
        v[j] = q.x;
        v[j + 1] = q.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < kPer; ++j) v[j] = lo + j < total_n ? x[lo + j] : 0;
    }
    int64_t s = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) s += v[j];
    int64_t incl = s;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int nw = blockDim.x >> 5;
      int64_t w = lane < nw ? wsum[lane] : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, w, off);
        if (lane >= off) w += y;
      }
      if (lane < nw) wsum[lane] = w;  // inclusive warp offsets
    }
    __syncthreads();
    const int64_t carry = carry_s;
    int64_t run = carry + (warp ? wsum[warp - 1] : 0) + incl - s;
    if (vec && lo + kPer <= total_n) {
#pragma unroll
      for (int j = 0; j < kPer; j += 2) {
        longlong2 q;
        q.x = run;
        run += v[j];
        q.y = run;
        run += v[j + 1];
        *reinterpret_cast<longlong2*>(x + lo + j) = q;
      }
    } else {
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        if (lo + j < total_n) x[lo + j] = run;
        run += v[j];
      }
    }
    __syncthreads();  // every thread has read carry_s and wsum
    if (threadIdx.x == blockDim.x - 1) carry_s = carry + wsum[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
}

}  // namespace

// Per aligned block of kChunkMaxLen source ordinals: the maxima of the
// prefix sums acc / mem / cpu over the block.  With them an item can tell,
// before touching a single source, that no source of its chunk can give any
// of its targets a feasible, improving block (the per-pair tests of
// scan_sources, taken over the block's extreme values) — such chunks only
// count their nested pairs.
__global__ void chunk_max_kernel(const SrcRec* __restrict__ srec, int64_t I, int64_t* __restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (c * kChunkMaxLen >= I) return;
  long long ma = LLONG_MIN, mm = LLONG_MIN, mc = LLONG_MIN;
  for (int64_t o = c * kChunkMaxLen + lane; o < min(I, (c + 1) * kChunkMaxLen); o += 32) {
    ma = max(ma, (long long)srec[o].acc);
    mm = max(mm, (long long)srec[o].mem);
    mc = max(mc, (long long)srec[o].cpu);
  }
  for (int off = 16; off > 0; off >>= 1) {
    ma = max(ma, __shfl_xor_sync(0xffffffffu, ma, off));
    mm = max(mm, __shfl_xor_sync(0xffffffffu, mm, off));
    mc = max(mc, __shfl_xor_sync(0xffffffffu, mc, off));
  }
  if (lane == 0) {
    out[4 * c] = ma;
    out[4 * c + 1] = mm;
    out[4 * c + 2] = mc;
    out[4 * c + 3] = 0;
  }
}

void launch_chunk_max(const SrcRec* srec, int64_t I, int64_t* out, cudaStream_t st) {
  const int64_t n = (I + kChunkMaxLen - 1) / kChunkMaxLen;
  if (n <= 0) return;
  chunk_max_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(srec, I, out);
  count_launch();
}

void launch_describe(const DescribeLaunch& L, bool fill, cudaStream_t st) {
  const int threads = kDescThreads, groups = kDescThreads / desc_group(L.g.W, L.I);
  const unsigned blocks = (unsigned)((L.I + groups - 1) / groups);
  const size_t smem = desc_smem(L.g.W, L.I);
  if (blocks == 0) return;
  // above the 48 KB default: opt in (per device context, so on every launch)
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(describe_kernel<int32_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(describe_kernel<int32_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(describe_kernel<int64_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(describe_kernel<int64_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  if (L.value_bits == 32) {
    if (fill) describe_kernel<int32_t, true><<<blocks, threads, smem, st>>>(L);
    else describe_kernel<int32_t, false><<<blocks, threads, smem, st>>>(L);
  } else {
    if (fill) describe_kernel<int64_t, true><<<blocks, threads, smem, st>>>(L);
    else describe_kernel<int64_t, false><<<blocks, threads, smem, st>>>(L);
  }
  count_launch();
}

void launch_scan_counts(int64_t* counts, int64_t I, int n_arrays, cudaStream_t st) {
  scan_counts_kernel<<<n_arrays, 1024, 0, st>>>(counts, I);
  count_launch();
}

}  // namespace dsg
