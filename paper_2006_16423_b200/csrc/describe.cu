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

template <typename V, bool FILL>
__global__ void __launch_bounds__(128) describe_kernel(DescribeLaunch a) {
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= a.I) return;
  const DevGraph& g = a.g;
  const int W = g.W;
  uint64_t A[kMaxWords], F[kMaxWords], T[kMaxWords];
  const uint64_t* J = a.sbits + (size_t)o * W;
  for (int w = 0; w < W; ++w) A[w] = J[w];
  if (a.training) {
    for_bits(J, W, [&](int v) {
      const uint64_t* tw = g.twins + (size_t)v * W;
      for (int w = 0; w < W; ++w) A[w] |= tw[w];
    });
  }
  // prefix sums, frontier F(A), Σ comm over F(A)
  int64_t cpu = 0, acc = 0, mem = 0, fwv = 0;
  int32_t un = 0, fwi = 0, nF = 0;
  for (int w = 0; w < W; ++w) F[w] = 0;
  for_bits(A, W, [&](int v) {
    cpu += g.cpu[v];
    acc += g.acc[v];
    mem += g.mem[v];
    un += g.unsup[v];
    bool leaves = false;
    for (int e = g.out_real_off[v]; e < g.out_real_off[v + 1] && !leaves; ++e)
      leaves = !bit_of(A, g.out_real_adj[e]);
    if (leaves) {
      F[v >> 6] |= 1ull << (v & 63);
      fwv += g.comm[v];
      fwi += g.comminf[v];
      ++nF;
    }
  });
  const int n_chunks = (nF + 63) / 64;
  int64_t* cnt = a.counts;
  const int64_t stride = a.I + 1;
  int64_t n_items = 0;
  // frontier chunks: producers ranked in index order, 64 per chunk
  int64_t chunk_base = FILL ? cnt[kCntChunks * stride + o] : 0;
  int64_t f_base = FILL ? cnt[kCntF * stride + o] : 0;
  int64_t n_base = FILL ? cnt[kCntN * stride + o] : 0;
  FChunk first{};
  for (int c = 0; c < n_chunks; ++c) {
    int lo = c * 64;
    int hi = min(nF, lo + 64);
    // chunk members and their upper neighbours
    for (int w = 0; w < W; ++w) T[w] = 0;
    int rank = 0;
    uint64_t infmask = 0;
    for_bits(F, W, [&](int u) {
      if (rank >= lo && rank < hi) {
        for (int e = g.out_real_off[u]; e < g.out_real_off[u + 1]; ++e) {
          int x = g.out_real_adj[e];
          if (!bit_of(A, x)) T[x >> 6] |= 1ull << (x & 63);
        }
        if (FILL) {
          V* fp = (V*)a.fpool;
          fp[f_base + rank] = (V)g.comm[u];
          if (g.comminf[u]) infmask |= 1ull << (rank - lo);
        }
      }
      ++rank;
    });
    int nN = 0;
    for (int w = 0; w < W; ++w) nN += __popcll(T[w]);
    if (FILL) {
      int idx = 0;
      for_bits(T, W, [&](int x) {
        uint64_t pm = 0;
        int r = 0;
        for_bits(F, W, [&](int u) {
          if (r >= lo && r < hi && bit_of(g.succ_real + (size_t)u * W, x)) pm |= 1ull << (r - lo);
          ++r;
        });
        NItem it;
        it.word = (uint32_t)(x >> 6);
        it.bit = (uint32_t)(x & 63);
        it.predmask = pm;
        a.nitems[n_base + n_items + idx] = it;
        ++idx;
      });
      FChunk ch;
      ch.n_f = hi - lo;
      ch.n_n = nN;
      ch.off_f = (int32_t)(f_base + lo);
      ch.off_n = (int32_t)(n_base + n_items);
      ch.infmask = infmask;
      a.chunks[chunk_base + c] = ch;
      if (c == 0) first = ch;
    }
    n_items += nN;
  }
  int64_t nP = 0, nLI = 0;
  uint8_t up = 1;
  if (a.training) {
    // P'(A) = L(A) = real predecessors of A outside A
    for (int w = 0; w < W; ++w) T[w] = 0;
    for_bits(A, W, [&](int v) {
      for (int e = g.in_real_off[v]; e < g.in_real_off[v + 1]; ++e) {
        int u = g.in_real_adj[e];
        if (!bit_of(A, u)) T[u >> 6] |= 1ull << (u & 63);
      }
    });
    int64_t p_base = FILL ? cnt[kCntP * stride + o] : 0;
    int64_t l_base = FILL ? cnt[kCntL * stride + o] : 0;
    int64_t li_base = FILL ? cnt[kCntLItems * stride + o] : 0;
    for_bits(T, W, [&](int u) {
      const uint64_t* su = g.succ_real + (size_t)u * W;
      int items = 0;
      for (int w = 0; w < W; ++w) {
        uint64_t m = su[w] & A[w];
        if (m) {
          if (FILL) {
            MaskItem mi;
            mi.word = (uint32_t)w;
            mi.pad = 0;
            mi.mask = m;
            a.litems[li_base + nLI + items] = mi;
          }
          ++items;
        }
      }
      if (FILL) {
        PItem pi;
        pi.word = (uint32_t)(u >> 6);
        pi.bit = (uint32_t)(u & 63);
        pi.inf = g.comminf[u];
        pi.pad = 0;
        pi.weight = g.comm[u];
        a.pitems[p_base + nP] = pi;
        LEntry le;
        le.n_items = items;
        le.off_items = (int32_t)(li_base + nLI);
        le.inf = g.comminf[u];
        le.pad = 0;
        le.weight = g.comm[u];
        a.lentries[l_base + nP] = le;
      }
      nLI += items;
      ++nP;
    });
    // Φ(J) = A ∩ backward: an up-set of the backward part?
    if (a.has_bw) {
      for_bits(A, W, [&](int b) {
        if (!bit_of(g.bwset, b)) return;
        const uint64_t* bs = g.bw_succ + (size_t)b * W;
        for (int w = 0; w < W; ++w)
          if (bs[w] & ~A[w]) up = 0;
      });
    }
  }
  if (!FILL) {
    cnt[kCntChunks * stride + o] = n_chunks;
    cnt[kCntF * stride + o] = nF;
    cnt[kCntN * stride + o] = n_items;
    cnt[kCntP * stride + o] = nP;
    cnt[kCntL * stride + o] = nP;
    cnt[kCntLItems * stride + o] = nLI;
    return;
  }
  for (int w = 0; w < a.AW; ++w) a.abits[(size_t)o * a.AW + w] = w < W ? A[w] : 0ull;
  if (a.training) {
    for (int w = 0; w < W; ++w) a.intbits[(size_t)o * W + w] = A[w] & ~F[w];
    a.upset[o] = up;
  }
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
__global__ void __launch_bounds__(1024) scan_counts_kernel(int64_t* counts, int64_t n) {
  int64_t* x = counts + (size_t)blockIdx.x * (n + 1);
  const int64_t total_n = n + 1;
  const int T = blockDim.x;
  const int64_t seg = (total_n + T - 1) / T;
  const int64_t lo = threadIdx.x * seg;
  const int64_t hi = min(total_n, lo + seg);
  int64_t s = 0;
  for (int64_t i = lo; i < hi; ++i) s += x[i];
  __shared__ int64_t sh[1024];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int off = 1; off < T; off <<= 1) {
    int64_t v = threadIdx.x >= off ? sh[threadIdx.x - off] : 0;
    __syncthreads();
    sh[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t run = sh[threadIdx.x] - s;  // exclusive
  for (int64_t i = lo; i < hi; ++i) {
    int64_t v = x[i];
    x[i] = run;
    run += v;
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
  int threads = 128;
  unsigned blocks = (unsigned)((L.I + threads - 1) / threads);
  if (L.value_bits == 32) {
    if (fill) describe_kernel<int32_t, true><<<blocks, threads, 0, st>>>(L);
    else describe_kernel<int32_t, false><<<blocks, threads, 0, st>>>(L);
  } else {
    if (fill) describe_kernel<int64_t, true><<<blocks, threads, 0, st>>>(L);
    else describe_kernel<int64_t, false><<<blocks, threads, 0, st>>>(L);
  }
  count_launch();
}

void launch_scan_counts(int64_t* counts, int64_t I, int n_arrays, cudaStream_t st) {
  scan_counts_kernel<<<n_arrays, 1024, 0, st>>>(counts, I);
  count_launch();
}

}  // namespace dsg
