// persistent.cu — host side of the dataflow level kernel: variant dispatch
// (the kernels live in persistent_impl.cuh, instantiated by persistent_v*.cu)
// and the device-built, readiness-ordered work-item list.
#include <climits>
#include <cstdint>
#include <cstdlib>

#include "persistent_impl.cuh"

namespace dsg {

namespace {

void dispatch(const LevelLaunch& L, const PersistPlan* P, cudaStream_t st, PersistInfo* info) {
  if (L.value_bits == 32) {
    if (L.training) {
      if (!dispatch_exact_i32_train(L, P, st, info)) dispatch_general_i32_train(L, P, st, info);
    } else {
      if (!dispatch_exact_i32_inf(L, P, st, info)) dispatch_general_i32_inf(L, P, st, info);
    }
  } else {
    if (L.training) dispatch_general_i64_train(L, P, st, info);
    else if (!dispatch_exact_i64_inf(L, P, st, info)) dispatch_general_i64_inf(L, P, st, info);
  }
}

// ---- item list on the device
struct PairInfo {
  int s, dep, bucket;
  int64_t c, units_r, n_items;
};

__device__ PairInfo pair_info(const PersistPlan& p, const ItemBuild& b, int64_t q) {
  int lo = 1, hi = b.n_levels - 1;  // largest s with pair_off[s] <= q
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (b.pair_off[mid] <= q) lo = mid;
    else hi = mid - 1;
  }
  PairInfo r;
  r.s = lo;
  r.c = q - b.pair_off[lo];
  const int64_t S = p.level_off[lo], T = p.level_off[lo + 1] - S;
  const int mode = p.mode[lo];
  int64_t s0, s1;
  if (mode == 0) {
    mode0_chunk(p, lo, r.c, s0, s1);
  } else {
    s1 = r.c < p.n_chunks[lo] - 1 ? p.chunk_lo[p.chunk_base[lo] + r.c + 1] : -1;
  }
  r.dep = s1 < 0 ? lo - 1 : p.level_of[s1 - 1];  // the cover chunk waits for level s-1
  const int64_t units = mode == 0 ? (T + kGroup - 1) / kGroup : T;
  r.units_r = b.world > 1 ? (units > b.rank ? (units - b.rank + b.world - 1) / b.world : 0) : units;
  // scheduling bucket: a chunk for a far-future level waits in the list until
  // `lag` levels before its target, so each bucket holds a bounded amount of
  // near-term work and the critical items are not queued behind the future
  r.bucket = max(r.dep, lo - b.lag);
  r.n_items = r.units_r;
  // the chain runner's finishers are not listed (capi.cu builds its list)
  if (b.runner_max_t > 0 && mode != 0 && r.c == p.n_chunks[lo] - 1 && T <= b.runner_max_t)
    r.n_items = 0;
  return r;
}

// Sort key of an item.  One queue (b.split == 0): by dependency bucket, and
// inside a bucket the critical items (target level = dep + 1, i.e. the cover
// chunks) first — a mode-1 target's finisher after them, after all the
// target's other chunks, which it waits for —, then the rest.  Two queues
// (b.split != 0): the cover items first (keys [0, 2n)), by level, then the
// background items by bucket (keys [2n, 3n)).
// Background items of a bucket are ordered near-first: the chunks of level
// dep + 2 (they gate the level after the one being finished) before the
// chunks of later levels.
__device__ __forceinline__ int item_key(const PersistPlan& p, const ItemBuild& b,
                                        const PairInfo& r) {
  const bool crit = r.s == r.dep + 1;
  const int cls = crit ? ((p.mode[r.s] != 0 && r.c == p.n_chunks[r.s] - 1) ? 1 : 0)
                       : (r.s == r.dep + 2 ? 2 : 3);
  if (!b.split) return 4 * r.bucket + cls;
  return crit ? 2 * r.bucket + cls : 2 * b.n_levels + 2 * r.bucket + (cls - 2);
}

__global__ void item_count_kernel(const PersistPlan p, const ItemBuild b) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= b.n_pairs) return;
  const PairInfo r = pair_info(p, b, q);
  if (r.n_items)
    atomicAdd(b.cnt + item_key(p, b, r), (unsigned long long)r.n_items);
}

// exclusive scan of cnt[0, n) in place, one CTA
__global__ void __launch_bounds__(1024) item_scan_kernel(unsigned long long* cnt, int n) {
  __shared__ unsigned long long warp_sum[32];
  const int tid = threadIdx.x, per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  unsigned long long local = 0;
  for (int i = lo; i < hi; ++i) local += cnt[i];
  unsigned long long incl = local;
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, off);
    if ((tid & 31) >= off) incl += t;
  }
  if ((tid & 31) == 31) warp_sum[tid >> 5] = incl;
  __syncthreads();
  if (tid < 32) {
    unsigned long long w = tid < (int)(blockDim.x >> 5) ? warp_sum[tid] : 0ull;
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, w, off);
      if (tid >= off) w += t;
    }
    warp_sum[tid] = w;  // inclusive over warps
  }
  __syncthreads();
  unsigned long long run = incl - local + ((tid >> 5) ? warp_sum[(tid >> 5) - 1] : 0ull);
  for (int i = lo; i < hi; ++i) {
    const unsigned long long v = cnt[i];
    cnt[i] = run;
    run += v;
  }
}

__global__ void item_fill_kernel(const PersistPlan p, const ItemBuild b) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= b.n_pairs) return;
  const PairInfo r = pair_info(p, b, q);
  if (!r.n_items) return;
  const unsigned long long pos =
      atomicAdd(b.cnt + item_key(p, b, r), (unsigned long long)r.n_items);
  for (int64_t k = 0; k < r.n_items; ++k) {
    const int64_t u = b.world > 1 ? b.rank + k * b.world : k;
    b.items[pos + k] = make_int4(r.s, (int)u, (int)r.c, r.dep);
  }
}

}  // namespace

size_t chain_smem_need(int C, int AW, int W, size_t vsz) { return chain_smem_bytes(C, AW, W, vsz); }

void launch_build_items(const PersistPlan& P, const ItemBuild& B, cudaStream_t st) {
  const int n = 4 * B.n_levels;
  cudaMemsetAsync(B.cnt, 0, sizeof(unsigned long long) * (n + 1), st);
  const int threads = 256;
  const unsigned blocks = (unsigned)((B.n_pairs + threads - 1) / threads);
  if (blocks == 0) return;
  item_count_kernel<<<blocks, threads, 0, st>>>(P, B);
  item_scan_kernel<<<1, 1024, 0, st>>>(B.cnt, n);
  item_fill_kernel<<<blocks, threads, 0, st>>>(P, B);
  count_launch();
  count_launch();
  count_launch();
}

void query_persistent(const LevelLaunch& L, const PersistPlan& P, PersistInfo* info) {
  info->query_only = 1;
  dispatch(L, &P, nullptr, info);
  info->query_only = 0;
}

void launch_persistent(const LevelLaunch& L, const PersistPlan& P, cudaStream_t st,
                       PersistInfo* info) {
  dispatch(L, &P, st, info);
  count_launch();
}

}  // namespace dsg
