// dsg_internal.h — host-side launch interfaces between the C-ABI driver
// (capi.cu) and the kernel translation units.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "dsg_device.cuh"

namespace dsg {

void count_launch();  // kernels launched by this library (bench evidence)

// ---------------------------------------------------------------- K1
struct EnumStatus {
  int32_t code;      // 0 ok, 1 budget exceeded, 2 capacity, 3 candidate capacity,
                     // 4 a level wider than one CTA's frontier: resume on a cluster
  int32_t n_levels;
  int64_t total;
  int64_t needed;
  int64_t resume_lo, resume_hi;  // code 4: the level [lo, hi) to expand next
  int64_t resume_level;
};

struct EnumLaunch {
  int W, n;
  const uint64_t* pred_u;
  const uint64_t* succ_u;
  const uint8_t* in_universe;
  // universe-restricted adjacency, unique entries (nullptr: bitset path)
  const int32_t* pu_off;  // [n + 1] predecessors
  const int32_t* pu_adj;
  const int32_t* su_off;  // [n + 1] successors
  const int32_t* su_adj;
  int n_pu, n_su;
  int32_t* spill_par;  // [cap] scratch
  int32_t* spill_v;
  uint64_t* bits;
  uint64_t* maxm;
  uint64_t* addm;
  int32_t* level_of;
  int64_t cap, budget;
  int64_t* level_off;
  EnumStatus* status;
  int hash_mode;
  uint64_t* cand_bits;
  uint64_t* cand_maxm;
  uint64_t* cand_addm;
  int64_t cand_cap;
  int64_t* table;
  int64_t table_cap;
  int resume;        // 1: continue from status->resume_* on the cluster kernel
};

void launch_enumerate(const EnumLaunch& L, cudaStream_t st);
// level order (size-major, NodeSet::lex_less within a level); max_level =
// the largest level size, perm_a / perm_b: [total] scratch for large levels
// [n][W] bitset rows of the universe predecessors / successors and the real
// successors, from their CSR lists (rows zeroed by the caller)
void launch_adj_bits(int n, int W, const int32_t* pu_off, const int32_t* pu_adj, const int32_t* su_off,
                     const int32_t* su_adj, const int32_t* out_off, const int32_t* out_adj,
                     uint64_t* pred_u, uint64_t* succ_u, uint64_t* succ_real, cudaStream_t st);

// returns whether lvl_d (each level's common word prefix) was filled
bool launch_lex_rank(int W, int64_t total, const uint64_t* bits, const uint64_t* maxm,
                     const int32_t* level_of, const int64_t* level_off, uint64_t* out_bits,
                     uint64_t* out_maxm, int64_t max_level, int64_t* perm_a, int64_t* perm_b,
                     int* lvl_d, int n_levels, cudaStream_t st);
// lower covers of every ideal (ordinals one level down), CSR over ordinals
void launch_cover_count(int W, int64_t I, const uint64_t* smax, int64_t* cnt, cudaStream_t st);
void launch_cover_fill(int W, int64_t I, const uint64_t* sbits, const uint64_t* smax,
                       const int32_t* level_of, const int64_t* level_off, const int64_t* cov_off,
                       int32_t* cov, const int* lvl_pre, int* err, cudaStream_t st);

// ------------------------------------------------------- descriptors
// Per-ideal table sizes (pass 1) -> exclusive offsets (scan) -> fill (pass 2).
enum CountSlot { kCntChunks = 0, kCntF, kCntN, kCntP, kCntL, kCntLItems, kNumCounts };

struct DescribeLaunch {
  DevGraph g;
  int training;
  int has_bw;        // graph has backward nodes (bw_reach exists)
  int value_bits;    // 32 or 64
  int64_t I;
  int AW;            // abits row stride: W rounded up to even (16-byte rows)
  const uint64_t* sbits;  // sorted ideal bitsets [I][W]
  // outputs
  uint64_t* abits;   // [I][AW]
  uint64_t* intbits; // [I][W] training
  void* pfx_cpu;     // V[I]
  void* pfx_acc;
  void* pfx_mem;
  int32_t* unsup;
  void* fw;          // V[I]
  int32_t* fwinf;
  uint8_t* upset;    // training: Φ(J) is an up-set of the backward part
  SrcRec* srec;      // [I] source records
  int64_t* counts;   // [kNumCounts][I + 1]  (pass 1 output, scanned in place)
  // pools (pass 2)
  FChunk* chunks;
  void* fpool;       // V
  NItem* nitems;
  PItem* pitems;
  LEntry* lentries;
  MaskItem* litems;
};

void launch_describe(const DescribeLaunch& L, bool fill, cudaStream_t st);
// maxima of the source prefix sums (acc, mem, cpu, pad) per aligned block of
// kChunkMaxLen ordinals: out[4 * block + {0, 1, 2}]
constexpr int kChunkMaxLen = 64;
void launch_chunk_max(const SrcRec* srec, int64_t I, int64_t* out, cudaStream_t st);
void launch_scan_counts(int64_t* counts, int64_t I, int n_arrays, cudaStream_t st);

// ------------------------------------------------------- transition
struct LevelLaunch {
  int value_bits;
  int training;
  int has_bw;
  int fastgate;
  int K, L, C, W;
  int AW;              // abits row stride (even: 16-byte vector loads)
  int64_t mlim;        // fixed point (clamped)
  int memcheck;
  int interleave;
  int repl;            // replicated solve (dp_solver.cpp:100-108)
  int repl_combine;    // 0 Sum, 1 Max
  int64_t repl_bn;     // |bandwidth numerator|
  int64_t repl_bd;     // bandwidth denominator
  int repl_sign;       // sign of the bandwidth
  int no_prune;        // negative comm under Sum: the generic (unpruned) cells
  int64_t t_lo, t_hi;  // targets
  int64_t s_hi;        // sources [0, s_hi)
  int64_t n_chunks;
  int64_t chunk_len;
  // tables
  const uint64_t* abits;
  const uint64_t* intbits;
  const void* pfx_cpu;
  const void* pfx_acc;
  const void* pfx_mem;
  const int32_t* unsup;
  const void* fw;
  const int32_t* fwinf;
  const uint8_t* upset;
  const SrcRec* srec;
  const int64_t* chunk_off;   // counts[kCntChunks] scanned, [I+1]
  const FChunk* chunks;
  const void* fpool;
  const NItem* nitems;
  const int64_t* p_off;
  const PItem* pitems;
  const int64_t* l_off;
  const LEntry* lentries;
  const MaskItem* litems;
  const uint64_t* bwset;
  const uint64_t* bw_from;
  const uint64_t* bw_to;
  int n_nodes;
  // lower covers of every ideal: ordinals one level down, CSR over ordinals
  const int64_t* cov_off;     // [I + 1]
  const int32_t* cov;
  // [ceil(I / kChunkMaxLen)][4] maxima of the source prefix sums (launch_chunk_max)
  const int64_t* cmax;
  // dp
  void* dp;                   // V[I][C]
  int32_t* bp;                // [I][C]
  void* part_val;             // V[n_chunks][C][T]
  int32_t* part_arg;
  unsigned long long* pair_counter;
  // DSG_PAIR_STATS builds only: [0] pairs counted in count-only chunks,
  // [1] nested pairs dropped by the per-pair candidate test, [2] pairs whose
  // frontier walk (block cost) ran, [3] pairs whose min-max update ran
  unsigned long long* stats;
};

void launch_transition(const LevelLaunch& L, cudaStream_t st);

// One virtual rank of a sharded solve emulated on one GPU (dsg_options::
// shard_count): everything a rank of a multi-GPU solve owns on its own GPU.
// The cooperative launch gives CTA b to rank b % world.
struct VRank {
  const int4* items;          // this rank's readiness-ordered item list
  int64_t total_items;
  unsigned* ctl;              // [0] stop [1] err [2..3] claim counter [32 + s] level s done
  unsigned* tile_count;       // arrival counters of this rank's units
  unsigned long long* keys;   // merge keys of this rank's targets
  void* dp;                   // this rank's replica of the dp table (read by its CTAs)
  const int4* run_items;      // the rank's chain-runner items (finishers, level order)
  int64_t run_total;
};

// One cooperative launch for all levels (transition.cu).
struct PersistPlan {
  int n_levels;
  const int64_t* level_off;  // [n_levels + 1]
  const int32_t* mode;       // [n_levels] 0: lanes own targets, 1: lanes own sources
  const int64_t* n_chunks;   // [n_levels] source chunks per target (group)
  const int64_t* chunk_len;  // [n_levels] (unused by the dataflow kernel)
  // mode-0 chunks are implicit: with R = level_off[s-1] (start of the
  // newest source level) and n_old = ceil(R / chunk_len0), chunk c < n_old
  // covers [c*chunk_len0, min(.. + chunk_len0, R)) and chunk n_old + j the
  // newest level's [R + j*chunk_len1, min(.. + chunk_len1, S)) — short,
  // because those items gate level s.  Mode-1 levels list their
  // boundaries: [chunk_lo[b+c], chunk_lo[b+c+1]), b = chunk_base[s].
  int chunk_len0, chunk_len1;
  int grade;                 // recent levels chunked by slack (see mode0_chunk)
  int stage;                 // stage old mode-0 chunks in shared memory
  int dead_skip;             // count-only scans of chunks that cannot change a cell
  unsigned poll_ns_max;      // dependency-wait backoff cap
  unsigned fin_poll_ns;    // narrow-level cell polls: backoff cap (0 = spin)
  int chain;               // runner lists hold chain blocks (persistent_impl.cuh)
  const int64_t* chunk_lo;
  const int64_t* chunk_base;
  const int64_t* tile_base;  // [n_levels] prefix of arrival counters over levels
  // Work items (s, unit, chunk, dep) sorted by readiness: dep = the level
  // of the chunk's last source (the only level the item waits for — levels
  // complete in order), then target level s.  CTAs claim them in this order
  // from one atomic counter, so a CTA never sits on an unready item while
  // ready ones are queued behind it.
  const int4* items;         // [total_items]
  unsigned long long* next;  // claim counter, zeroed per solve
  unsigned long long* crit_next;  // claim counter of the cover-item queue
  int crit_ctas;                  // CTAs that run only cover items (0: one queue)
  const unsigned long long* crit_end;  // -> number of cover items (after the build)
  const int32_t* level_of;   // [I] level of each ordinal
  int64_t total_items;
  unsigned* tile_count;      // [total counters], zeroed
  unsigned* done;            // [n_levels] finished targets per level, zeroed
  int* stop;                 // deadline reached / abort
  int* err;                  // watchdog fired
  int64_t deadline_ns;       // %globaltimer deadline, 0 = none
  uint64_t* trace;           // optional [total_items][4] timestamps (DSG_TRACE_FILE)
  unsigned long long* keys;  // [I][C] packed (value^sign, arg) for mode-0 merges of
                             // 32-bit values; 0xff.. = no candidate
  // Wavefront sharding over GPUs (one process per GPU): this rank owns the
  // target units with unit % world == rank; finalized dp/bp rows are stored
  // into every rank's tables over NVLink (peer pointers from CUDA IPC) and
  // every rank's level counter is bumped with a system-scope atomic.
  // world == 1: the tables point at this GPU's own buffers.
  int rank, world;
  void* const* peer_dp;        // [world] dp table of each rank
  int32_t* const* peer_bp;     // [world]
  unsigned* const* peer_done;  // [world] level counters of each rank (ctl + 32:
                               // the rank's stop / err words sit at -32 / -31)
  // virt != 0: all `world` ranks run in this one launch (virtual shards on
  // one GPU); CTA b is rank b % world and takes its tables from vrank[rank]
  int virt;
  const VRank* vrank;          // [world]
  // Chain runner: one CTA per rank (blockIdx.x == rank, or 0) first runs the
  // finishers of the narrow mode-1 levels in level order from its own list —
  // no claims, no queueing behind other items on the level-to-level chain —
  // then joins the shared queue.  run_items / run_total: this launch's own
  // rank (virtual ranks: VRank::run_items).
  int runner_max_t;
  int runners;               // CTAs per rank sharing the run list round-robin, so each
                             // prepares its next finisher while the chain advances
  const int4* run_items;
  int64_t run_total;
};

struct PersistInfo {
  int query_only;
  int blocks;      // in: requested grid (0 = full residency); out: launched grid
  int per_sm;      // resident CTAs per SM
  int launch_error;
};

// Device-side item list (persistent.cu): counting sort of every (level,
// chunk) pair's units by dependency level, the critical items (target level
// = dep + 1) first inside each bucket.
struct ItemBuild {
  int n_levels;
  int runner_max_t;          // > 0: finishers of mode-1 levels with <= this many
                             // targets go to the chain runner, not the list
  int lag;                   // list bucket = max(dep, s - lag)
  int split;                 // cover items in their own queue at the front
  const int64_t* pair_off;   // [n_levels + 1] prefix of chunks over levels
  int64_t n_pairs;
  unsigned long long* cnt;   // [2 * n_levels + 1] scratch
  int4* items;               // [total_items] out
  int rank, world;
};
// chain blocks (persistent_impl.cuh): fold sources per chain level, and the
// shared memory a chain block needs (inside the old-chunk staging area)
constexpr int kChainSrcMax = 32;
size_t chain_smem_need(int C, int AW, int W, size_t vsz);

void launch_build_items(const PersistPlan& P, const ItemBuild& B, cudaStream_t st);

void query_persistent(const LevelLaunch& L, const PersistPlan& P, PersistInfo* info);
void launch_persistent(const LevelLaunch& L, const PersistPlan& P, cudaStream_t st,
                       PersistInfo* info);
void launch_read_globaltimer(uint64_t* out, cudaStream_t st);
void launch_fill_u32(unsigned* p, int64_t n, unsigned value, cudaStream_t st);
void launch_finalize(const LevelLaunch& L, cudaStream_t st);
void launch_init_empty(int value_bits, int K, int L, void* dp, cudaStream_t st);
// *bad = 1 if the two tables differ anywhere (virtual-shard replicas)
void launch_compare_tables(const void* a, const void* b, size_t bytes, int* bad, cudaStream_t st);
void launch_fill_inf(int value_bits, void* p, int64_t n, cudaStream_t st);
// dp cells -> VTraits<V>::PENDING (rows polled by narrow-level items)
void launch_fill_pending(int value_bits, void* p, int64_t n, cudaStream_t st);
void launch_level_of(const int64_t* level_off, int n_levels, int64_t I, int32_t* level_of,
                     cudaStream_t st);

// Traceback state on the device (transition.cu).
struct TraceState {
  int64_t ord;
  int32_t k, l;
  int32_t status;   // 0 walking, 1 done, 2 infeasible, 3 stuck
  int32_t n_blocks;
  int32_t best_k, best_l;
  int64_t best_value;
  uint32_t arrivals;  // search CTAs done this step; the last one decides
};

struct TraceBuffers {
  TraceState* state;
  void* part_v;          // [n_parts] per-CTA direct minimum
  int32_t* part_g;       // [n_parts] its smallest argmin
  int n_parts;
  int64_t* ords;         // [K+L+1] one entry per block
  int64_t* prevs;
  int32_t* kinds;        // cpu | repl << 1
  uint64_t* block_bits;  // [K+L+1][W]
  int64_t* loads;        // [K+L+1] per-device load of each block (INT64_MAX = inf)
  const int* abort;      // [2] persistent stop / watchdog flags, or null: set -> status 3
};

void launch_traceback(const LevelLaunch& L, const int32_t* level_of, const int64_t* level_off,
                      int64_t I, int sm_count, TraceBuffers& b, cudaStream_t st);

}  // namespace dsg
