// dsg_device.cuh — shared definitions for the sm_100a max-load DP kernels.
//
// Data layout in HBM (all arrays are structure-of-arrays, indexed by the
// reference ordinal of an ideal, i.e. size-major then lex order exactly as
// enumerate_ideals produces, ideals.cpp:66):
//
//   abits   [I][W]   u64   closure bitset A(J): J itself (inference) or
//                          J ∪ paired backward nodes (training, dp_solver.cpp:235-250)
//   pfx_*   [I]      V     prefix sums over A(J): cpu, acc (supported), mem
//   unsup   [I]      i32   # accelerator-unsupported members of A(J)
//   fw/fwinf[I]      V/i32 Σ comm over F(A) (members with a real successor outside)
//   ftab             per-ideal source frontier table (FChunk + NItem + F weights)
//   dp      [I][C]   V     dp[ord][k][l], cell = k*(L+1)+l (dp_solver.cpp:168-170)
//   bp      [I][C]   i32   argmin: 2*prev + (cpu?1:0) for a block transition,
//                          -3/-4 waste moves (kinds 3/4), -1 none
//
// V is int32_t when the host proves every partial sum fits in 30 bits at
// the common denominator D, else int64_t.  INF is the type's max value.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace dsg {

template <typename V>
struct VTraits;
// INF: +infinity.  PENDING: a dp cell not yet final inside the persistent
// kernel (tables are reset to it before every solve; no finite value can
// reach it — the host bounds |values| below 2^30 / 2^62).
template <>
struct VTraits<int32_t> {
  static constexpr int32_t INF = 0x7fffffff;
  static constexpr int32_t PENDING = (int32_t)0x80000000;
};
template <>
struct VTraits<int64_t> {
  static constexpr int64_t INF = 0x7fffffffffffffffLL;
  static constexpr int64_t PENDING = (int64_t)0x8000000000000000ULL;
};

constexpr int kMaxWords = 64;       // bitset words supported (4096 nodes)
constexpr int kTileTargets = 128;   // targets (threads) per transition CTA

// One chunk of <= 64 frontier producers F(A') of a source ideal, with the
// upper neighbours N(A') that any of them feeds.
struct FChunk {
  int32_t n_f;      // producers in this chunk (<= 64)
  int32_t n_n;      // neighbour items
  int32_t off_f;    // into the F-weight pool
  int32_t off_n;    // into the NItem pool
  uint64_t infmask; // producers whose comm is the infinite sentinel
};

// Everything the transition kernel needs about a SOURCE ideal before its
// frontier walk, in one 64-byte record (4 x 16-byte broadcast loads):
// prefix sums over A(J) and the first frontier chunk inline.
struct __align__(16) SrcRec {
  int64_t cpu, acc, mem;
  int32_t unsup, n_chunks;
  int32_t chunk0, n_f, n_n, off_f;
  int32_t off_n, pad;
  uint64_t infmask;
};
static_assert(sizeof(SrcRec) == 64, "SrcRec is one 64-byte record");

// Upper neighbour n of the source closure: bit position of n in the target
// closure bitset, and which chunk-local producers have a real edge to n.
struct NItem {
  uint32_t word;
  uint32_t bit;
  uint64_t predmask;
};

// Training-only per-ideal lists (empty for inference graphs):
//   P'(A) = Pred_real(A) \ A  as (word, bit, weight)  [source side: comm_out]
//   L(A)  = Pred_real(A) \ A  with s_u = succ_real(u) ∩ A as (word, mask)
//           items                                    [target side: comm_in]
struct PItem {
  uint32_t word;
  uint32_t bit;
  int32_t inf;
  int32_t pad;
  int64_t weight;
};

struct LEntry {
  int32_t n_items;
  int32_t off_items;
  int32_t inf;
  int32_t pad;
  int64_t weight;
};

struct MaskItem {
  uint32_t word;
  uint32_t pad;
  uint64_t mask;
};

// Device-side view of the flattened graph (dense indices, fixed point).
struct DevGraph {
  int n;
  int W;
  const int64_t* cpu;    // fixed point
  const int64_t* acc;    // fixed point, 0 for unsupported
  const int64_t* comm;   // fixed point, 0 for the infinite sentinel
  const int64_t* mem;    // fixed point
  const uint8_t* unsup;  // acc_time infinite
  const uint8_t* comminf;// comm_time infinite
  const uint64_t* succ_real;   // [n][W]
  const uint64_t* pred_real;   // [n][W]
  const uint64_t* pred_u;      // [n][W] in_all preds restricted to the universe
  const uint64_t* succ_u;      // [n][W] out_all succs restricted to the universe
  const uint64_t* twins;       // [n][W] paired backward nodes of a forward node
  const uint64_t* bw_succ;     // [n][W] out_all succs within the backward part
  const uint64_t* bw_from;     // [n][W] reachability_within(bw).from
  const uint64_t* bw_to;       // [n][W] reachability_within(bw).to
  const uint64_t* bwset;       // [W]
  const int32_t* out_real_off; // CSR of real successors
  const int32_t* out_real_adj;
  const int32_t* in_real_off;  // CSR of real predecessors
  const int32_t* in_real_adj;
};

__device__ __forceinline__ bool bit_of(const uint64_t* s, int v) {
  return (s[v >> 6] >> (v & 63)) & 1ull;
}

}  // namespace dsg
