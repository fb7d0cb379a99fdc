// persistent_x_i32_inf.cu — exact-word / small-W i32 inference variants of the dataflow level kernel
// (persistent_impl.cuh), in their own translation unit so nvcc compiles the
// variants in parallel.
#include "persistent_impl.cuh"

namespace dsg {

bool dispatch_exact_i32_inf(const LevelLaunch& L, const PersistPlan* P, cudaStream_t st,
                              PersistInfo* info) {
  using V = int32_t;
  constexpr bool TRAIN = false;
  const int lp1 = L.L + 1, kp1 = L.K + 1;
  // replication and unprunable weights: generic cells (no pruning)
  if (L.repl || L.no_prune) return false;
  if (lp1 == 1 && kp1 == 9) {
    // exact words and cells: no predicates in the hot loop (C2: K=8, L=0;
    // the sweep up to 2,048 nodes: C5 top, AW = 12, DP 13.5 -> 9.8 ms)
    if (L.AW == 2) return run_variant<V, 1, 9, TRAIN, 2, true>(L, P, st, info), true;
    if (L.AW == 4) return run_variant<V, 1, 9, TRAIN, 4, true>(L, P, st, info), true;
    if (L.AW == 6) return run_variant<V, 1, 9, TRAIN, 6, true>(L, P, st, info), true;
    if (L.AW == 8) return run_variant<V, 1, 9, TRAIN, 8, true>(L, P, st, info), true;
#ifndef DSG_NO_WIDE_EXACT  // (A/B builds)
    if (L.AW == 10) return run_variant<V, 1, 9, TRAIN, 10, true>(L, P, st, info), true;
    if (L.AW == 12) return run_variant<V, 1, 9, TRAIN, 12, true>(L, P, st, info), true;
    if (L.AW == 16) return run_variant<V, 1, 9, TRAIN, 16, true>(L, P, st, info), true;
    if (L.AW == 24) return run_variant<V, 1, 9, TRAIN, 24, true>(L, P, st, info), true;
    if (L.AW == 32) return run_variant<V, 1, 9, TRAIN, 32, true>(L, P, st, info), true;
#endif
  }
  if (lp1 == 3 && kp1 == 7) {  // C3: K=6, L=2
    if (L.AW == 2) return run_variant<V, 3, 7, TRAIN, 2, true>(L, P, st, info), true;
    if (L.AW == 4) return run_variant<V, 3, 7, TRAIN, 4, true>(L, P, st, info), true;
  }
  // small bitsets: target words in registers
  if (L.W <= 8) {
    if (lp1 == 1 && kp1 <= 9) return run_variant<V, 1, 9, TRAIN, 8>(L, P, st, info), true;
    if (lp1 == 1 && kp1 <= 17) return run_variant<V, 1, 17, TRAIN, 8>(L, P, st, info), true;
    if (lp1 == 2 && kp1 <= 9) return run_variant<V, 2, 9, TRAIN, 8>(L, P, st, info), true;
  }
  return false;
}

}  // namespace dsg
