// persistent_g_i64_inf.cu — general i64 inference variants of the dataflow level kernel
// (persistent_impl.cuh), in their own translation unit so nvcc compiles the
// variants in parallel.
#include "persistent_impl.cuh"

namespace dsg {

bool dispatch_exact_i64_inf(const LevelLaunch& L, const PersistPlan* P, cudaStream_t st,
                            PersistInfo* info) {
  // exact words and cells for K = 8, L = 0 on the 64-bit path (graphs whose
  // proven bound passes 2^30, e.g. many-decimal weights)
  using V = int64_t;
  constexpr bool TRAIN = false;
  if (L.repl || L.no_prune || L.L != 0 || L.K != 8) return false;
  if (L.AW == 2) return run_variant<V, 1, 9, TRAIN, 2, true>(L, P, st, info), true;
  if (L.AW == 4) return run_variant<V, 1, 9, TRAIN, 4, true>(L, P, st, info), true;
  if (L.AW == 6) return run_variant<V, 1, 9, TRAIN, 6, true>(L, P, st, info), true;
  if (L.AW == 8) return run_variant<V, 1, 9, TRAIN, 8, true>(L, P, st, info), true;
  return false;
}

void dispatch_general_i64_inf(const LevelLaunch& L, const PersistPlan* P, cudaStream_t st,
                                PersistInfo* info) {
  using V = int64_t;
  constexpr bool TRAIN = false;
  const int lp1 = L.L + 1, kp1 = L.K + 1;
  // replication and unprunable weights: generic cells (no pruning)
  if (L.repl || L.no_prune) return run_variant<V, 0, 0, TRAIN>(L, P, st, info);
  if (lp1 == 1 && kp1 <= 9) return run_variant<V, 1, 9, TRAIN>(L, P, st, info);
  if (lp1 == 1 && kp1 <= 17) return run_variant<V, 1, 17, TRAIN>(L, P, st, info);
  if (lp1 == 2 && kp1 <= 9) return run_variant<V, 2, 9, TRAIN>(L, P, st, info);
  if (lp1 == 3 && kp1 <= 9) return run_variant<V, 3, 9, TRAIN>(L, P, st, info);
  if (lp1 == 5 && kp1 <= 9) return run_variant<V, 5, 9, TRAIN>(L, P, st, info);
  return run_variant<V, 0, 0, TRAIN>(L, P, st, info);
}

}  // namespace dsg
