// persistent_g_i64_train.cu — general i64 training variants of the dataflow level kernel
// (persistent_impl.cuh), in their own translation unit so nvcc compiles the
// variants in parallel.
#include "persistent_impl.cuh"

namespace dsg {

bool dispatch_exact_i64_train(const LevelLaunch&, const PersistPlan*, cudaStream_t, PersistInfo*) {
  return false;  // exact variants are int32-only
}

void dispatch_general_i64_train(const LevelLaunch& L, const PersistPlan* P, cudaStream_t st,
                                PersistInfo* info) {
  using V = int64_t;
  constexpr bool TRAIN = true;
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
