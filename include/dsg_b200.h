/*
 * dsg_b200.h — C-ABI of the B200-native max-load DP over ideals.
 *
 * This is the drop-in boundary for the hot path of the reference `dagsplit`
 * library (Tarnawski et al. 2020, arXiv 2006.16423).  Everything here is plain
 * C: POD structs, pointers and sizes, no C++ or torch types.  The same struct
 * layout is implemented by three libraries:
 *
 *   libdsg_b200.so      the product: CUDA kernels for sm_100a   (dsg_*)
 *   libdsg_oracle.so    CPU restatement used only by tests      (dsgo_*)
 *   libdsg_ref.so       the unmodified reference, test-only     (dsgref_*)
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/proj):
 *
 *   dsg_dp_solve(DSG_MODE_INFERENCE, ...)
 *       Split solve_maxload_inference(const Graph&, const DeviceConfig&,
 *                                     const SolveOptions&)
 *       include/dagsplit/dp_solver.hpp:21-22, src/dp_solver.cpp:387-390
 *   dsg_dp_solve(DSG_MODE_TRAINING, ...)
 *       Split solve_maxload_training(...)
 *       include/dagsplit/dp_solver.hpp:28-29, src/dp_solver.cpp:392-395
 *   dsg_dp_solve(DSG_MODE_REPLICATED, ...)
 *       Split solve_maxload_replicated(...)
 *       include/dagsplit/dp_solver.hpp:36-37, src/dp_solver.cpp:397-405
 *   dsg_enumerate_ideals(...)
 *       IdealIndex enumerate_ideals(const Graph&, long long budget)
 *       IdealIndex enumerate_ideals_within(const Graph&, const NodeSet&, ...)
 *       include/dagsplit/graph.hpp:253-258, src/ideals.cpp:79-86
 *
 * The graph is passed exactly as the reference's Graph holds it
 * (include/dagsplit/graph.hpp:19-39, 152-186): nodes with external ids and
 * exact rational weights, real edges (carry communication) and artificial
 * edges (precedence only), by external id.  Edges whose endpoints do not
 * resolve are skipped, and on duplicate ids the first node wins, as in
 * Graph::Graph (src/graph.cpp:132-158).
 *
 * Errors: the reference throws C++ exceptions; here every entry point
 * returns a dsg_status and fills `message`.  The mapping back to the
 * reference's exception types is in INTEGRATION.md.
 */
#ifndef DSG_B200_H
#define DSG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSG_ABI_VERSION 2
#define DSG_NO_PAIR INT32_MIN
/* reference kDefaultIdealBudget, include/dagsplit/graph.hpp:251 */
#define DSG_DEFAULT_IDEAL_BUDGET 5000000LL

/* Exact rational like the reference Rat (include/dagsplit/rational.hpp:18-78):
 * den > 0 for finite values, den == 0 means +infinity. */
typedef struct dsg_rat {
  int64_t num;
  int64_t den;
} dsg_rat;

typedef struct dsg_graph {
  int32_t n_nodes;
  const int32_t* ids;         /* external ids, n_nodes */
  const dsg_rat* cpu_time;    /* Node::cpu_time */
  const dsg_rat* acc_time;    /* Node::acc_time; infinite = unsupported */
  const dsg_rat* comm_time;   /* Node::comm_time */
  const dsg_rat* mem_size;    /* Node::mem_size */
  const uint8_t* is_backward; /* may be NULL (inference graph) */
  const int32_t* forward_pair;/* external id or DSG_NO_PAIR; may be NULL */
  int32_t n_edges;            /* real edges (communication + precedence) */
  const int32_t* edge_from;
  const int32_t* edge_to;
  int32_t n_artificial;       /* artificial edges (precedence only) */
  const int32_t* art_from;
  const int32_t* art_to;
} dsg_graph;

enum dsg_interleaving {
  DSG_INTERLEAVE_SUM = 0,             /* Interleaving::Sum */
  DSG_INTERLEAVE_HALF_DUPLEX_MAX = 1, /* Interleaving::HalfDuplexMax */
  DSG_INTERLEAVE_FULL_DUPLEX_MAX = 2  /* Interleaving::FullDuplexMax */
};

enum dsg_replication_combine { DSG_REPL_SUM = 0, DSG_REPL_MAX = 1 };

/* DeviceConfig, include/dagsplit/graph.hpp:98-106 */
typedef struct dsg_config {
  int32_t accelerators; /* k */
  int32_t cpus;         /* l */
  dsg_rat memory_limit; /* den == 0: unlimited */
  int32_t q;            /* unused by the DP (contiguous, q = 1) */
  int32_t interleaving;
  int32_t has_bandwidth;
  dsg_rat bandwidth;
  int32_t replication_combine;
} dsg_config;

enum dsg_mode {
  DSG_MODE_INFERENCE = 0,
  DSG_MODE_TRAINING = 1,
  DSG_MODE_REPLICATED = 2
};

/* SolveOptions, include/dagsplit/dp_solver.hpp:11-14, plus device knobs. */
typedef struct dsg_options {
  int64_t ideal_budget;    /* IdealBudgetExceeded iff #ideals > budget */
  double deadline_seconds; /* relative to the call; <= 0 means no deadline */
  int32_t device;          /* CUDA ordinal, -1 = current device */
  int32_t shard_count;     /* wavefront shards (virtual on one GPU); 0/1 = off */
  int32_t flags;           /* DSG_FLAG_* */
  int32_t reserved;        /* > 0: cap on persistent-kernel CTAs (testing) */
} dsg_options;

#define DSG_FLAG_FORCE_INT64 1   /* never use the 32-bit value path */
#define DSG_FLAG_NO_FASTGATE 2   /* training: always run the general gate */
#define DSG_FLAG_HASH_ENUM 4     /* enumerate with the GPU hash set */
#define DSG_FLAG_KEEP_TABLES 8   /* keep ideal list + dp table for inspection */
#define DSG_FLAG_TIME_KERNELS 16 /* CUDA-event time every transition launch */
#define DSG_FLAG_LEVEL_LAUNCH 32 /* one launch pair per level instead of the
                                    persistent cooperative level kernel */

enum dsg_status {
  DSG_OK = 0,
  DSG_INFEASIBLE = 1,        /* InfeasibleError          errors.hpp:8-10 */
  DSG_BUDGET = 2,            /* IdealBudgetExceeded{limit} graph.hpp:239-241 */
  DSG_DEADLINE = 3,          /* DeadlineExceeded         errors.hpp:12-14 */
  DSG_INVALID = 4,           /* std::invalid_argument    dp_solver.cpp:143,152-157 */
  DSG_OVERFLOW = 5,          /* std::overflow_error      rational.cpp:16-21 */
  DSG_MISSING_BANDWIDTH = 6, /* MissingBandwidth         errors.hpp:21-24 */
  DSG_CUDA_ERROR = 7,        /* no reference analogue: device failure */
  DSG_LOGIC = 8,             /* std::logic_error         dp_solver.cpp:357 */
  DSG_UNSUPPORTED = 9        /* valid request this build does not implement */
};

/* One device block of the optimal split, before canonical numbering
 * (SplitBlock, include/dagsplit/graph.hpp:279-283). */
typedef struct dsg_block {
  int32_t cpu;       /* 1 = CPU device, 0 = accelerator */
  int32_t repl;      /* accelerator replica count (1 unless replicated) */
  int32_t n_members;
  int32_t offset;    /* into dsg_result::members */
  int64_t load_num;  /* per-device load of the block (acc_cost / cpu_cost /
                        replicated_load, graph.cpp:397-479) recomputed by the
                        device at denominator dsg_result::denominator;
                        INT64_MAX = infinite; valid iff dsg_result::block_loads */
} dsg_block;

typedef struct dsg_result {
  int32_t status;
  char message[256];
  int64_t budget_limit;   /* DSG_BUDGET: the limit that was exceeded */
  dsg_rat objective;      /* reduced; equals the reference Rat */
  int32_t best_k, best_l; /* fewest-devices cell, dp_solver.cpp:337-351 */
  int32_t n_blocks;
  dsg_block* blocks;      /* callee-allocated; free with dsg_result_free */
  int32_t* members;       /* dense node indices (graph order) */
  int64_t n_ideals;
  int64_t n_pairs;        /* nested pairs I' < I evaluated (transitions) */
  int32_t n_levels;
  int32_t value_bits;     /* 32 or 64: fixed-point width used on device */
  int64_t denominator;    /* common fixed-point denominator D */
  int64_t kernel_launches;
  double t_prepare_ms;    /* host flatten + fixed point + H2D */
  double t_enumerate_ms;  /* K1 lattice enumeration + lex ordering */
  double t_describe_ms;   /* per-ideal descriptors */
  double t_dp_ms;         /* all transition levels */
  double t_traceback_ms;  /* traceback + D2H */
  double t_total_ms;
  double t_transition_kernel_ms; /* sum of transition-kernel event times */
  double t_device_ms;     /* CUDA-event time of the device pipeline (first
                             enumeration launch .. last result copy) */
  int64_t h2d_bytes;      /* host->device bytes copied by this call */
  int64_t d2h_bytes;      /* device->host bytes copied by this call */
  int32_t persistent_blocks; /* CTAs of the persistent level kernel (0: per-level launches) */
  int32_t block_loads;       /* 1: dsg_block::load_num is filled */
  /* DSG_FLAG_KEEP_TABLES: */
  int32_t words;            /* 64-bit words per ideal bitset */
  uint64_t* ideal_bits;     /* n_ideals * words, reference ordinal order */
  int64_t* dp_values;       /* n_ideals * (k+1)*(l+1), fixed point, INT64_MAX = inf */
} dsg_result;

typedef struct dsg_ideals {
  int32_t status;
  char message[256];
  int64_t budget_limit;
  int64_t count;
  int32_t words;          /* 64-bit words per bitset = ceil(n_nodes/64) */
  uint64_t* bits;         /* count * words, size-major then lex (ideals.cpp:66) */
  int32_t n_levels;
  int64_t* level_offsets; /* n_levels + 1 */
  double t_ms;
} dsg_ideals;

/* Max-load DP.  Returns result->status. */
int dsg_dp_solve(int32_t mode, const dsg_graph* graph, const dsg_config* config,
                 const dsg_options* options, dsg_result* result);
void dsg_result_free(dsg_result* result);

/* Ideal enumeration.  within: per dense node index, nonzero = inside the
 * universe; NULL = whole graph (enumerate_ideals). */
int dsg_enumerate_ideals(const dsg_graph* graph, const uint8_t* within,
                         int64_t budget, const dsg_options* options,
                         dsg_ideals* out);
void dsg_ideals_free(dsg_ideals* out);

/* Resident session: flatten + fixed point + upload once, then run the device
 * pipeline any number of times with the graph already in HBM (the same
 * computation as dsg_dp_solve minus the host preparation and input copies).
 * status_out->status reports creation errors; NULL on failure. */
typedef struct dsg_session dsg_session;
dsg_session* dsg_session_create(int32_t mode, const dsg_graph* graph, const dsg_config* config,
                                const dsg_options* options, dsg_result* status_out);
int dsg_session_run(dsg_session* session, dsg_result* result);
void dsg_session_destroy(dsg_session* session);

/* Multi-GPU wavefront (one process per GPU).  Every rank
 * creates a session for the same graph, then:
 *   dsg_session_shard_prepare(s, rank, world, &mine)   lattice + tables, export IPC handles
 *   <all-gather the world handles in rank order>       (e.g. torch.distributed)
 *   dsg_session_shard_attach(s, all)                   open the peers' tables (NVLink P2P)
 * and per solve:
 *   dsg_session_shard_reset(s)  ->  <barrier across ranks>  ->  dsg_session_run(s)
 *   ->  <barrier across ranks>.
 * Rank r owns the target units u with u % world == r; its finalizers store
 * the finished dp rows into every rank's table and bump every rank's level
 * counter, so no host-side collective runs per level.  Rank 0 returns the
 * split; the others return status and their transition counts. */
#define DSG_MAX_SHARDS 64
typedef struct dsg_shard_handle {
  int32_t rank;
  int32_t device;
  int64_t n_ideals;
  uint8_t dp[64];   /* cudaIpcMemHandle_t of the dp table */
  uint8_t bp[64];   /* ... back pointers */
  uint8_t ctl[64];  /* ... control words (level counters at +32) */
} dsg_shard_handle;

int dsg_session_shard_prepare(dsg_session* session, int32_t rank, int32_t world,
                              dsg_shard_handle* handle_out, dsg_result* status_out);
int dsg_session_shard_attach(dsg_session* session, const dsg_shard_handle* all_handles,
                             dsg_result* status_out);
int dsg_session_shard_reset(dsg_session* session, dsg_result* status_out);
/* Re-flatten and re-upload a (same-shaped) graph into a session: the
 * host->device leg of an end-to-end solve without re-attaching peers. */
int dsg_session_reload(dsg_session* session, const dsg_graph* graph, const dsg_config* config,
                       dsg_result* status_out);

void dsg_default_options(dsg_options* options);
const char* dsg_version(void);
/* Number of CUDA devices visible (0 if none); never fails. */
int dsg_device_count(void);
/* Number of kernels this library launched since load (for bench evidence). */
int64_t dsg_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* DSG_B200_H */
