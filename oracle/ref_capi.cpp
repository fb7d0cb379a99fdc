// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// Exposes the UNMODIFIED reference solver (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/) behind the
// same POD ABI as the product (include/dsg_b200.h), so tests and bench.py's
// reference arm can run both on identical inputs.  Nothing here reimplements
// the algorithm: it converts POD <-> dagsplit::Graph/Split and calls
//   solve_maxload_inference / _training / _replicated  (src/dp_solver.cpp:387-405)
//   enumerate_ideals / enumerate_ideals_within         (src/ideals.cpp:79-86)
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "dagsplit/dp_solver.hpp"
#include "dagsplit/errors.hpp"
#include "dagsplit/graph.hpp"
#include "dsg_oracle.h"

using namespace dagsplit;

namespace {

Rat to_rat(dsg_rat r) {
  if (r.den == 0) return Rat::infinity();
  return Rat(static_cast<long long>(r.num), static_cast<long long>(r.den));
}

dsg_rat from_rat(const Rat& r) {
  dsg_rat o;
  if (r.is_infinite()) {
    o.num = 1;
    o.den = 0;
  } else {
    o.num = r.numerator();
    o.den = r.denominator();
  }
  return o;
}

Graph to_graph(const dsg_graph* g) {
  std::vector<Node> nodes;
  nodes.reserve(g->n_nodes);
  for (int i = 0; i < g->n_nodes; ++i) {
    Node n;
    n.id = g->ids[i];
    n.cpu_time = to_rat(g->cpu_time[i]);
    n.acc_time = to_rat(g->acc_time[i]);
    n.comm_time = to_rat(g->comm_time[i]);
    n.mem_size = to_rat(g->mem_size[i]);
    n.is_backward = g->is_backward ? g->is_backward[i] != 0 : false;
    if (g->forward_pair && g->forward_pair[i] != DSG_NO_PAIR) n.forward_pair = g->forward_pair[i];
    nodes.push_back(std::move(n));
  }
  std::vector<Edge> edges, art;
  for (int e = 0; e < g->n_edges; ++e) edges.push_back(Edge{g->edge_from[e], g->edge_to[e], {}});
  for (int e = 0; e < g->n_artificial; ++e) art.push_back(Edge{g->art_from[e], g->art_to[e], {}});
  return Graph(std::move(nodes), std::move(edges), std::move(art));
}

DeviceConfig to_config(const dsg_config* c) {
  DeviceConfig cfg;
  cfg.accelerators = c->accelerators;
  cfg.cpus = c->cpus;
  cfg.memory_limit = to_rat(c->memory_limit);
  cfg.q = c->q > 0 ? c->q : 1;
  cfg.interleaving = c->interleaving == DSG_INTERLEAVE_HALF_DUPLEX_MAX ? Interleaving::HalfDuplexMax
                     : c->interleaving == DSG_INTERLEAVE_FULL_DUPLEX_MAX ? Interleaving::FullDuplexMax
                                                                        : Interleaving::Sum;
  if (c->has_bandwidth) cfg.bandwidth = to_rat(c->bandwidth);
  cfg.replication_combine =
      c->replication_combine == DSG_REPL_MAX ? ReplicationCombine::Max : ReplicationCombine::Sum;
  return cfg;
}

void set_msg(char* dst, const std::string& s) {
  std::strncpy(dst, s.c_str(), 255);
  dst[255] = 0;
}

template <typename F>
int guarded(char* msg, int64_t* budget_limit, F&& f) {
  try {
    f();
    return DSG_OK;
  } catch (const InfeasibleError& e) {
    set_msg(msg, e.what());
    return DSG_INFEASIBLE;
  } catch (const DeadlineExceeded& e) {
    set_msg(msg, e.what());
    return DSG_DEADLINE;
  } catch (const MissingBandwidth& e) {
    set_msg(msg, e.what());
    return DSG_MISSING_BANDWIDTH;
  } catch (const IdealBudgetExceeded& e) {
    if (budget_limit) *budget_limit = e.limit;
    set_msg(msg, "ideal budget exceeded");
    return DSG_BUDGET;
  } catch (const std::overflow_error& e) {
    set_msg(msg, e.what());
    return DSG_OVERFLOW;
  } catch (const std::invalid_argument& e) {
    set_msg(msg, e.what());
    return DSG_INVALID;
  } catch (const std::domain_error& e) {
    set_msg(msg, e.what());
    return DSG_INVALID;
  } catch (const std::logic_error& e) {
    set_msg(msg, e.what());
    return DSG_LOGIC;
  } catch (const std::exception& e) {
    set_msg(msg, e.what());
    return DSG_LOGIC;
  }
}

}  // namespace

namespace {

// mode DSG_MODE_* or kModeDpl (solve_dpl with `seed`, dp_solver.cpp:462-477)
constexpr int32_t kModeDpl = 100;

int solve_into(int32_t mode, uint64_t seed, const dsg_graph* graph, const dsg_config* config,
               const dsg_options* options, dsg_result* result) {
  std::memset(result, 0, sizeof *result);
  result->best_k = result->best_l = -1;
  result->n_pairs = -1;
  auto t0 = std::chrono::steady_clock::now();
  int st = guarded(result->message, &result->budget_limit, [&] {
    Graph g = to_graph(graph);
    DeviceConfig cfg = to_config(config);
    SolveOptions opt;
    opt.ideal_budget = options ? options->ideal_budget : kDefaultIdealBudget;
    if (options && options->deadline_seconds > 0) {
      opt.deadline = std::chrono::steady_clock::now() +
                     std::chrono::nanoseconds(static_cast<long long>(options->deadline_seconds * 1e9));
    }
    Split s = mode == kModeDpl              ? solve_dpl(g, cfg, seed, opt)
              : mode == DSG_MODE_TRAINING   ? solve_maxload_training(g, cfg, opt)
              : mode == DSG_MODE_REPLICATED ? solve_maxload_replicated(g, cfg, opt)
                                            : solve_maxload_inference(g, cfg, opt);
    result->objective = from_rat(s.objective_value);
    // group the canonical assignment back into blocks
    std::map<std::string, std::vector<int>> by_label;
    std::map<std::string, bool> is_cpu;
    for (const auto& [id, pl] : s.assignment) {
      auto idx = g.index_of(id);
      if (!idx) continue;
      by_label[pl.label()].push_back(*idx);
      is_cpu[pl.label()] = pl.is_cpu();
    }
    int n_blocks = static_cast<int>(by_label.size());
    result->blocks = static_cast<dsg_block*>(std::calloc(n_blocks + 1, sizeof(dsg_block)));
    result->members = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (g.size() + 1)));
    int b = 0, off = 0;
    for (auto& [label, mem] : by_label) {
      dsg_block& blk = result->blocks[b++];
      blk.cpu = is_cpu[label] ? 1 : 0;
      auto rit = s.replication.find(label);
      blk.repl = rit == s.replication.end() ? 1 : rit->second;
      blk.offset = off;
      blk.n_members = static_cast<int32_t>(mem.size());
      for (int v : mem) result->members[off++] = v;
    }
    result->n_blocks = n_blocks;
  });
  result->status = st;
  result->t_total_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return st;
}

}  // namespace

extern "C" int dsgref_dp_solve(int32_t mode, const dsg_graph* graph, const dsg_config* config,
                               const dsg_options* options, dsg_result* result) {
  return solve_into(mode, 0, graph, config, options, result);
}

// solve_dpl (dp_solver.cpp:462-477) and seeded_topo_order (407-438): the
// checkers for the DPL row of SURVEY 8(f).
extern "C" int dsgref_dpl_solve(const dsg_graph* graph, const dsg_config* config, uint64_t seed,
                                const dsg_options* options, dsg_result* result) {
  return solve_into(kModeDpl, seed, graph, config, options, result);
}

extern "C" int dsgref_topo_order(const dsg_graph* graph, uint64_t seed, int32_t* out) {
  Graph g = to_graph(graph);
  std::vector<int> order = seeded_topo_order(g, seed);
  for (size_t i = 0; i < order.size(); ++i) out[i] = order[i];
  return static_cast<int>(order.size());
}

extern "C" void dsgref_result_free(dsg_result* r) {
  if (!r) return;
  std::free(r->blocks);
  std::free(r->members);
  std::free(r->ideal_bits);
  std::free(r->dp_values);
  r->blocks = nullptr;
  r->members = nullptr;
  r->ideal_bits = nullptr;
  r->dp_values = nullptr;
}

extern "C" int dsgref_enumerate_ideals(const dsg_graph* graph, const uint8_t* within,
                                       int64_t budget, const dsg_options*, dsg_ideals* out) {
  std::memset(out, 0, sizeof *out);
  auto t0 = std::chrono::steady_clock::now();
  int st = guarded(out->message, &out->budget_limit, [&] {
    Graph g = to_graph(graph);
    IdealIndex ix;
    if (within) {
      NodeSet w(g.size());
      for (int v = 0; v < g.size(); ++v)
        if (within[v]) w.insert(v);
      ix = enumerate_ideals_within(g, w, budget);
    } else {
      ix = enumerate_ideals(g, budget);
    }
    int W = (g.size() + 63) / 64;
    out->count = ix.count();
    out->words = W;
    out->bits = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (ix.count() * W + 1)));
    for (long long i = 0; i < ix.count(); ++i) {
      auto words = ix.ideals[i].words();
      for (int w = 0; w < W; ++w) out->bits[i * W + w] = words[w];
    }
    std::vector<int64_t> offs{0};
    int prev = 0;
    for (long long i = 0; i < ix.count(); ++i) {
      int c = ix.ideals[i].count();
      if (i > 0 && c != prev) offs.push_back(i);
      prev = c;
    }
    offs.push_back(ix.count());
    out->n_levels = static_cast<int32_t>(offs.size() - 1);
    out->level_offsets = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * offs.size()));
    for (size_t i = 0; i < offs.size(); ++i) out->level_offsets[i] = offs[i];
  });
  out->status = st;
  out->t_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return st;
}

extern "C" void dsgref_ideals_free(dsg_ideals* out) {
  if (!out) return;
  std::free(out->bits);
  std::free(out->level_offsets);
  out->bits = nullptr;
  out->level_offsets = nullptr;
}
