// dp_solver_b200.cpp — the reference-side binding: a drop-in replacement
// for /root/reference/proj/src/dp_solver.cpp and src/ideals.cpp that runs
// the DP and the ideal enumeration on the B200 through the C-ABI
// (include/dsg_b200.h).
//
// It is compiled against the reference's own headers
// (include/dagsplit/*.hpp) and linked with the rest of the reference
// library, so every caller — the CLI's cmd_solve, the acceptance suite, the
// unit suites — is source-compatible.  Implements, with the
// reference's signatures, contracts and exception types:
//
//   solve_maxload_inference / _training / _replicated   dp_solver.hpp:21-37
//   seeded_topo_order / linearize / solve_dpl           dp_solver.hpp:41-52
//   enumerate_ideals / enumerate_ideals_within          graph.hpp:253-258
//
// The split is finished exactly like MaxloadDp::run does (dp_solver.cpp:381):
// make_canonical_split over the traceback blocks.
#include <algorithm>
#include <chrono>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dagsplit/dp_solver.hpp"
#include "dagsplit/errors.hpp"
#include "dagsplit/graph.hpp"
#include "dagsplit/rng.hpp"
#include "dsg_b200.h"

namespace dagsplit {

namespace {

dsg_rat to_pod(const Rat& r) {
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

struct PodGraph {
  std::vector<int32_t> ids, pair, ef, et, af, at;
  std::vector<dsg_rat> cpu, acc, comm, mem;
  std::vector<uint8_t> bw;
  dsg_graph g{};

  explicit PodGraph(const Graph& graph) {
    for (const Node& n : graph.nodes()) {
      ids.push_back(n.id);
      cpu.push_back(to_pod(n.cpu_time));
      acc.push_back(to_pod(n.acc_time));
      comm.push_back(to_pod(n.comm_time));
      mem.push_back(to_pod(n.mem_size));
      bw.push_back(n.is_backward ? 1 : 0);
      pair.push_back(n.forward_pair ? *n.forward_pair : DSG_NO_PAIR);
    }
    for (const Edge& e : graph.edges()) {
      ef.push_back(e.from);
      et.push_back(e.to);
    }
    for (const Edge& e : graph.artificial_edges()) {
      af.push_back(e.from);
      at.push_back(e.to);
    }
    g.n_nodes = graph.size();
    g.ids = ids.data();
    g.cpu_time = cpu.data();
    g.acc_time = acc.data();
    g.comm_time = comm.data();
    g.mem_size = mem.data();
    g.is_backward = bw.data();
    g.forward_pair = pair.data();
    g.n_edges = (int32_t)ef.size();
    g.edge_from = ef.data();
    g.edge_to = et.data();
    g.n_artificial = (int32_t)af.size();
    g.art_from = af.data();
    g.art_to = at.data();
  }
};

dsg_options options_from(const SolveOptions& opt) {
  dsg_options o;
  dsg_default_options(&o);
  o.ideal_budget = opt.ideal_budget;
  if (opt.deadline) {
    const double left =
        std::chrono::duration<double>(*opt.deadline - std::chrono::steady_clock::now()).count();
    o.deadline_seconds = std::max(left, 1e-9);
  }
  return o;
}

// dsg_status -> the reference's exception vocabulary (errors.hpp,
// graph.hpp:239-241, rational.cpp:16-21)
[[noreturn]] void throw_status(int status, const char* msg, long long budget_limit) {
  switch (status) {
    case DSG_INFEASIBLE:
      throw InfeasibleError();
    case DSG_DEADLINE:
      throw DeadlineExceeded();
    case DSG_BUDGET:
      throw IdealBudgetExceeded{budget_limit};
    case DSG_MISSING_BANDWIDTH:
      throw MissingBandwidth();
    case DSG_INVALID:
      if (std::string(msg) == "subtracting infinity" || std::string(msg) == "invalid rational")
        throw std::domain_error(msg);
      throw std::invalid_argument(msg);
    case DSG_OVERFLOW:
      throw std::overflow_error(msg);
    case DSG_LOGIC:
      throw std::logic_error(msg);
    default:
      throw std::runtime_error(std::string("dsg_b200: ") + msg);
  }
}

Split device_solve(int mode, const Graph& g, const DeviceConfig& config, const SolveOptions& opt) {
  PodGraph pg(g);
  dsg_config c{};
  c.accelerators = config.accelerators;
  c.cpus = config.cpus;
  c.memory_limit = to_pod(config.memory_limit);
  c.q = config.q;
  c.interleaving = static_cast<int32_t>(config.interleaving);
  c.has_bandwidth = config.bandwidth ? 1 : 0;
  c.bandwidth = config.bandwidth ? to_pod(*config.bandwidth) : dsg_rat{0, 1};
  c.replication_combine = static_cast<int32_t>(config.replication_combine);
  dsg_options o = options_from(opt);
  dsg_result r;
  dsg_dp_solve(mode, &pg.g, &c, &o, &r);
  if (r.status != DSG_OK) {
    std::string msg = r.message;
    const long long limit = r.budget_limit;
    const int st = r.status;
    dsg_result_free(&r);
    throw_status(st, msg.c_str(), limit);
  }
  std::vector<SplitBlock> blocks;
  for (int b = 0; b < r.n_blocks; ++b) {
    SplitBlock blk;
    blk.cpu = r.blocks[b].cpu != 0;
    blk.repl = r.blocks[b].repl;
    blk.members.assign(r.members + r.blocks[b].offset,
                       r.members + r.blocks[b].offset + r.blocks[b].n_members);
    blocks.push_back(std::move(blk));
  }
  const Rat objective = r.objective.den == 0 ? Rat::infinity()
                                             : Rat(static_cast<long long>(r.objective.num),
                                                   static_cast<long long>(r.objective.den));
  dsg_result_free(&r);
  return make_canonical_split(g, config, std::move(blocks), objective);
}

IdealIndex device_enumerate(const Graph& g, const NodeSet* within, long long budget) {
  PodGraph pg(g);
  std::vector<uint8_t> w;
  if (within) {
    w.assign(g.size() + 1, 0);
    for (int v = 0; v < g.size(); ++v) w[v] = within->contains(v) ? 1 : 0;
  }
  dsg_options o;
  dsg_default_options(&o);
  dsg_ideals out;
  dsg_enumerate_ideals(&pg.g, within ? w.data() : nullptr, budget, &o, &out);
  if (out.status != DSG_OK) {
    std::string msg = out.message;
    const long long limit = out.budget_limit;
    const int st = out.status;
    dsg_ideals_free(&out);
    throw_status(st, msg.c_str(), limit);
  }
  IdealIndex index;
  index.ideals.reserve(out.count);
  for (long long i = 0; i < out.count; ++i) {
    NodeSet s(g.size());
    for (int wd = 0; wd < out.words; ++wd) {
      uint64_t x = out.bits[i * out.words + wd];
      while (x) {
        s.insert(wd * 64 + __builtin_ctzll(x));
        x &= x - 1;
      }
    }
    index.by_hash[s.hash()].push_back(static_cast<int>(i));
    index.ideals.push_back(std::move(s));
  }
  dsg_ideals_free(&out);
  return index;
}

// Same contract as chain_along (dp_solver.cpp:444-455): artificial
// precedence edges along `order`, skipping pairs already connected.
Graph chain(const Graph& g, const std::vector<int>& order) {
  std::set<std::pair<int, int>> have;
  for (const Edge& e : g.edges()) have.insert({e.from, e.to});
  for (const Edge& e : g.artificial_edges()) have.insert({e.from, e.to});
  std::vector<Edge> art = g.artificial_edges();
  for (size_t i = 1; i < order.size(); ++i) {
    const int u = g.id_of(order[i - 1]), v = g.id_of(order[i]);
    if (have.insert({u, v}).second) art.push_back(Edge{u, v, {}});
  }
  return Graph(g.nodes(), g.edges(), std::move(art));
}

}  // namespace

Split solve_maxload_inference(const Graph& g, const DeviceConfig& config, const SolveOptions& opt) {
  return device_solve(DSG_MODE_INFERENCE, g, config, opt);
}

Split solve_maxload_training(const Graph& g, const DeviceConfig& config, const SolveOptions& opt) {
  return device_solve(DSG_MODE_TRAINING, g, config, opt);
}

Split solve_maxload_replicated(const Graph& g, const DeviceConfig& config, const SolveOptions& opt) {
  return device_solve(DSG_MODE_REPLICATED, g, config, opt);
}

// Host-side ordering helper (not on the hot path): a DFS topological order
// with seeded tie-breaking (dp_solver.hpp:39-41).  Same seeding and shuffle
// sequence as the reference so DPL results coincide: roots shuffled, then
// every adjacency list shuffled in node order, iterative DFS, reversed
// post-order.
std::vector<int> seeded_topo_order(const Graph& g, uint64_t seed) {
  SplitMix64 rng(seed * 0x9e3779b97f4a7c15ULL + 0x2545f4914f6cdd1dULL);
  const int n = g.size();
  std::vector<int> roots(n);
  for (int i = 0; i < n; ++i) roots[i] = i;
  rng.shuffle(roots);
  std::vector<std::vector<int>> succ(n);
  for (int v = 0; v < n; ++v) {
    succ[v] = g.out_all(v);
    rng.shuffle(succ[v]);
  }
  std::vector<char> seen(n, 0);
  std::vector<int> post;
  post.reserve(n);
  std::vector<std::pair<int, size_t>> st;
  for (int r : roots) {
    if (seen[r]) continue;
    seen[r] = 1;
    st.assign(1, {r, 0});
    while (!st.empty()) {
      auto& top = st.back();
      if (top.second < succ[top.first].size()) {
        const int w = succ[top.first][top.second++];
        if (!seen[w]) {
          seen[w] = 1;
          st.push_back({w, 0});
        }
      } else {
        post.push_back(top.first);
        st.pop_back();
      }
    }
  }
  std::reverse(post.begin(), post.end());
  return post;
}

Graph linearize(const Graph& g, uint64_t seed) { return chain(g, seeded_topo_order(g, seed)); }

// DPL heuristic (dp_solver.hpp:47-52): chain the forward part (training) or
// the whole graph, then the exact DP on the collapsed |V|+1 lattice.
Split solve_dpl(const Graph& g, const DeviceConfig& config, uint64_t seed, const SolveOptions& opt) {
  const bool training = g.has_backward_nodes();
  std::vector<int> order = seeded_topo_order(g, seed);
  if (training)
    order.erase(std::remove_if(order.begin(), order.end(),
                               [&](int v) { return g.node(v).is_backward; }),
                order.end());
  const Graph chained = chain(g, order);
  return training ? solve_maxload_training(chained, config, opt)
                  : solve_maxload_inference(chained, config, opt);
}

IdealIndex enumerate_ideals(const Graph& g, long long budget) {
  return device_enumerate(g, nullptr, budget);
}

IdealIndex enumerate_ideals_within(const Graph& g, const NodeSet& within, long long budget) {
  return device_enumerate(g, &within, budget);
}

}  // namespace dagsplit
