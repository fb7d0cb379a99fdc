"""dagsplit on B200: the max-load DP over ideals of a DNN operator DAG
(Tarnawski et al. 2020, arXiv 2006.16423) as hand-written sm_100a kernels
behind the reference's solver API.

Reference API → this package:
  solve_maxload_inference / _training   (dp_solver.hpp:21-29)  → solver.*
  solve_maxload_replicated, seeded_topo_order, linearize, solve_dpl
                                        (dp_solver.hpp:36-52)  → solver.*
  enumerate_ideals / _within            (graph.hpp:253-258)     → solver.*
  Graph, Node, Edge, DeviceConfig, Split (graph.hpp)             → graph.*
  InfeasibleError, DeadlineExceeded, …  (errors.hpp)            → errors.*
"""
from .errors import (DeadlineExceeded, DeviceError, IdealBudgetExceeded, InfeasibleError,
                     MissingBandwidth, Unsupported)
from .graph import (INF, AccParts, DeviceConfig, Edge, Graph, Interleaving, Node, Placement,
                    ReplicationCombine, Split, SplitBlock, acc_cost, acc_cost_parts,
                    combine_interleaving, cpu_cost, is_contiguous, is_ideal, make_canonical_split,
                    make_node, recompute_maxload, verify_split)
from .solver import (IdealIndex, SolveOptions, enumerate_ideals, enumerate_ideals_within,
                     kernel_launch_count, linearize, load_library, seeded_topo_order,
                     solve_dpl, solve_maxload_inference,
                     solve_maxload_replicated, solve_maxload_training)

__all__ = [
    "DeadlineExceeded", "DeviceError", "IdealBudgetExceeded", "InfeasibleError",
    "MissingBandwidth", "Unsupported", "INF", "AccParts", "DeviceConfig", "Edge", "Graph",
    "Interleaving", "Node", "Placement", "ReplicationCombine", "Split", "SplitBlock", "acc_cost",
    "acc_cost_parts", "combine_interleaving", "cpu_cost", "is_contiguous", "is_ideal",
    "make_canonical_split", "make_node", "recompute_maxload", "verify_split", "IdealIndex",
    "SolveOptions", "enumerate_ideals", "enumerate_ideals_within", "kernel_launch_count",
    "linearize", "load_library", "seeded_topo_order", "solve_dpl", "solve_maxload_inference", "solve_maxload_replicated",
    "solve_maxload_training",
]
