"""B200-native build/solve engine for the Gillman–Martinsson nested-dissection
DtN build (arXiv 1302.5995): leaf elimination, batched FP64 merges and the
batched solve on sm_100a, behind the C ABI in include/dtn_gpu.h."""
from .dtn import (AccelOptions, BoxTree, Context, DiscreteOperator, Engine, FactorizationError, Lattice,  # noqa: F401
                  ProblemMode, ProblemSpec, SolutionOperator, apply_dtn, apply_schur, baseline_problem,
                  build_root_accel, build_root_dense_op, build_root_gpu, CompressedSolutionOperator, build_tree, build_tree_uniform, build_with_loads, catalog, shard_info,
                  catalog_names, default_context, densify_dtn, discrete_eigenvalue, discrete_eigenvalue_kth,
                  discretize, dump_schur, load_schur, make_load_set, ring_dtn, ring_nodes, root_boundary,
                  solve_with_load, nccl_unique_id, collective_context)
