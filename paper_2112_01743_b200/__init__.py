"""paper_2112_01743_b200 — B200-native CPAA (Chebyshev-polynomial PageRank, arXiv 2112.01743).

A drop-in for the reference chebpr library's hot path: graph build (K1 device CSR
builder), ``run_cpaa`` (degree-binned fused term kernels for sm_100a), the Power
comparator and the staged API, all behind the C-ABI in include/chebpr_cuda.h.
"""
from .api import (  # noqa: F401
    ApproxPlan, BuildOptions, BuildResult, CapacityError, CoefficientTable, CudaError,
    DeviceGraph, DomainError, Error, GraphStats, IterationState, MODE_BITEXACT, MODE_FAST,
    NumericError, PageRankResult, ParseError, PowerConfig, SolverConfig, TraceRow,
    UndirectedGraph, ValidationError, VertexRange, accumulate_stage, beta, build_device_graph,
    build_graph, coefficients, run_cpaa_batch, BatchResult, device_count, err_bound, generate_stage, init_state, kahan_sum,
    normalize, partition_vertices, plan_iterations, reference_pagerank, run_cpaa, run_power,
    sigma, transition_apply, upload, validate, LoadOptions, LoadedGraph, load_edge_list,
    load_matrix_market, load_device_graph, parse_text, PartitionGroup,
)

__version__ = "0.1.0"
