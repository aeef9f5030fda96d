"""B200-native Hash-based Partition (HBP) SpMV (arXiv 2504.08860).

Drop-in for the reference package's hot path (hbp_spmv, __init__.py:13-32):

    csr = coo_to_csr(trip)
    config = PartitionConfig()
    grid = make_grid(csr, config)
    params = sample_hash_params(grid, config)
    hbp = build_hbp(csr, grid, hash_permutations(grid, params))
    y = hbp_spmv(hbp, x)

Every step runs as hand-written sm_100a CUDA kernels in libhbp.so (C ABI:
include/hbp.h); arrays are device-resident torch tensors.  There is no CPU
fallback.
"""
from .formats import (CsrMatrix, TripletMatrix, coo_to_csr, csr_spmv, csr_to_triplets,
                      dense_oracle_spmv, to_dense)
from .mtx import (MatrixMarketError, MatrixMarketHeader, expand_symmetric, load_mtx,
                  parse_matrix_market, save_mtx, write_matrix_market)
from .synth import SyntheticSpec, generate
from .partition import BlockGrid, PartitionConfig, block_rows_of, make_grid
from .reorder import (BUCKET_MAX, BlockPermutations, HashParams, OpCounter,
                      build_block_permutation, hash_permutations, hash_slot,
                      identity_permutations, perm_for_block, sample_hash_params,
                      sort_permutation, sort_permutations)
from .hbp import (HbpFormatError, HbpMatrix, build_hbp, deserialize_hbp, hbp_to_triplets,
                  load_hbp, save_hbp, serialize_hbp)
from .engine import (ExecutionLog, ExecutionPlan, HostPipeline, PartialVector, SpmvOperator,
                     block2d_spmv_baseline, block_spmv, combine, hbp_spmv, plan_execution,
                     run_spmv, scale, sumsq)
from .metrics import (BenchReport, GroupStats, GroupStatsTable, Timing, gflops, group_stats,
                      group_stats_csv, mean_group_std, reduction_summary, time_kernel)

__version__ = "0.1.0"

__all__ = [
    "BUCKET_MAX", "BlockGrid", "BlockPermutations", "CsrMatrix", "ExecutionLog",
    "ExecutionPlan", "HashParams", "HostPipeline", "HbpFormatError", "HbpMatrix", "OpCounter", "PartialVector",
    "PartitionConfig", "SpmvOperator", "TripletMatrix", "block2d_spmv_baseline", "block_rows_of",
    "block_spmv", "csr_spmv", "scale", "sumsq",
    "build_block_permutation", "build_hbp", "combine", "coo_to_csr", "csr_to_triplets",
    "deserialize_hbp", "hash_permutations", "hash_slot", "hbp_spmv", "hbp_to_triplets",
    "identity_permutations", "load_hbp", "make_grid", "perm_for_block", "plan_execution",
    "run_spmv", "sample_hash_params", "save_hbp", "serialize_hbp", "sort_permutation",
    "sort_permutations",
    "MatrixMarketError", "MatrixMarketHeader", "expand_symmetric", "load_mtx",
    "parse_matrix_market", "save_mtx", "write_matrix_market", "dense_oracle_spmv", "to_dense",
    "SyntheticSpec", "generate",
    "BenchReport", "GroupStats", "GroupStatsTable", "Timing", "gflops", "group_stats",
    "group_stats_csv", "mean_group_std", "reduction_summary", "time_kernel",
]
