"""B200-native hot path of the adaptive H-matrix BEM for the Lame equations
(Bauer & Bebendorf, arXiv 2205.04752): batched ACA of Kelvin collocation
blocks, near-field fill and the H-matvec on sm_100a, behind the C ABI of
include/hmgpu.h, with a host layer mirroring the reference's operator API.
"""
from .api import (AcaStop, admissible, gauss_rule, random_vector, fp64_peak_tflops, dmma_peak_tflops, dmma_peak_sustained_tflops, AmvmConfig, AmvmIteration, AmvmReport, AssemblyConfig,
                  AssemblyStats, BlockTerm, ClusterTree, ConfigError, DeviceError,
                  DimensionError, Error, GammaContributions, HMatrix, LameSingleLayer, Mesh,
                  OperatorSet, lame_constants, InteriorEvaluator, pair_rule, sparse_op, BacaConfig, BacaReport, VddPreconditioner,
                  baca_solve, pcg_spd, estimator_vh, doerfler_mark, DofLayout, SaddleSystem,
                  SolveStats, bpcg_solve, SaddleEstimator, baca_solve_saddle,
                  MeshError, Mode, amvm_multiply, assemble, device_count, gamma_contributions,
                  host_tree_and_partition, nccl_available, nccl_unique_id,
                  mark_blocks_sharded, amvm_multiply_occurrences, rhs_occurrences,
                  assemble_rhs)

__all__ = [
    "AcaStop", "admissible", "gauss_rule", "random_vector", "fp64_peak_tflops", "dmma_peak_tflops", "dmma_peak_sustained_tflops", "AmvmConfig", "AmvmIteration", "AmvmReport", "AssemblyConfig",
    "AssemblyStats", "BlockTerm", "ClusterTree", "ConfigError", "DeviceError",
    "DimensionError", "Error", "GammaContributions", "HMatrix", "LameSingleLayer", "Mesh",
    "OperatorSet", "lame_constants", "InteriorEvaluator", "pair_rule", "sparse_op", "BacaConfig", "BacaReport", "VddPreconditioner",
    "baca_solve", "pcg_spd", "estimator_vh", "doerfler_mark", "DofLayout", "SaddleSystem",
    "SolveStats", "bpcg_solve", "SaddleEstimator", "baca_solve_saddle",
    "MeshError",
    "Mode", "amvm_multiply", "assemble", "device_count", "gamma_contributions",
    "host_tree_and_partition", "nccl_available", "nccl_unique_id", "mark_blocks_sharded",
    "amvm_multiply_occurrences", "rhs_occurrences", "assemble_rhs",
]
