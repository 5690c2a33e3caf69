"""B200-native hot path of the arXiv:1210.5128 order-space MCMC BN learner.

The product is ``libbnmc_b200.so`` (C-ABI: include/bnmc_gpu.h) — hand-written
sm_100a kernels for the local-score precompute, the order scan and the
device-resident MCMC loop. This package is the reference-shaped host mirror
(``api``) over that library plus multi-GPU plumbing (``dist``).
"""
from .api import (AlphaMode, CapacityError, CountTable, DataError, Dataset, EngineConfig, Error,
                  McmcResult, count_statistics,
                  Order, OrderScorer, PriorMatrix, RunConfig, ScoreCache, ScoredGraph, UsageError,
                  baseline_instance, parallel_score_order, read_bnsc, run_chains, run_chains_batch, run_mcmc,
                  synth_instance, synth_priors, write_bnsc)

__all__ = ["AlphaMode", "CapacityError", "CountTable", "count_statistics", "DataError", "Dataset", "EngineConfig", "Error",
           "McmcResult", "Order", "OrderScorer", "PriorMatrix", "RunConfig", "ScoreCache",
           "ScoredGraph", "UsageError", "baseline_instance", "parallel_score_order", "read_bnsc",
           "run_chains", "run_chains_batch", "run_mcmc", "synth_instance", "synth_priors", "write_bnsc"]
