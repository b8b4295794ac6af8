"""B200-native bucketed approximate top-k (arxiv 2412.04358), drop-in for the
reference package `bucketed_topk`'s selection API.

Public names mirror the reference's `bucketed_topk/__init__.py`:
core types and validation, exact selection, and the two-stage bucketed
selection.  Every selection call runs hand-written sm_100a kernels from
`libbtk.so` through its C ABI (include/btk.h); there is no CPU fallback.
"""

from .core import (Assignment, BucketScheme, ConfigError, NonFiniteInputError, ProblemShape,
                   bucket_of, bucket_sizes, check_parameters, describe_scheme, max_bucket_size,
                   stage1_candidate_count, validate)
from .exact import (ScoredIndex, TopKResult, exact_topk_oracle, priority_queue_topk,
                    topk_with_indices)
from .approx import (ApproxTopK, ChunkedMerge, ExecutionMode, PerBucket, Stage1Candidates,
                     approx_topk, select_mode, stage1)
from .shard import approx_topk_sharded, distributed_approx_topk, row_blocks
from .recall import MonteCarloRecall, empirical_recall, empirical_recall_rows, monte_carlo_recall
from . import simdata

__version__ = "0.1.0"

__all__ = [
    "Assignment", "BucketScheme", "ConfigError", "NonFiniteInputError", "ProblemShape",
    "bucket_of", "bucket_sizes", "check_parameters", "describe_scheme", "max_bucket_size",
    "stage1_candidate_count", "validate",
    "ScoredIndex", "TopKResult", "exact_topk_oracle", "priority_queue_topk", "topk_with_indices",
    "ApproxTopK", "ChunkedMerge", "ExecutionMode", "PerBucket", "Stage1Candidates", "approx_topk",
    "select_mode", "stage1",
    "approx_topk_sharded", "distributed_approx_topk", "row_blocks",
    "MonteCarloRecall", "empirical_recall", "empirical_recall_rows", "monte_carlo_recall", "simdata",
]
