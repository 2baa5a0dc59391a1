"""B200-native LCN-Sinkhorn hot path (arXiv 2107.06876).

The product is the C-ABI library paper_2107_06876_b200/_build/liblcn_b200.so
(include/lcn_b200.h): hand-written sm_100a CUDA for k-means LSH bucketing,
Nystrom landmarks, the bucket-blocked K_sp / LCN correction and the
log-stabilised Sinkhorn loop. `native` mirrors the reference's lcn:: API over
it; `configs` holds the seeded BASELINE.json inputs.
"""
from . import configs  # noqa: F401
from .native import (  # noqa: F401
    COSINE_DERIVED, EUCLIDEAN, LANDMARK_KMEANS, LANDMARK_KMEANSPP, LSH_CROSS_POLYTOPE, LSH_HIERARCHICAL_KMEANS,
    LSH_KMEANS, NEGATIVE_DOT, SQEUCLIDEAN, Context, CudaError,
    DimensionError, Error, FactorizationError, InvalidArgument, KernelOperator, LoopbackGroup, LshConfig,
    NegativeKernelError, ShardPlan, build_correction, build_factors, build_sparse, lsh_neighbor_pairs,
    select_landmarks,
    SinkhornOptions, SinkhornResult, StabilizationError, assign_nearest, batched_lcn, cross_polytope_buckets, distance_lcn, grad_cost, kmeans_pp_indices, library,
    lloyd, lsh_buckets, lsh_kmeans_buckets, multihead, nccl_unique_id, read_points_file, sample_clustered,
    sample_uniform_ball, sinkhorn, sinkhorn_device, write_points_file)
