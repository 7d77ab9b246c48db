"""B200-native DTW distance-matrix fill + k-medoids sweeps (arXiv 2307.04904 hot path).

The product is libdtwgpu.so (sm_100a CUDA kernels + native C++ host behind the C-ABI in
include/dtwgpu.h). This package mirrors the reference's dtwclust interface for that
path on top of it (api.py), shards it over GPUs (distributed.py) and generates the
seeded synthetic workloads (generators.py).
"""
from .api import (  # noqa: F401
    FP32, FP64, BandInfeasibleError, BuildStats, ClusterResult, DeviceError, DistanceMatrix,
    DistanceMatrixInvalidError, EmptyDatasetError, Engine, Error, IndexOutOfRangeError,
    InvalidArgumentsError, InvalidSeriesError, KMedoidsConfig, KOutOfRangeError, ScoreReport,
    SingleClusterUndefinedError, TimeSeries, WarpWindow, assign_to_medoids, assignment_cost,
    build_matrix, build_matrix_packed, dtw_distance, engine, kmedoids, silhouette_scores, update_medoids,
    validate, validate_dataset,
)
