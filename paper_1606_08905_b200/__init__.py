"""B200-native Lloyd / MTI k-means: a drop-in for numakmeans' ``kmeans()`` path.

The reference (knor, arXiv 1606.08905, packaged as ``numakmeans``) runs
Lloyd's algorithm with minimal-triangle-inequality pruning on NUMA CPU
threads.  This package keeps its API -- ``kmeans(matrix, EngineConfig)`` ->
``KmeansResult`` with ``CentroidSet`` and per-iteration ``IterationStats`` --
and runs every pass over the points in hand-written sm_100a CUDA kernels
(``csrc/``, exported through the C ABI in ``include/knor_b200.h``), sharded
over GPUs with one NCCL all-reduce per iteration (``kmeans_sharded``).
"""

from . import synth
from .centroids import INIT_METHODS, CentroidSet
from .engine import (
    EngineConfig,
    IoDelta,
    IterationStats,
    KmeansResult,
    Lloyd,
    SchedCounters,
    kmeans,
    kmeans_sharded,
)
from .fileio import HEADER_SIZE, MatrixIOError, load_matrix, save_matrix
from .matrix import MatrixFormatError, RowRange, check_matrix, partition_rows
from .outofcore import CacheSchedule, RowStore, kmeans_ondisk
from ._native import release_memory
from .parallel import LocalComm, TorchComm, shard_of
from .primitives import (
    CentroidGeometry,
    block_distances,
    centroid_geometry,
    euclidean_distance,
    init_centroids,
    nearest_centroid,
    row_sqnorms,
    rowwise_distances,
)
from .report import deterministic_view, format_report, parse_report

__version__ = "0.1.0"

__all__ = [
    "CacheSchedule",
    "CentroidGeometry",
    "block_distances",
    "centroid_geometry",
    "euclidean_distance",
    "init_centroids",
    "nearest_centroid",
    "row_sqnorms",
    "rowwise_distances",
    "CentroidSet",
    "RowStore",
    "kmeans_ondisk",
    "HEADER_SIZE",
    "MatrixIOError",
    "deterministic_view",
    "format_report",
    "load_matrix",
    "parse_report",
    "save_matrix",
    "EngineConfig",
    "INIT_METHODS",
    "IoDelta",
    "IterationStats",
    "KmeansResult",
    "LocalComm",
    "Lloyd",
    "MatrixFormatError",
    "RowRange",
    "SchedCounters",
    "TorchComm",
    "check_matrix",
    "kmeans",
    "kmeans_sharded",
    "release_memory",
    "partition_rows",
    "shard_of",
]
