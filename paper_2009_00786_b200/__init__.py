"""B200-native tsidx hot path: iSAX index build + exact Euclidean 1-NN.

The compute path is libtsgpu.so (hand-written sm_100a CUDA behind the C ABI
in include/tsgpu.h); this package is the host-side mirror of the
reference's tsidx API over that ABI.
"""
from .tsidx import (  # noqa: F401
    BuildStats, Context, Index, IndexConfig, InvalidArgument, LogicError, Measure, MeasureKind, QueueMode,
    SearchOptions, SearchResult, SearchStats, TsgError, approximate_search, breakpoints, build_index, comm_unique_id, exact_search,
    build_index_from_file, exact_search_batch, exact_search_batch_records, RESULT_DTYPE, generate_device, generate_random_walk_device, launch_count,
    load_dataset, save_dataset, summarise, ValidationReport, validate_index,
)
