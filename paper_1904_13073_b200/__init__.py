"""B200-native SurfelWarp per-frame non-rigid tracking + fusion (arXiv 1904.13073).

Hot path: hand-written sm_100a CUDA kernels in csrc/ behind the C ABI
include/dynsurf_b200.h; this package is the host mirror of the reference's
`dynsurf::Pipeline` API (pipeline.hpp:38-62) plus the stage entry points.
"""
from .errors import (CapacityExceeded, ConfigError, CorruptFrame, CudaError,  # noqa: F401
                     DimensionMismatch, EmptyGeometry, Error, InvalidArgument, IoFailure,
                     MissingInput, UnknownScenario)
from .pipeline import (Context, Pipeline, SyntheticSequence, camera_config,  # noqa: F401
                       make_config, stats_to_dict)
from .sequence_io import (PipelineOptions, SequenceSummary, export_pointcloud,  # noqa: F401
                          frame_stats_to_json, process_sequence, read_depth_png,
                          read_pointcloud, timings_to_json, write_depth_png)

__all__ = [
    "Pipeline", "Context", "SyntheticSequence", "make_config", "camera_config",
    "stats_to_dict", "Error", "DimensionMismatch", "EmptyGeometry", "ConfigError",
    "CapacityExceeded", "CudaError", "InvalidArgument", "UnknownScenario", "MissingInput",
    "CorruptFrame", "IoFailure", "PipelineOptions", "SequenceSummary", "process_sequence",
    "read_depth_png", "write_depth_png", "export_pointcloud", "read_pointcloud",
    "frame_stats_to_json", "timings_to_json",
]
