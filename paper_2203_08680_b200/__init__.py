"""B200-native parallel Gene-pool Optimal Mixing (GOM) on Max-Cut.

Hot path: hand-written sm_100a CUDA in libgomix_b200.so behind the C-ABI of
include/gomix_gpu.h.  There is no CPU fallback: without the library (or a
GPU) the engine raises.
"""
from .maxcut import (Fos, MaxCutInstance, ParseError, bounded_flt_fos, generate_regular, generate_torus, load_edge_list,  # noqa: F401
                     neighbourhood_fos, save_edge_list, univariate_fos)
from .engine import (FitnessComparator, GpuLocalGroup, GpuParallelEngine, GpuProblem,  # noqa: F401
                     RecordingSink, RunContext, RunControl, TerminationConfig, TraceRecord, TraceSink, gpu_color, mix64,
                     nccl_unique_id, population_seed, shard_range)
from .ims import DeviceBest, GpuImsDriver, ImsConfig, RunResult, run_gpu  # noqa: F401
from .trace_io import TRACE_HEADER, CsvTraceWriter, format_double, parse_trace, trace_monotone  # noqa: F401

__all__ = ["Fos", "MaxCutInstance", "ParseError", "bounded_flt_fos", "generate_regular", "generate_torus", "load_edge_list", "neighbourhood_fos",
           "save_edge_list", "univariate_fos", "FitnessComparator", "GpuLocalGroup", "GpuParallelEngine", "GpuProblem",
           "RecordingSink", "RunContext", "RunControl", "TerminationConfig", "TraceRecord", "TraceSink", "gpu_color", "mix64",
           "nccl_unique_id", "population_seed", "shard_range", "DeviceBest", "GpuImsDriver", "ImsConfig",
           "RunResult", "run_gpu", "TRACE_HEADER", "CsvTraceWriter", "format_double", "parse_trace",
           "trace_monotone"]
