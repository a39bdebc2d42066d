"""paper_2305_01886_b200 -- B200-native batched energy prediction for CUDA
kernels (arXiv 2305.01886): analytical cycles x tree-ensemble power, with the
reference package's predictor API (gpukalc) as the drop-in surface.

Importing the package loads neither torch nor the CUDA library; the first
device call does (and raises DeviceError if either is unavailable -- there is
no CPU fallback).
"""

from .api import (
    EnergyReport,
    FeatureVector,
    KernelSchedule,
    LaunchConfig,
    extract_features,
    extract_features_batch,
    predict_energy,
    predict_launches,
    predict_power,
    predict_power_batch,
    schedule_batch,
    schedule_kernel,
)
from .ensemble import TreeEnsemble, load_ensemble
from .errors import (
    DeviceError,
    EnsembleError,
    FitError,
    GpukalcError,
    ProfileError,
    PtxParseError,
    ScheduleError,
)
from .ir import BasicBlock, InstClass, KernelGraph, PtxInstruction, Resource
from .pack import FEATURE_ORDER, SELECTED_FEATURES
from .profiles import (
    ArchProfile,
    cycles_from_us,
    global_mem_latency,
    latency_of,
    launch_overhead_us,
    list_shipped_profiles,
    load_profile,
    mem_throughput,
    resolve_profile,
    us_from_cycles,
)
from .featio import features_csv, features_from_csv, features_from_csv_arrays, features_to_csv
from .ptx import parse_ptx
from .ptx_native import pack_ptx

__version__ = "0.1.0"

__all__ = [
    "ArchProfile", "BasicBlock", "DeviceError", "EnergyReport", "EnsembleError", "FEATURE_ORDER",
    "FeatureVector", "FitError", "GpukalcError", "InstClass", "KernelGraph", "KernelSchedule",
    "LaunchConfig", "ProfileError", "PtxInstruction", "PtxParseError", "Resource",
    "SELECTED_FEATURES", "ScheduleError", "TreeEnsemble", "cycles_from_us", "extract_features",
    "extract_features_batch", "features_csv", "features_from_csv", "features_from_csv_arrays",
    "features_to_csv", "global_mem_latency", "latency_of", "launch_overhead_us",
    "list_shipped_profiles", "load_ensemble", "load_profile", "mem_throughput", "pack_ptx",
    "parse_ptx",
    "predict_energy", "predict_launches", "predict_power", "predict_power_batch",
    "resolve_profile", "schedule_batch", "schedule_kernel", "us_from_cycles",
]
