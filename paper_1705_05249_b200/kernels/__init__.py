"""Kernel layer: parameter family and constraint filter, launch bookkeeping,
and the ctypes binding of the sm_100a CUDA library (libtbgemm.so)."""

from .engine import WorkGrid, assert_launch_resources, launch_grid
from .params import (
    Configuration,
    FAMILIES,
    GemmParams,
    PARAM_NAMES,
    curated_configurations,
    default_config,
    enumerate_search_space,
    full_grid,
    full_grid_size,
    local_mem_usage,
    random_configuration,
    require_valid,
    validate_config,
    validate_gemm_params,
    work_group_threads,
)

__all__ = [
    "Configuration", "FAMILIES", "GemmParams", "PARAM_NAMES", "WorkGrid",
    "assert_launch_resources", "curated_configurations", "default_config",
    "enumerate_search_space", "full_grid", "full_grid_size", "launch_grid",
    "local_mem_usage", "random_configuration", "require_valid",
    "validate_config", "validate_gemm_params", "work_group_threads",
]
