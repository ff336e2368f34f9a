"""Drop-in for the reference `gpushare` hot path (probe -> placement).

``from paper_2107_08538_b200.gpushare import Scheduler, DeviceState, ...``
replaces ``from gpushare import ...`` for the placement path
(gpushare/__init__.py:9-56): same names, argument meanings, errors and
decision-log schema; decisions are computed by sm_100a kernels in libgs.
"""

from .device_model import (
    GIB,
    KIB,
    MIB,
    PRESETS,
    DeviceSpec,
    DeviceState,
    PlacementPlan,
    device_spec,
    occupancy_limit_per_sm,
)
from .errors import (
    AnalysisError,
    ConfigError,
    ContractViolation,
    GpuShareError,
    LazyBindingError,
)
from .lazy_runtime import (
    GpuOp,
    LazyState,
    OpKind,
    PseudoAddress,
    kernel_launch_prepare,
    lazy_alloc,
    queued_bytes,
    record_op,
    release_bound,
    replay,
    set_heap_limit,
)
from .schedulers import (
    ASSIGN,
    DEFER,
    REJECT,
    Decision,
    PolicyConfig,
    ScheduleRequest,
    Scheduler,
    parse_policy,
)
from .task_builder import (
    BYTE_LIMIT,
    DEFAULT_HEAP_LIMIT,
    WARP_SIZE,
    LaunchShape,
    ResourceRequest,
    compute_resource_request,
)

__all__ = [
    "ASSIGN", "DEFER", "REJECT", "GIB", "KIB", "MIB", "PRESETS", "BYTE_LIMIT",
    "DEFAULT_HEAP_LIMIT", "WARP_SIZE", "AnalysisError", "ConfigError",
    "ContractViolation", "Decision", "DeviceSpec", "DeviceState", "GpuShareError",
    "LaunchShape", "LazyBindingError", "PlacementPlan", "PolicyConfig",
    "ResourceRequest", "ScheduleRequest", "Scheduler", "compute_resource_request",
    "device_spec", "occupancy_limit_per_sm", "parse_policy",
    "GpuOp", "LazyState", "OpKind", "PseudoAddress", "kernel_launch_prepare", "lazy_alloc",
    "queued_bytes", "record_op", "release_bound", "replay", "set_heap_limit",
]
