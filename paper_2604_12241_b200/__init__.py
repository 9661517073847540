"""B200-native mining stage of the tempmine engine (arXiv 2604.12241).

Drop-in for the reference's mining path: `mine(graph, plans)`
with the reference's signature and FeatureMatrix result, backed by
hand-written sm_100a kernels in libtempmine_b200.so behind a C ABI
(include/tempmine_b200.h).  Plans may be the reference's own compiled
ExecutionPlans or the structurally identical ones `builtin_plan` builds.
"""

from ._lib import TempmineError, UnsupportedPlanError, kernel_launch_count
from .engine import (EngineInvariantError, FeatureMatrix, InstanceRecord, collect_instance_records,
                     last_stats, lower_all, merge_features, mine,
                     mine_members, mine_members_device, mine_rows, mine_rows_device, order_plans,
                     prepare_views, release_views, write_instances)
from .graph import DeviceGraph, GraphStats, as_device_graph
from .plan import (BUILTIN_COLUMNS, EXTENDED_COLUMNS, FULL_PATTERN_SET, ExecutionPlan, PlanDesc,
                   builtin_plan, canonical_shape, full_pattern_set, load_builtin, lower_plan, recognize)

__all__ = [
    "BUILTIN_COLUMNS", "EXTENDED_COLUMNS", "FULL_PATTERN_SET", "DeviceGraph", "EngineInvariantError",
    "ExecutionPlan", "FeatureMatrix", "InstanceRecord", "collect_instance_records", "GraphStats", "PlanDesc", "TempmineError",
    "UnsupportedPlanError", "as_device_graph", "builtin_plan", "canonical_shape", "full_pattern_set",
    "kernel_launch_count", "last_stats", "load_builtin", "lower_all", "lower_plan", "merge_features",
    "mine", "mine_members", "mine_members_device", "mine_rows", "mine_rows_device", "order_plans",
    "prepare_views", "recognize", "release_views", "write_instances",
]

__version__ = "0.1.0"
