"""B200-native (sm_100a) per-layer hot path of Zeppelin (arXiv 2509.21841).

Drop-in for the reference package ``varlenplan`` on its hot path: the same
planner / schedule / remap names (``build_plan``, ``build_schedule``,
``solve_remap``, ...; reference ``__init__.py:3-40``) with bit-identical
results, plus execution entry points that run the plan on B200s
(``attention_forward``, ``remap_forward``, ``remap_inverse``,
``ZeppelinLayer``).  The device work is done by hand-written sm_100a kernels
behind the C ABI in ``include/zeppelin_b200.h``; there is no CPU fallback.
"""

from .baselines import STRATEGIES, plan_hybrid_dp, plan_llama_cp, plan_te_cp
from .batch import LengthDistribution, SequenceBatch, load_batch, preset, sample_batch, save_batch
from .cluster import ClusterSpec, ConfigError, single_box
from .plan import (
    Fragment,
    InfeasibleBatch,
    InfeasibleNode,
    PlacementPlan,
    PlanValidationError,
    build_plan,
    load_plan,
    partition_inter_node,
    partition_intra_node,
    plan_from_json,
    plan_to_json,
    save_plan,
    validate_plan,
)
from .remap import (
    RemapLayout,
    RemapResult,
    cost_matrix,
    remap_cost_pair,
    remap_layout,
    solve_remap,
    target_distribution,
)
from .routing import RoutePlan, RouteStep, build_route, route_schedule, routed_time, select_proxies
from .schedule import (
    AttentionSchedule,
    LocalTask,
    RingGroup,
    RingRound,
    RingSchedule,
    RingSequence,
    build_schedule,
    causal_pairs,
    split_even,
    visible_pairs,
    zigzag_chunks,
)

__version__ = "0.1.0"


def __getattr__(name):
    # execution entry points pull in torch + the native library lazily, so the
    # planner API stays importable on hosts without CUDA.
    if name in ("attention_forward", "remap_forward", "remap_inverse", "ZeppelinLayer", "RankContext"):
        from . import engine
        return getattr(engine, name)
    raise AttributeError(name)
