"""B200-native module-level scaling data path of CoCoServe (arxiv 2507.18006).

Drop-in for the reference package ``modscale`` on the north-star path: the
module registry (``PlacementState``), the scaling operator (``apply`` and the
op types), the batch splitter / replica router (``split_batch``,
``replica_runs``, ``schedule``) and the executor hook (``step_batch``) -- with
the data path itself (decoder-layer forward, KV cache, scatter/gather,
replication/migration copies) running as sm_100a kernels in libcocob200.so.
"""
from .domain import (  # noqa: F401
    ClusterSpec,
    DeviceSpec,
    DeviceUsage,
    DomainError,
    ModelSpec,
    ModuleCatalog,
    ModuleKind,
    PlacementState,
    Replica,
    UnknownDeviceError,
    derive_parallelism_vector,
    device_usage,
    kv_resident_layer_count,
    vacancy_rate,
)
from .ops import (  # noqa: F401
    BatchApplyError,
    EvictReplica,
    InfeasibleOpError,
    MigrateLayer,
    MigrateSubModule,
    MissingReplicaError,
    OpCostModel,
    OpError,
    OpRecord,
    ReplicateLayer,
    TransitionCost,
    aggregate_cost,
    apply,
    batch_apply,
    replica_runs,
    split_batch,
)

__version__ = "0.1.0"
