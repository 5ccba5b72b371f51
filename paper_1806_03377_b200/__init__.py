"""B200-native PipeDream (arXiv 1806.03377) pipeline-parallel training runtime.

Drop-in for the reference package ``pipesim``'s hot path: the same plan,
schedule, config, ledger and result types, and ``run(cfg, ctx, schedule)``
executes the 1F1B-RR schedule on B200s (tcgen05 GEMM kernels, on-device
weight-version ring, peer-store inboxes) instead of simulating it.
"""

__version__ = "0.1.0"

import os as _os

# Every hosted worker issues on its own stream (plus a reduction stream per replicated worker):
# give them their own hardware work queues when this process creates its CUDA context (the default
# of 8 folds more streams onto shared queues, serialising independent stages).
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from .errors import (  # noqa: F401
    ConsistencyError,
    NativeError,
    PipesimError,
    ProfileFormatError,
    SimulationError,
    ValidationError,
)
from .executor import Executor, run  # noqa: F401
from .ledger import (  # noqa: F401
    Mode,
    SimConfig,
    SimReport,
    SimResult,
    StalenessViolation,
    TraceEvent,
    VersionLedger,
    analytic_throughput,
    build_report,
    compare_analytic,
    staleness_check,
    write_trace_csv,
)
from .models import (  # noqa: F401
    ConvNetSpec,
    GPTSpec,
    LayerDef,
    gpt2_medium,
    MLPSpec,
    init_params,
    init_params_any,
    make_data,
    make_data_any,
    mlp,
    mlp_context,
    mlp_profile,
    vgg16,
)
from .orders import (  # noqa: F401
    Direction,
    Schedule,
    WorkItem,
    assigned_minibatches,
    build_schedule,
    replica_for,
    stage_inflight_caps,
    worker_order,
    write_schedule_csv,
)
from .plans import (  # noqa: F401
    Plan,
    Stage,
    load_plan,
    noam,
    noam_for,
    parse_config,
    plan_from_dict,
    replicated_plan,
    solve,
    straight_plan,
)
from .profiles import (  # noqa: F401
    CostContext,
    HardwareSpec,
    LayerProfile,
    ModelProfile,
    build_context,
    comm_time_activations,
    comm_volume_bsp,
    comm_volume_pp,
    compute_time,
    load_profile,
    save_profile,
    stage_time,
    weight_sync_time,
)
from .profiler import profile_mlp, profile_model  # noqa: F401
from .program import Program, compile_program, resolve_versions  # noqa: F401
