"""B200-native SPECTRE decode loop (arxiv 2605.08151).

Public names mirror the reference package's decoder surface
(/root/reference/pkg/src/specsim/__init__.py:48-88) for the hot path:
`run`, `run_sweep`, `SimConfig`, `PolicyVariant`, `MetricsReport`,
`RunResult`, `TokenStreamOracle`, `VerifyOutcome`, `Mode`, `PAD`, plus the
model-mode engine (`paper_2605_08151_b200.model`).  Every compute path runs
in libspectre.so (hand-written sm_100a CUDA); importing a compute entry point
without the library raises — there is no CPU fallback.
"""

from .analytics import (
    ThroughputParams,
    critical_fallback_ratio,
    expected_committed_per_round,
    generalized_critical_ratio,
    ordinary_throughput,
    parallel_throughput,
    preferred_mode,
)
from .core import PAD, ConfigError, Mode, SimConfig, SpeculativeSegment, validate_config
from .decoder import (
    OutsideDeviceDomain,
    PolicyVariant,
    ProtocolViolation,
    RoundTrace,
    RunResult,
    SimLivelock,
    SweepEntry,
    Workload,
    run,
    run_sweep,
)
from .metrics import (
    REPORT_COLUMNS,
    MetricsReport,
    export_report,
    import_report,
    mean_accepted_length,
    write_report,
)
from .oracle_pair import TokenStreamOracle, VerifyOutcome

__version__ = "0.1.0"

__all__ = [
    "PAD", "ConfigError", "MetricsReport", "Mode", "OutsideDeviceDomain", "PolicyVariant",
    "ProtocolViolation", "REPORT_COLUMNS", "RoundTrace", "RunResult", "SimConfig",
    "SimLivelock", "SpeculativeSegment", "SweepEntry", "ThroughputParams",
    "TokenStreamOracle", "VerifyOutcome", "Workload", "critical_fallback_ratio",
    "expected_committed_per_round", "export_report", "generalized_critical_ratio",
    "import_report", "mean_accepted_length", "ordinary_throughput", "parallel_throughput",
    "preferred_mode", "run", "run_sweep", "validate_config", "write_report", "__version__",
]
