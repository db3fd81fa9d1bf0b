"""B200-native TP-EP hybrid MoE layer (MixServe, arxiv 2601.08800).

Drop-in for the hot path of the reference ``moeplan`` toolkit: the fused
AG-dispatch / expert / RS-combine MoE layer forward and its routing table,
plus the reference-compatible trace.  The data path runs in hand-written
sm_100a CUDA kernels behind the C-ABI in ``include/mixserve_b200.h``.
"""

__version__ = "0.1.0"

from .errors import (AnalyzerError, CalibrationError, CapacityError,  # noqa: F401
                     ConfigError, GrammarError, MoeplanError, SaturationError,
                     SchedulingError, StrategyError, VerificationError)
from .analyzer import (ProfilingObservation, RankedStrategies, calibrate,  # noqa: F401
                       compare_report, select_strategy)
from .config import (CalibrationCoefficients, ClusterConfig, ConfigBundle,  # noqa: F401
                     ModelHyperparams, WorkloadSpec, load_config)
from .costmodel import (CostEstimate, indicators, lambda_ep_baseline,  # noqa: F401
                        lambda_mix)
from .layer_model import LayerCalibration, predict_layer, select_layout  # noqa: F401
from .plan import GateSpec  # noqa: F401
from .skew import host_loads, host_skew, zipf_logits, zipf_popularity  # noqa: F401
from .strategy import (ParallelStrategy, check_memory, enumerate_strategies,  # noqa: F401
                       format_strategy, parse_strategy)
from .simcluster import (ExpertSpec, FP8SwiGLUExperts, RouterSpec, SimCluster, SwiGLUExperts,  # noqa: F401
                         TraceEvent, build_cluster, build_routing_table,
                         fused_ag_dispatch, fused_rs_combine, moe_oracle,
                         run_moe_block, verify_against_oracle)

__all__ = [
    "__version__",
    "CalibrationCoefficients", "ClusterConfig", "ConfigBundle", "CostEstimate",
    "ModelHyperparams", "ParallelStrategy", "ProfilingObservation",
    "RankedStrategies", "WorkloadSpec", "calibrate", "check_memory",
    "compare_report", "enumerate_strategies", "format_strategy", "indicators",
    "lambda_ep_baseline", "lambda_mix", "load_config", "parse_strategy",
    "select_strategy", "GateSpec", "LayerCalibration", "predict_layer", "select_layout", "host_loads", "host_skew", "zipf_logits", "zipf_popularity",
    "AnalyzerError", "CalibrationError", "CapacityError", "ConfigError",
    "ExpertSpec", "FP8SwiGLUExperts", "GrammarError", "MoeplanError", "RouterSpec",
    "SaturationError", "SchedulingError", "SimCluster", "StrategyError",
    "SwiGLUExperts", "TraceEvent", "VerificationError", "build_cluster",
    "build_routing_table", "fused_ag_dispatch", "fused_rs_combine",
    "moe_oracle", "run_moe_block", "verify_against_oracle",
]
