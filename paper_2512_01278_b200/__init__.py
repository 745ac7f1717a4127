"""B200-native SparseSpec / PillarAttn decode hot path (arXiv 2512.01278).

Drop-in for the reference ``spardec`` package's hot-path API: attention
operators (``forward_full``, ``forward_sparse``), KV-cache manager
(``KvCache``, ``KvPool``), selection, the draft/verify engine and the
unified draft/verify scheduler.  The arithmetic runs in the in-tree sm_100a
C-ABI library ``_lib/libspardec_b200.so`` (see ``include/spardec_b200.h``);
there is no CPU fallback.
"""

from . import _native
from .engine import (DecodeRequest, RequestState, RoundOutcome, RoundRecord, RoundStats, decode_to_completion,
                     draft_step, greedy_decode, prefill, verify_round)
from .errors import (CalibrationError, ConfigurationError, ContractError, DegenerateParameterError,
                     ImpossibleRequestError, SimulationError, SpardecError, StateMachineError)
from .kvpool import KvPolicy, KvPool, page_bytes_per_token
from .model import (KvCache, KVEntry, ModelConfig, ToyModel, forward_full, forward_sparse, greedy_token, init_model,
                    plant_attention_concentration)
from .scheduler import (BatchCandidate, IterationBatch, PhaseBuckets, PipelineMode, PipelineSlot, SchedPolicy,
                        assign_new_request, balance_metric, first_round_draft_len, form_batch, step_pipeline)
from .selection import (AttentionScoreLog, CriticalTokenSet, ScoreRow, aggregate_scores, compute_budget,
                        importance_from_log, pad_rows, rematerialize_scores, select_critical_tokens)
from .simulate import KvPoolConfig, SimConfig, SimReport, run_token_sim
from .workload import ArrivalKind, ArrivalSpec, LengthDist, LengthSpec, SimRequest, WorkloadSpec, generate_workload

try:  # load the in-tree CUDA library eagerly when it has been built
    _native.load_library()
except ImportError:  # calls into kernels raise loudly until it is built
    pass

__version__ = "0.1.0"

__all__ = [
    "ArrivalKind", "ArrivalSpec", "KvPoolConfig", "LengthDist", "LengthSpec", "ScoreRow", "SimConfig", "SimReport",
    "SimRequest", "WorkloadSpec", "aggregate_scores", "generate_workload", "pad_rows", "rematerialize_scores",
    "run_token_sim",
    "AttentionScoreLog", "BatchCandidate", "CalibrationError", "ConfigurationError", "ContractError",
    "CriticalTokenSet", "DecodeRequest", "DegenerateParameterError", "ImpossibleRequestError", "IterationBatch",
    "KVEntry", "KvCache", "KvPolicy", "KvPool", "ModelConfig", "PhaseBuckets", "PipelineMode", "PipelineSlot",
    "RequestState", "RoundOutcome", "RoundRecord", "RoundStats", "SchedPolicy", "SimulationError", "SpardecError",
    "StateMachineError", "ToyModel", "assign_new_request", "balance_metric", "compute_budget",
    "decode_to_completion", "draft_step", "first_round_draft_len", "form_batch", "forward_full", "forward_sparse",
    "greedy_decode", "greedy_token", "importance_from_log", "init_model", "page_bytes_per_token",
    "plant_attention_concentration", "prefill", "select_critical_tokens", "step_pipeline", "verify_round",
]
