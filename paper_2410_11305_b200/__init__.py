"""B200-native QSpec decode hot path (arXiv 2410.11305) -- drop-in for the reference's public API.

Names and config fields follow pkg/src/qspec/__init__.py:9-95 for the decode
path: quantise, forward, draft, verify, accept, generate.  Device work runs in
the in-tree sm_100a extension ``libqspec_b200.so`` (C ABI: include/qspec_b200.h);
importing this package does not need a GPU, calling a device op does.
"""

from .errors import (CheckpointError, ConfigError, QSpecError, SequenceOverflowError, ShapeError, TokenIdError,
                     TraceError, WorkloadError)
from .model import (CostCounter, KVCache, LayerWeights, LogitsBlock, ModelConfig, TransformerModel, WriteTarget,
                    forward, kv_commit, kv_memory_report, kv_reset)
from .numerics import rmsnorm
from .quant import (ExecutionMode, QuantizedTensor, activation_quant_calls, dequantize,
                    fake_quantize_activations, pack_int4, qlinear_forward, quantize_groupwise,
                    reset_activation_quant_calls, start_qlinear_log, stop_qlinear_log, unpack_int4)
from .specdec import (CycleRecord, GenerationConfig, GenerationResult, SequenceEngine, TokenSource, accept_greedy,
                      draft_phase, format_cycle_record, format_trace, generate_greedy, generate_qspec, parse_trace,
                      verify_phase)
from .storage import (config_from_text, config_to_text, load_checkpoint, model_from_float_tensors, random_init,
                      read_checkpoint, save_checkpoint)
from .serving import (LatencySplit, RejectedRequest, Request, ServingStats, format_stats, parse_workload,
                      per_valid_token_latency, run_fcfs)

__version__ = "0.1.0"
