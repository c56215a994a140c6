"""B200-native Bottleneck-aware Tensor Parallelism (BTP) for CoLA low-rank decoder blocks.

Drop-in for the BTP path of the reference package `btpsim` (pkg/src/btpsim/__init__.py:9-42):
the same config / plan / execution names, with the block computed on sm_100a tensor cores
through libbtp.so (include/btp.h) and the TP collectives on NCCL. Additions the reference does
not have: `train_step` (forward + backward), `BlockTrainer` (resident, CUDA-graph replayed
training step with fused AdamW), the naive-TP / full-rank executors on the same kernels, the
multi-layer model (`build_model`, `ModelTrainer`) and the peer-memory chunk boundaries
(`boundary="peer"`).
"""

from .tensor import DimensionError, DivisibilityError, Tensor, seeded_fill, tensor, zeros
from .model import (
    COLA_60M,
    PRESETS,
    DecoderBlockWeights,
    ModelConfig,
    RunShape,
    Variant,
    build_block,
    ModelWeights,
    build_model,
    fan_in_scaled,
    preset,
    projection_dims,
    seeded_h_prev,
    token_batch,
    zero_h_prev,
)
from .plan import NormMode, PlanError, ShardPlan, Strategy, apply_grouping, describe, enumerate_collectives, plan
from .trace import CollectiveRecord, Trace, ring_transfer_elements, trace_volume
from .api import (BlockTrainer, ModelTrainer, SimResult, StepResult, execute_forward, make_executor,
                  reference_forward, train_step)
from .tensor_ops import batched_matmul, matmul, swiglu
from .checkpointing import CkptPolicy, CkptReport, eff_ckpt, run_with_ckpt
from .config import (ConfigError, Scenario, add_config_flags, apply_overrides, build_plan, load_scenario,
                     run_scenario, scenario_from_dict)
from . import config as cli  # the reference keeps its config API in `btpsim.cli` (cli.py:55-304)
import sys as _sys

_sys.modules.setdefault(__name__ + ".cli", cli)   # `import paper_2512_12131_b200.cli as cli` works too

__all__ = [
    "Tensor", "tensor", "zeros", "seeded_fill", "DimensionError", "DivisibilityError",
    "ModelConfig", "RunShape", "Variant", "PRESETS", "COLA_60M", "preset", "projection_dims",
    "DecoderBlockWeights", "build_block", "fan_in_scaled", "ModelWeights", "build_model", "token_batch",
    "zero_h_prev", "seeded_h_prev",
    "Strategy", "NormMode", "ShardPlan", "PlanError", "plan", "apply_grouping", "describe",
    "enumerate_collectives",
    "CollectiveRecord", "Trace", "trace_volume", "ring_transfer_elements",
    "execute_forward", "reference_forward", "matmul", "batched_matmul", "swiglu", "train_step", "make_executor", "BlockTrainer", "ModelTrainer", "SimResult", "StepResult",
    "CkptPolicy", "CkptReport", "eff_ckpt", "run_with_ckpt",
    "ConfigError", "Scenario", "scenario_from_dict", "load_scenario", "apply_overrides", "build_plan",
    "add_config_flags", "run_scenario", "cli",
]

__version__ = "0.1.0"
