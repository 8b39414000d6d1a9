"""paper_2601_16991_b200 -- B200-native (sm_100a) SALR linear hot path.

A drop-in for the hot path of the reference ``salr`` package (SALR,
arXiv 2601.16991): bitmap encoding of the pruned base weight, concatenated
adapters, and the SALR linear forward ``y = x @ W_hat + (x @ A_cat) @ B_cat``.
Names and signatures mirror the reference's public API
(``pkg/src/salr/__init__.py:10-84``, hot-path subset); arrays live on the GPU
as torch tensors and every compute step runs in the hand-written CUDA
library ``libsalr_b200.so`` (no CPU fallback).
"""

from .errors import (BoundsError, ConfigError, CorruptionError, DomainError, FormatError, SalrError,
                     ShapeError, VerificationError)
from .linalg import SvdResult, as_matrix, matmul, matmul_call_count, reset_matmul_count, svd
from .residual import (AdapterPair, ResidualTrainConfig, StepSizeMode, build_residual_adapter,
                       lipschitz_constant, optimal_step_size, power_iteration_sigma_max, residual_gradient,
                       residual_loss, train_residual, truncation_error_bound)
from .fusion import FusedAdapters, apply_fused, apply_sequential, forward, fuse
from .bitmap import (BitmapSparseMatrix, build_lut, bytes_per_row, compression_ratio, container_size_bytes,
                     decode, decode_block, encode, header_bytes, kept_count, popcount8, read_container,
                     write_container)
from .pipeline import (BenchResult, PipelineConfig, PipelineProbe, SlotState, bench, launch_count,
                       pipelined_forward, pipelined_matmul, reset_launch_count, salr_chain, salr_linear,
                       validate_transitions)
from .prune import PruneConfig, PruneMethod, build_mask, prune

__version__ = "0.1.0"
