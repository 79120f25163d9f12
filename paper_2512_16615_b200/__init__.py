"""B200-native Log-linear Sparse Attention (arXiv 2512.16615) hot path.

Hand-written sm_100a CUDA kernels behind a C ABI (include/llsa_cuda.h); this
package is the Python mirror of the reference operator API (ops.py) plus the
autograd wrapper (autograd.py).  No CPU fallback: importing the ops loads
lib/libllsa_cuda.so and raises if it was not built.
"""
from . import _lib
from ._lib import (ArgumentError, ConfigError, CudaError, DivisibilityError, Error,
                   IndexOutOfRange, LevelError, NonFiniteError, NotSquareBlock, ShapeMismatch,
                   StaleState,
                   TopKError, Unsupported)
from .ops import (ForwardState, LLSAConfig, LLSAHandle, ValidatedConfig, apply_permutation,
                  build_plan, build_pyramid, build_pyramid_permuted, build_reorder,
                  dump_selection, effective_block_count, hierarchical_topk,
                  kv_backward, llsa_backward, llsa_forward, mask_kv_backward, max_levels, pool_backward,
                  pyramid_levels, select_coarsest, select_level, split_tables, sync_status,
                  transpose_all, transpose_indices, validate_config)

__all__ = [n for n in dir() if not n.startswith("__")]
from .autograd import LLSAAttention  # noqa: E402
