"""B200-native (sm_100a) QFT quantized model-state update path.

Drop-in for the reference's quantizer/optimizer API (qft::quantize_state,
decompose_weight, requantize_weight, reconstruct, lion_step_quantized; the
``qft_engine`` Python functions) over a C-ABI (include/qft_b200.h).  Importing
fails loudly when the CUDA library has not been built: there is no CPU path.
"""
from . import _native  # noqa: F401  (raises ImportError if the .so is missing)
from .engine import QftModelState
from .quantize import (AffineParams, DenseSparseWeight, GradientStack, LionHyper, LionState,
                       accumulate,
                       QuantizedTensor, SparseOutliers, affine_params_from_bounds, byte_size,
                       channel_minmax, compute_affine_params, compute_outlier_thresholds,
                       decompose_dense_sparse, decompose_weight, dequantize, lion_apply,
                       lion_step_quantized, quantize, quantize_state, reconstruct,
                       requantize_weight, synth)

__all__ = [
    "QftModelState", "accumulate", "AffineParams", "DenseSparseWeight", "GradientStack", "LionHyper",
    "LionState", "QuantizedTensor", "SparseOutliers", "affine_params_from_bounds", "byte_size",
    "channel_minmax", "compute_affine_params", "compute_outlier_thresholds",
    "decompose_dense_sparse", "decompose_weight", "dequantize", "lion_apply",
    "lion_step_quantized", "quantize", "quantize_state", "reconstruct", "requantize_weight",
    "synth",
]
