"""B200-native MASQuant hot path (arXiv 2603.04800): modality-aware smoothed quantized linear.

C ABI: include/masq.h (libmasq.so, sm_100a kernels in csrc/).  Python binding: masq.py.
"""
from . import masq  # noqa: F401
from .masq import (  # noqa: F401
    MasqError, Workspace, adam_init, adam_step, calib_loss, calib_loss_grad, calibrate_stats, check, init_factors, keep_best, linear_forward, loss_finalize,
    quantize_activations, quantize_weight, reference_output, workspace_size, smooth_factors, calibrate_meanabs,
    range_stats, count_modalities, cmc_factors, cmc_gram, cmc_factors_from_gram, calib_layer, quantize_weight_int4, unpack_int4, linear_decode,
    quantize_weight_w4g, linear_forward_w4g,
)
