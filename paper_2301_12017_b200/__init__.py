"""paper_2301_12017_b200 -- B200-native (sm_100a) W4A4 encoder hot path of arXiv
2301.12017 ("Understanding INT4 Quantization for Transformer Models", §"Highly Optimized
INT4 Encoder Inference").

The product is the C-ABI library libq4.so (include/q4.h, csrc/); this package is its
thin Python binding.  PyTorch provides device memory, streams, CUDA graphs and
torch.distributed -- plumbing, not the product.  There is no CPU fallback."""
from ._lib import (EPI_F16, EPI_GELU_Q4, EPI_I32, EPI_RESLN_Q4, MAINLOOP_AUTO,
                   MAINLOOP_MMA_SYNC_S4, MAINLOOP_MMA_SYNC_S8, MAINLOOP_TCGEN05, MAINLOOP_TCGEN05_W8,
                   MAINLOOP_TCGEN05_W8_1CTA, Q4Error,
                   launch_count, lib, version)
from .ops import (attention_f16_q4, encoder_layer, encoder_layer_workspace_bytes, prepack_weights, quantize_layer, quantize_rows,
                  quantize_rows_i8, w4a4_linear, w8a8_linear, attention_f16_q8, f16_linear, quantize_rows_asym, weight_code_sums,
                  w4a4_asym_linear, launch_floor, attention_f16_q4_asym,
                  prune_24, sparse24_compress, w4a4_sparse24_linear)
from .encoder import W4A4Encoder, W8A8Encoder
from . import tune

__all__ = [
    "EPI_I32", "EPI_F16", "EPI_GELU_Q4", "EPI_RESLN_Q4", "MAINLOOP_AUTO", "MAINLOOP_TCGEN05",
    "MAINLOOP_MMA_SYNC_S8", "MAINLOOP_MMA_SYNC_S4", "MAINLOOP_TCGEN05_W8", "MAINLOOP_TCGEN05_W8_1CTA", "prepack_weights", "Q4Error", "lib", "version", "launch_count", "launch_floor", "attention_f16_q4_asym", "prune_24", "sparse24_compress", "w4a4_sparse24_linear",
    "quantize_rows", "w4a4_linear", "quantize_rows_i8", "w8a8_linear", "attention_f16_q4", "encoder_layer", "encoder_layer_workspace_bytes", "quantize_layer",
    "W4A4Encoder", "W8A8Encoder", "attention_f16_q8", "f16_linear", "quantize_rows_asym", "weight_code_sums", "w4a4_asym_linear",
]
