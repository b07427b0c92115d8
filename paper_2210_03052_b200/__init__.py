"""paper_2210_03052_b200 -- B200-native (sm_100a) padding-free BERT encoder
forward, a drop-in for the reference package ``packbert``'s encoder path
(ByteTransformer, arXiv 2210.03052).

Same public names as ``packbert`` for the hot path: ``SeqLengths``,
``build_mask``, ``compute_plan``, ``plan_for_lengths``, ``pack``, ``unpack``,
``AttentionInput``, ``dispatch_mha``, ``add_bias_residual_layernorm``,
``ModelConfig``, ``OptFlags``, ``init_weights``, ``encoder_layer``,
``forward`` ...  All compute runs in ``libbt200.so`` (hand-written tcgen05 /
TMA / TMEM CUDA for sm_100a) through the C ABI in ``include/bt200.h``.
"""

__version__ = "0.1.0"

from .attention import AttentionInput, dispatch_mha, mha_fused_long, mha_fused_short
from .encoder import (
    BERT_LARGE,
    PRESETS,
    BertEncoderB200,
    EncoderWeights,
    LayerWeights,
    ModelConfig,
    OptFlags,
    encoder_layer,
    engine_for,
    forward,
    forward_stream,
    init_weights,
    load_weights,
    parse_config_file,
    parse_config_text,
    preset_config,
    save_weights,
)
from .errors import ConfigError, PackbertError, ShapeError, WeightFormatError
from .fusion import LayernormParams, add, add_bias_residual_layernorm, add_rowvec, bias_gelu_epilogue, gelu, layernorm
from .packing import PackedBatch, PackingPlan, SeqLengths, build_mask, compute_plan, pack, plan_for_lengths, unpack
from .tensor import EpilogueHook, EpilogueKind, FlopCounter, Tensor, batched_gemm, gemm
from .partition import forward_sharded, token_balanced_partition
