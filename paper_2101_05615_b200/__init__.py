"""B200-native quantized u8 x s8 -> s32 GEMM with fused requantization — the
hot path of arXiv 2101.05615 (FBGEMM), behind the reference q8gemm API."""
from .api import (  # noqa: F401
    ROUND_F32_RNE,
    ROUND_REF,
    BiasAdd,
    BlockingParams,
    DepthwiseFilter,
    KernelCache,
    KernelVariant,
    OutputPipeline,
    PackedWeight,
    ReluQuantized,
    Requantize,
    RequantParams,
    QuantParams,
    SparseWeightCSC,
    SpMDMAdd,
    SplitWeight,
    WriteDequantF32,
    WriteRawI32,
    execute_conv3x3,
    execute_dwconv3x3,
    execute_gemm,
    i16_accumulation_exact,
    partition_stripes,
    stripe_rows,
    split_outliers,
    prepack_conv3x3_weights,
    prepack_weights,
    select_blocking,
)
from ._lib import InvalidArgument, Q8GError, launch_count, launch_stats  # noqa: F401
from .nshard import NShardedGemm, column_shard, execute_gemm_to_peers  # noqa: F401,E402
