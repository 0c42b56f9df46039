"""B200-native tile-wise (TW) sparse GEMM (arXiv 2008.13006), drop-in for the
hot path of the reference package `tilewise`: masks -> packed plans ->
one persistent sm_100a tcgen05 kernel, plus the TEW CSR SpMM and the
N-sharded multi-GPU launcher.  See DESIGN.md."""

from .matrix import (
    ConfigError,
    CscMatrix,
    DenseMatrix,
    DimensionError,
    FormatError,
    GemmShape,
    Layout,
    csc_to_dense,
    to_csc,
    transpose,
)
from .pattern import (
    CompactTile,
    CompactTileSet,
    PatternStats,
    Tile,
    TileConfig,
    TilePattern,
    compact,
    dense_pattern,
    exact_count,
    mask_words_to_indices,
    pack_mask_words,
    partition,
    pattern_stats,
    pruned_columns,
    random_uniform_pattern,
    reorganize_columns,
    unpack_mask_words,
    zero_fill,
)
from .sharded import ShardedTwPlan, all_gather_rows, shard_ranges
from .layers import TwMlp, engine_logits
from .pruning import ScoreMap, TewConfig, magnitude_scores, prune_stage, tew_overlay
from .formats import (plan_from_files, read_csc, read_matrix, read_model, read_pattern, write_csc, write_matrix,
                      write_pattern)
from .engine import (
    PRECISIONS,
    BatchGroup,
    DeviceCsc,
    TileTask,
    execute_batched,
    gather_rows,
    group_by_shape,
    prep_activations_split,
    FlopReport,
    PackedPlan,
    TwPlan,
    flop_report,
    gemm_dense,
    gemm_tew,
    gemm_tw,
    prep_activations,
    spmm_csc,
    spmm_csc_device,
    time_median,
)

__version__ = "0.1.0"
