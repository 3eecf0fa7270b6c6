"""B200-native tree-ensemble scoring engine (drop-in for the reference
``treescore`` predict path; arXiv 1212.2287's computation on sm_100a).

Model and data layers mirror the reference names (``Node``, ``Tree``,
``Ensemble``, ``CompleteTree``, ``expand_to_complete``, ``parse_model``,
``serialize_model``, ``Dataset``, ``read_fvec`` ...).  Scoring runs only in
the native library ``_ts_gpu.so`` (C ABI ``include/treescore_gpu.h``) through
``build`` / ``build_gpu`` -> :class:`GpuEvaluator`; there is no CPU fallback.
"""

from .data import (DataFormatError, Dataset, as_feature_vector, fvec_header, read_fvec,
                   read_fvec_into, write_fvec)
from .evaluator import (ALL_STRATEGIES, CoverageReport, GpuEvaluator, GpuModel, StrategyKind, TracedPrediction,
                        build, build_gpu, measure_feature_coverage, predict_ensemble_traced)
from .model import (DUMMY_FID, DUMMY_THETA, MAX_DEPTH, CompleteTree, DepthLimitError,
                    Ensemble, FlatModel, ModelError, ModelSemanticError, ModelSyntaxError,
                    Node, Tree, expand_to_complete, load_flat_model, load_model, parse_model,
                    parse_model_native,
                    reference_predict, save_model, serialize_model, traverse_to_leaf,
                    TreeStats, tree_stats)
from ._lib import NativeLibraryError

__version__ = "0.1.0"

__all__ = [
    "ALL_STRATEGIES",    "CompleteTree", "CoverageReport", "TracedPrediction", "DataFormatError", "Dataset", "DepthLimitError", "DUMMY_FID",
    "DUMMY_THETA", "Ensemble", "FlatModel", "GpuEvaluator", "GpuModel", "MAX_DEPTH",
    "ModelError", "ModelSemanticError", "ModelSyntaxError", "NativeLibraryError", "Node",
    "StrategyKind", "Tree", "as_feature_vector", "build", "build_gpu", "expand_to_complete",
    "fvec_header", "load_flat_model", "measure_feature_coverage", "predict_ensemble_traced", "load_model", "parse_model", "parse_model_native",
    "read_fvec", "read_fvec_into",
    "reference_predict", "save_model", "serialize_model", "traverse_to_leaf", "TreeStats", "tree_stats",
    "write_fvec",
]
