"""B200-native DartMinHash sketching: weighted minhashes, 1-bit sketches and
(L, K) LSH keys for batches of sparse weighted sets, computed by hand-written
sm_100a CUDA kernels behind a C ABI (include/dsk_b200.h).

The public names mirror the reference package `dartsketch`
(/root/reference/pkg/src/dartsketch/__init__.py) for the hot path; see
DESIGN.md for the boundary and INTEGRATION.md for the ctypes binding.
"""

from .constants import ValidationError, derive_seed, minhash_density
from . import io, shard, workloads
from .api import (
    DSK_STATUS_TIE,
    IcwsBatch,
    IcwsHashValue,
    IcwsSketcher,
    icws_batch,
    icws_estimate_jaccard,
    icws_fingerprints,
    icws_minhash,
    BottomKBatch,
    BottomKFingerprints,
    BottomKSketch,
    bottom_k,
    bottom_k_batch,
    dump_sketch,
    dump_sketches,
    iter_sketches,
    l1_batch,
    load_sketch,
    Dart,
    DartBatch,
    DartHasher,
    HashFamily,
    LshBatch,
    LshParams,
    MinhashBatch,
    MinHashSketch,
    OneBitSketch,
    WeightedSet,
    as_u64,
    dart_minhash,
    darts_batch,
    lsh_batch,
    lsh_key,
    make_weighted_set,
    minhash_batch,
    one_bit,
    raise_for_status,
    weight_class,
    exact_jaccard,
)

__all__ = [
    "ValidationError", "minhash_density", "DSK_STATUS_TIE", "Dart", "DartBatch", "DartHasher",
    "HashFamily", "LshBatch", "LshParams", "MinhashBatch", "MinHashSketch", "OneBitSketch",
    "WeightedSet", "as_u64", "dart_minhash", "darts_batch", "lsh_batch", "lsh_key",
    "make_weighted_set", "minhash_batch", "one_bit", "raise_for_status", "weight_class",
    "BottomKBatch", "BottomKFingerprints", "BottomKSketch", "bottom_k", "bottom_k_batch",
    "dump_sketch", "dump_sketches", "iter_sketches", "l1_batch", "load_sketch",
    "IcwsBatch", "IcwsHashValue", "IcwsSketcher", "icws_batch", "icws_estimate_jaccard",
    "icws_fingerprints", "icws_minhash", "exact_jaccard", "derive_seed",
]

from .lsh_index import LshIndex, probe_classes  # noqa: E402

__all__ += ["LshIndex", "probe_classes"]
