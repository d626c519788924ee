"""B200-native modular-arithmetic privacy-amplification hash (arxiv 1910.04429).

Drop-in for the hot path of the reference package ``modpa``: the same names
as ``modpa.pa`` / ``modpa.bignum`` (pkg/src/modpa/__init__.py:10-35), with the
hash and the big-integer product computed by hand-written sm_100a CUDA behind
the C ABI in ``include/pa_b200.h``.  ``batch`` adds the batched,
device-resident API used for throughput (many blocks per launch, streams,
one worker per GPU).
"""
from .bignum import (
    BigNat,
    DEFAULT_THRESHOLDS,
    MulAlgorithm,
    ThresholdTable,
    WordOrder,
    from_words,
    fused_mul_add,
    mod_pow2,
    mul,
    select_algorithm,
    shift_right,
    to_words,
)
from .pa import (
    BitBlock,
    HashSeed,
    PAParams,
    SecurityBoundError,
    compress,
    derive_block_seed,
    export_block,
    gen_seed,
    import_block,
    pa_round,
)
from .security import max_key_length, validate

__version__ = "0.1.0"

__all__ = [
    "BigNat", "MulAlgorithm", "ThresholdTable", "DEFAULT_THRESHOLDS", "WordOrder",
    "from_words", "to_words", "mul", "fused_mul_add", "mod_pow2", "shift_right",
    "select_algorithm",
    "BitBlock", "HashSeed", "PAParams", "SecurityBoundError",
    "import_block", "export_block", "gen_seed", "derive_block_seed", "compress", "pa_round",
    "max_key_length", "validate",
    "__version__",
]
