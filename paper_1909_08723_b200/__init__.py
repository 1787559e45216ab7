"""B200-native fused look-ahead beam decoder (Espresso, arXiv 1909.08723).

Drop-in for the reference ``fusedbeam`` decoding path: same public names
(``decode_batch``, ``decode_corpus``, ``DecodeConfig``, ``DecodeResult``,
``LookaheadFusion``, ``PrefixTreeAutomaton``/``build_trie``,
``TokenDictionary``), computed by hand-written sm_100a kernels behind the C ABI
in ``include/fusedbeam_b200.h``.  See DESIGN.md.
"""

__version__ = "0.1.0"

from .errors import ConfigError, FormatError, FusedBeamError  # noqa: F401
from .token_dict import TokenDictionary, load_dictionary  # noqa: F401
from .lexicon_trie import NO_STATE, PrefixTreeAutomaton, build_trie  # noqa: F401
from .kaldi_io import (FeatureMatrix, ScpEntry, read_ark_matrix, read_feature,  # noqa: F401
                       read_features_pinned, read_scp, write_ark_matrix)
from .fusion import (DEFAULT_OOV_PENALTY, OOV_STATE, FusionScorer, LookaheadBatch,  # noqa: F401
                     LookaheadFusion, MultilevelBatch, MultilevelFusion, SubwordBatch,
                     SubwordFusion, cumsum_distribution)
from .decoder import (AcousticScorer, DecodeConfig, DecodeResult, coverage_improved,  # noqa: F401
                      coverage_original, decode_batch, decode_corpus, eos_allowed)
