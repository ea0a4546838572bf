"""B200-native cascade-hashing feature matcher (hot path of arXiv 2505.22089).

Drop-in for the reference bandmatch library's matching path: hash codes,
bucket tables, Hamming top-K, Euclidean re-rank and ratio test run as
hand-written sm_100a kernels behind the C ABI in include/bandmatch_gpu.h
(libbmg.so, built in-tree by ``__graft_entry__.build()``).  This package is the
Python face of the same API (names follow include/bandmatch/hashmatch.hpp and
engine.hpp).  There is no CPU fallback.
"""
from ._lib import BandmatchError, LIB_PATH, load  # noqa: F401
from .hashmatch import (FeatureSet, HashCodeSet, HashFunctions, HashParams, Matcher,  # noqa: F401
                        MatchParams, PairMatches, compute_codes, make_hash_functions, match_pair,
                        read_matches_binary, read_matches_text, seed_for, write_matches_binary,
                        write_matches_text)
from .engine import (BlockRow, DeviceArena, ExecuteOptions, ExecutionResult,  # noqa: F401
                     PipelineMetrics, ScheduleBlock, ScheduleIteration, SchedulePlan,
                     arena_units_for, execute_plan, flatten_plan, read_plan, write_plan)
from .retrieval import (Codebook, VladVector, encode_vlad, encode_vlad_batch,  # noqa: F401
                        read_codebook, train_codebook, write_codebook)

__version__ = "0.1.0"
