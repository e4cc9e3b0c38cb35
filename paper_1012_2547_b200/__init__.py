"""B200-native exact string matching engine (drop-in for matchbench's search path).

Public surface mirrors the reference package's search entry points
(pkg/src/matchbench/__init__.py:73-132): ``brute_force_search``, every
``search_*``, ``AlgorithmDescriptor`` / ``REGISTRY`` / ``get_algorithm`` /
``select_applicable``, the domain types, plus engine-native ``search``,
``count`` and ``search_many`` (batched mode).  Every search runs on the
sm_100a kernels in libmatchb200.so; there is no CPU fallback.
"""
from .core import (
    WORD,
    ApplicabilityError,
    InstrumentedText,
    Pattern,
    Text,
    WordSpec,
    as_haystack,
    as_needle,
    brute_force_search,
    verify_equal,
)
from .differential import DifferentialReport, Mismatch, run_differential
from .harness import (
    ALLOWED_SIGMAS,
    CORPUS_EXPECTATIONS,
    DEFAULT_LENGTHS,
    BenchConfig,
    Measurement,
    generate_rand_text,
    load_corpus,
    run_benchmark,
    sample_patterns,
    sample_positions,
    standard_texts,
    state_word_count,
)
from .registry import (
    B200,
    DEFAULT_SELECTION_MAP,
    REGISTRY,
    AlgorithmDescriptor,
    SelectionMap,
    SizeClasses,
    applicable_algorithms,
    b200_descriptor_for,
    build_registry,
    classify,
    get_algorithm,
    select,
    select_applicable,
)
from .searchers import (
    compile_engine,
    compile_tensor,
    count,
    search,
    search_bmh_sbndm,
    search_bndm,
    search_bom,
    search_br,
    search_ebom,
    search_fjs,
    search_fsbndm,
    search_hashq,
    search_hor,
    search_lbndm,
    search_many,
    search_qs,
    search_sa,
    search_sbndm,
    search_sbndm_bmh,
    search_sbndmq,
    search_so,
    search_ssef,
    search_tvsbs,
)

__version__ = "0.1.0"
