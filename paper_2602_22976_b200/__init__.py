"""paper_2602_22976_b200 -- B200-native locally-maximal hypergraph matching (HLM).

Drop-in for the reference's CPU matching path (proj/include/hlm/local_max_par.hpp): hypergraph
CSR in, matched-edge set and weight out, bit-exact.  The work is done by hand-written sm_100a
CUDA kernels in lib/libhlm_b200.so (C-ABI: include/hlm_b200.h); this package is the thin host
mirror of the reference API.  There is no CPU fallback.
"""
from ._lib import LIB_PATH, load_library  # noqa: F401
from .api import (  # noqa: F401
    DeviceError,
    DeviceHypergraph,
    Hypergraph,
    InputError,
    MatchResult,
    Matching,
    ParallelConfig,
    RoundLimitError,
    RunReport,
    VerificationReport,
    WeightStream,
    CompactResult,
    WorkCounters,
    compact,
    default_max_rounds,
    eval_stream,
    generate_random,
    generate_tight_family,
    load_instance_file,
    local_max_crcw,
    local_max_crew,
    parse_hgr,
    parse_matching,
    parse_metis_graph,
    random_weights_1_100,
    run_variant,
    verify_matching,
    write_hgr,
    write_matching,
)
