"""paper_2410_10447_b200 — B200-native (sm_100a) rebuild of the AutoDock-GPU
scoring hot path of arXiv 2410.10447: warp-per-pose energy+gradient with the
paper's block float4 reduction (shuffle / tensor-core / split-precision
tensor-core), device-resident ADADELTA local search and LGA, behind the
reference's `mdreduce` operator API (C-ABI include/mdr.h, C++
include/mdreduce_b200.hpp, Python mirror in api.py)."""
from ._abi import (  # noqa: F401
    BASELINE,
    HALF,
    PAIR_FP32,
    PAIR_FP64,
    PAIR_FP64_FAST,
    SINGLE,
    TCU,
    TCU_SPLIT,
    DeviceError,
    Instance,
    LgaSettings,
    NumericDomainError,
    ParseError,
    SizeError,
    SyncStats,
    UnsupportedBlockSizeError,
    derive_rng,
    parse_instance,
    random_instance,
    random_pose,
    serialize_instance,
)
from .api import Device, DockResult, LocalSearchResult, ScoreResult, summarize, validate_pair  # noqa: F401

__version__ = "0.1.0"
