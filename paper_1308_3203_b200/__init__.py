"""B200-native concrete SIMD race checker for the §3 kernel language of
arXiv 1308.3203 (the data-parallel hot path of SURVEY.md §8).

    from paper_1308_3203_b200 import rc_load_program, rc_run, rc_explore

The compute path is librc.so (hand-written sm_100a CUDA behind the C ABI in
include/rc.h); this package is its thin ctypes binding plus the multi-GPU
report gather (gather.py).
"""
from .rc import (KINDS, REPORT_DTYPE, ExploreResult, Program, ProveResult, RCError, RunResult, lib,  # noqa: F401
                 rc_explore, rc_last_error, rc_load_program, rc_prove, rc_run)
