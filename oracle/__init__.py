"""TEST INFRASTRUCTURE ONLY — the CPU oracle (see oracle.c header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this package.  The product path (paper_1308_3203_b200/) never does.
"""
from .oracle import (Result, build, enumerate_interval, run, state_at, STATUS,
                     REPORT_DTYPE)  # noqa: F401
