"""CPU oracle (test infrastructure only; see oracle.c header)."""
from .oracle import *  # noqa: F401,F403
from .oracle import Config, Oracle, lib, run_workload, full_overflow, _p  # noqa: F401
