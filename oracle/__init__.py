"""CPU oracle for the mpkrylov hot path -- TEST INFRASTRUCTURE ONLY.

A C restatement of the reference (/root/reference/pkg/src/mpkrylov) built
from oracle/mpk_oracle.c into oracle/liborc.so.  Only tests/, the
``__graft_entry__.smoke()`` check and bench.py's CPU-baseline leg may use it;
the product package never imports it.  Pinned against reference-generated
golden vectors in tests/golden (tests/test_oracle_golden.py).
"""

from .oracle import *  # noqa: F401,F403
from .oracle import __all__  # noqa: F401
