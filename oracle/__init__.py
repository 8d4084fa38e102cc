"""CPU parity oracle for the Hadamard GA inner loop -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package.  The product package
``paper_2208_14961_b200`` never imports it; its CUDA path fails loudly when
its own extension is missing instead of falling back here.

See oracle/hga_oracle.c for the reference file:line each function restates.
"""

from .oracle import *  # noqa: F401,F403
from .oracle import __all__  # noqa: F401
