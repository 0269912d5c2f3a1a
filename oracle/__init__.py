"""fp64 CPU oracle (TEST INFRASTRUCTURE ONLY -- see cks_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.
"""
from .cks_oracle import *  # noqa: F401,F403
from . import cks_oracle  # noqa: F401
from . import cks_oracle3d  # noqa: F401  (3-D operators)
