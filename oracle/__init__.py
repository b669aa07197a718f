"""CPU oracle for the NoScope cascade hot path — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  See noscope_oracle.py."""
from .noscope_oracle import *  # noqa: F401,F403
from . import noscope_oracle  # noqa: F401
