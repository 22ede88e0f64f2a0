"""fp64 CPU oracle (TEST INFRASTRUCTURE ONLY -- see ztp_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package."""
from . import ztp_oracle  # noqa: F401
