"""Seeded synthetic workload generators (shared by oracle and CUDA path; no
arithmetic of the method lives here)."""
from . import inputs, configs  # noqa: F401
