"""Seeded synthetic input generators shared by oracle tests, CUDA parity tests and bench.py."""
from .configs import CONFIG_NAMES, Workload, chain, grid, make, multi_agent, random_stable

__all__ = ["CONFIG_NAMES", "Workload", "chain", "grid", "make", "multi_agent", "random_stable"]
