"""Seeded synthetic input generators shared by oracle tests, CUDA parity tests and bench.py."""
from .configs import CONFIG_NAMES, Workload, chain, grid, make, multi_agent, random_stable, rank_grid

__all__ = ["CONFIG_NAMES", "Workload", "chain", "grid", "make", "multi_agent", "random_stable", "rank_grid"]
