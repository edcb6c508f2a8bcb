"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no tableau recursion, no DG
operators, no mesh connectivity): only the problem definitions of the five
BASELINE.json configs -- level maps on the finest grid, analytic initial
conditions u0(x, y), time steps and step counts -- generated from a seed with
numpy's PCG64.  Both `oracle/` and `paper_2403_05144_b200/` consume these
arrays/callables; neither imports the other.  Recipes: DESIGN.md §3.
"""
from .configs import Workload, make, CONFIG_NAMES, leafify, balance  # noqa: F401
