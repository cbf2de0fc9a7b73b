"""Seeded synthetic workloads shared by the CUDA path's tests/bench and the oracle tests.

Holds only parameters and signal generators -- none of the method's arithmetic.
"""
from .configs import CONFIGS, SlicqConfig, plan_args  # noqa: F401
