"""Seeded synthetic input generators shared by the oracle-side tests and the CUDA path.

This package holds NONE of the method's arithmetic: it only draws random tensors
(torch generators, CPU or CUDA) shaped like the paper's workloads.
"""
from .generators import *  # noqa: F401,F403
