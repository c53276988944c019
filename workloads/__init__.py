"""Seeded synthetic input generators shared by tests, smoke() and bench.py.

This package holds NONE of the method's arithmetic (no quantisation, prefix
sum, fixed point, cells, trees or sampling).  It only produces inputs: float32
weight vectors p shaped like the paper's workloads and u32 fixed-point xi
sequences (xi/2^32, reading R11 in DESIGN.md).  Both the oracle and the CUDA
path consume exactly these arrays.  Recipes are stated in DESIGN.md section 4.
"""
from .generators import *  # noqa: F401,F403
