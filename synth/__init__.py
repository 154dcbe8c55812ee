"""Seeded synthetic inputs shared by the oracle tests, smoke() and bench.py.

This package holds NO arithmetic of the method (no dequant, norm, attention,
GEMM, acceptance).  It only turns (seed, tensor id, element index) into the
canonical input tensors described in DESIGN.md "Input recipe".  The CUDA side
re-implements the same counter-based generator (csrc/synth.cu) so that a 70B
model can be materialised on the device; tests check both produce the same
bytes on small shapes.
"""
from .generators import *  # noqa: F401,F403
