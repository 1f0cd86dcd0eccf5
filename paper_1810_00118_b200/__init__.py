"""B200-native cascadic multilevel primal-dual W1 solver (arXiv 1810.00118).

Drop-in for the reference's w1mg:: solver entry points: host code (the C++
shim in csrc/host and the Python mirror in w1mg.py) calls hand-written
sm_100a CUDA kernels through the C-ABI declared in include/w1mg_cuda.h.
Importing is cheap; the shared library is loaded on first use and its
absence is an error (no CPU fallback).  See DESIGN.md.
"""
from . import instances, w1mg  # noqa: F401
from ._lib import build, lib  # noqa: F401

__all__ = ["build", "lib", "instances", "w1mg"]
