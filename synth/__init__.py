"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no window, no B_opt, no FFT, no
spread/gather): only the node distributions the paper's experiments use and
seeded random right-hand sides.  Both sides of every parity test draw their
inputs from here; neither side's arithmetic lives here.

Node sets (PAPER.md = /root/reference/PAPER.md, cited as P:<line>):
  * jittered equispaced nodes, eq. (jittered_nodes)
  * Chebyshev nodes, eq. (tschebyscheff_nodes)
  * i.i.d. uniform nodes (BASELINE config 2), sorted
  * polar grid (BASELINE config 4; reading A12)
Random data follows DESIGN.md readings A13/A14: numpy PCG64 default_rng(seed),
per RHS a Re block then an Im block.
"""
from .nodes import jittered, chebyshev, iid_sorted, polar, equispaced, wrap_half_open
from .data import (uniform_complex, normal_complex, blob_image, CONFIGS, config,
                   make_nodes, make_rhs)

__all__ = ["jittered", "chebyshev", "iid_sorted", "polar", "equispaced", "wrap_half_open",
           "uniform_complex", "normal_complex", "blob_image", "CONFIGS", "config",
           "make_nodes", "make_rhs"]
