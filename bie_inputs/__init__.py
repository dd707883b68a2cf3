"""Seeded synthetic inputs for the five BASELINE.json configurations.

This module is shared by the oracle-side tests, the GPU tests and bench.py.
It holds NONE of the method's arithmetic (no quadrature, no kernels, no
harmonics): only geometry placement (random sequential addition), density
draws and target draws, following the recipes of SURVEY.md §8(d) "Inputs".

Seeds: cfg 1 densities use seed 0 (BASELINE.json configs[0]); otherwise cfg c
uses 1000c+1 (geometry), 1000c+2 (densities), 1000c+3 (oracle subsets),
1000c+4 (off-surface targets).
"""
from .gen import (CONFIGS, make_config, rsa_uniform, rsa_polydisperse,
                  offsurface_targets, rigid_field, node_count)

__all__ = ["CONFIGS", "make_config", "rsa_uniform", "rsa_polydisperse",
           "offsurface_targets", "rigid_field", "node_count"]
