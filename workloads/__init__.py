"""Seeded, synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This package builds *inputs only*: forest leaf lists (levels + tree ids in Morton order),
tree connectivities, physical boundary kinds, initial conditions and (for the cubed sphere)
the capacity/edge-velocity aux arrays.  It contains none of the method's arithmetic (no ghost
fill, no Riemann solve, no update), so neither the oracle nor the CUDA path can hide a mistake
in here.  See DESIGN.md "Input recipe" for the configs C1-C5 it produces.
"""
from .forests import (Connectivity, Forest, periodic_unit_square, walled_unit_square,
                      brick, forest_uniform, forest_refined)
from .configs import Workload, make_config, CONFIG_NAMES

__all__ = ["Connectivity", "Forest", "periodic_unit_square", "walled_unit_square", "brick",
           "forest_uniform", "forest_refined", "Workload", "make_config", "CONFIG_NAMES"]
