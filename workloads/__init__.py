"""Seeded synthetic workloads shared by the oracle tests, the GPU tests and bench.py.

This package holds ONLY input generation (grid coordinates, field values, seeded
random parameters).  It contains none of the method's arithmetic: no volumes,
areas, fluxes, stencils, diffusivity laws, RKL2 coefficients or solver steps.
"""
from .inputs import *  # noqa: F401,F403
