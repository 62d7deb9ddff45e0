"""Seeded synthetic inputs shared by the oracle, the tests and the bench.

This package holds NO arithmetic of the method (no bases, no quadrature, no
operators).  It only produces input arrays: vertex coordinates of structured
meshes, per-element coefficients and random vectors, all from a counter-based
generator so that every consumer sees identical data.
"""
from .gen import (  # noqa: F401
    counter_uniform,
    random_vector,
    cartesian_vertices,
    perturbed_vertices,
    graded_two_material,
    Problem,
    make_config,
    CONFIG_NAMES,
)
