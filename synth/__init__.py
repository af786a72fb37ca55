"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic: it only produces the raw inputs
(point clouds, probe vectors) that the paper's workloads are defined on
("uniform 3D distribution of points in a cube", L435-439 volume IE points,
BASELINE.json configs).  The random matrix Omega that Algorithm 1 draws (PAPER.md L203,
"batchedRand") is NOT produced here: the oracle (oracle/rng.py) and the CUDA path
(csrc/rand.cu) each implement the same counter-based Philox4x32-10 generator.
"""
from .inputs import uniform_points, grid_points, probe_vectors, lowrank_factor, workload, WORKLOADS  # noqa: F401
