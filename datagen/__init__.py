"""Seeded synthetic input generators shared by the oracle, the tests and bench.py.

This package holds NO arithmetic of the method (no hashing, no tables, no
aggregation): it only draws the matrices A~ (train), A (test/bench) and B with
the shapes and value distributions BASELINE.json names, standing in for the
paper's CIFAR / Caltech101 workloads,
which are not available here.
"""
from .synth import (  # noqa: F401
    CONFIGS,
    ConfigSpec,
    get_config,
    make_config_data,
    relu_lowrank_torch,
)
