"""Synthetic workload: layer shape tables and seeded input generators (no K-FAC arithmetic)."""
from . import shapes, inputs  # noqa: F401
