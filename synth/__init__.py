"""Seeded synthetic inputs for the k-means hot path (shared by oracle tests and the CUDA path).

This package holds NO k-means arithmetic: only the data recipe of SURVEY.md §8(d)
("Synthetic inputs") and the Forgy index draw.  Both the CPU oracle (``oracle/``) and
the product path (``paper_1902_09527_b200``) consume its outputs; neither imports the other.
"""
from .generate import CONFIGS, ConfigSpec, make_config, make_points, forgy_indices, sha256_points  # noqa: F401
