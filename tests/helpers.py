"""Shared test helpers (comparison metrics; no k-means arithmetic)."""
import numpy as np


def centroid_rel_err(Cg, Co):
    """Per-centroid ||dC||_2 / max(||C_c||_2, RMS_c' ||C_c'||_2) (SURVEY §8(c) parity protocol)."""
    Cg = np.asarray(Cg, float)
    Co = np.asarray(Co, float)
    norms = np.linalg.norm(Co, axis=1)
    rms = np.sqrt(np.mean(norms ** 2))
    den = np.maximum(norms, rms)
    den[den == 0] = 1.0
    return np.linalg.norm(Cg - Co, axis=1) / den


def near_tie_mask(d1, d2, rel=1e-5):
    """Points whose fp64 best/second-best squared-distance gap is < rel * d2 (BASELINE tier)."""
    return (d2 - d1) < rel * d2
