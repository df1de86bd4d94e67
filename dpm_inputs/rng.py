"""Seeded random draws (numpy PCG64 via default_rng).  No method arithmetic here.

The values are returned as flat arrays; each side (oracle / CUDA path) places them
on its OWN point list (M+ for cfg1, the band for cfg4), in ascending flat index
order (R7, R21, R22).
"""
import numpy as np


def uniform_values(seed: int, shape) -> np.ndarray:
    """i.i.d. U(-1, 1) fp64 values from ``np.random.default_rng(seed)``."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=shape)


def cfg1_particular_values(n_mplus: int) -> np.ndarray:
    """R22: U(-1,1) from seed 0, one value per M+ point (ascending flat index)."""
    return uniform_values(0, n_mplus)


def cfg4_band_values(batch: int, n_band: int, seed: int = 0) -> np.ndarray:
    """R21: ``default_rng(0).uniform(-1, 1, size=(batch, n_band))``; row b -> RHS b,
    column -> band point in ascending flat order."""
    return uniform_values(seed, (batch, n_band))


def random_boxes(seed: int, batch: int, n: int) -> np.ndarray:
    """Dense U(-1,1) boxes [batch][n][n][n] for AP-solver parity tests."""
    return uniform_values(seed, (batch, n, n, n))
