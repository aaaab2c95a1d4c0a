"""Seeded test fields: the reference tests' fixtures restated (proj/tests/*.cpp)."""
import numpy as np


def ramp(dims):
    """x + 2y + 4z (test_gradient.cpp:14-22, volume.cpp:122-130)."""
    nx, ny, nz = dims
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return (x + 2 * y + 4 * z).astype(np.float64).ravel()


def quantized(dims, levels, seed):
    """Tie-heavy field (test_grid.cpp:132-137 uses r() % 3)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, levels, size=int(np.prod(dims))).astype(np.float64)


def random_field(ref, dims, seed):
    """oracle::random_field (oracles.hpp:43-54) == generate_field(white_noise) (volume.cpp:151-156)."""
    return ref.generate("white-noise", dims, seed)
