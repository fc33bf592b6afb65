"""Randomized range finder / low-rank SVD configuration and the randomized
streaming update (reference linalg.py:33-62, 126-162)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class RandomSketchConfig:
    """Parameters of the randomized range finder (linalg.py:33-62).

    target_rank      rank of the approximation that is kept
    oversampling     extra sketch columns beyond target_rank
    power_iterations subspace iteration count (0 = plain sketch)
    seed             Philox seed for the Gaussian test matrix
    """

    target_rank: int
    oversampling: int = 10
    power_iterations: int = 1
    seed: int = 0

    def __post_init__(self):
        if self.target_rank < 1:
            raise ValueError(f"target_rank must be >= 1, got {self.target_rank}")
        if self.oversampling < 0:
            raise ValueError(f"oversampling must be >= 0, got {self.oversampling}")
        if self.power_iterations < 0:
            raise ValueError(f"power_iterations must be >= 0, got {self.power_iterations}")
        if self.seed < 0:
            raise ValueError(f"seed must be >= 0, got {self.seed}")

    @property
    def sketch_width(self):
        return self.target_rank + self.oversampling


def gaussian_test_matrix(n_cols, config):
    """The reference's Omega, drawn on the host exactly as linalg.py:141-142
    (Philox(seed).standard_normal((n_cols, width))) and uploaded by callers, so
    both implementations see identical bytes."""
    rng = np.random.Generator(np.random.Philox(config.seed))
    return rng.standard_normal((n_cols, config.sketch_width))


def randomized_update(U, sigma, A, sketch, ff, device):  # pragma: no cover - replaced below
    raise NotImplementedError("randomized update is not built yet")
