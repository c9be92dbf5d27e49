"""Squared-exponential hyperparameters (taskgp covariance.py:26-62).

The tile assembly itself (covariance.py:65-230) lives in the CUDA library
(``csrc/sek.cu``); this module keeps the parameter container and its
validation so user code written against the reference carries over.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import InvalidConfig


@dataclass(frozen=True)
class KernelParams:
    """SEK hyperparameters: lengthscale l, vertical scale nu, noise variance.

    Validation matches covariance.py:50-62 (l > 0, nu > 0, noise >= 0,
    three trainable flags ordered (lengthscale, vertical_scale, noise)).
    """

    lengthscale: float = 1.0
    vertical_scale: float = 1.0
    noise_variance: float = 0.1
    trainable: tuple[bool, bool, bool] = (True, True, True)

    def __post_init__(self) -> None:
        if not self.lengthscale > 0:
            raise InvalidConfig(f"lengthscale must be positive, got {self.lengthscale}")
        if not self.vertical_scale > 0:
            raise InvalidConfig(f"vertical_scale must be positive, got {self.vertical_scale}")
        if self.noise_variance < 0:
            raise InvalidConfig(
                f"noise_variance must be non-negative, got {self.noise_variance}"
            )
        if len(self.trainable) != 3:
            raise InvalidConfig("trainable must hold exactly three flags")
