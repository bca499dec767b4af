"""Nominal forecast container consumed by the closed loop (``forecast.py:18-50``
of the reference: ``ForecastSeries`` with the same fields and checks). The
forecasting methods themselves are data preparation outside the hot path."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class ForecastSeries:
    """H_p-step nominal forecasts: demands (m^3/s) and prices per flow."""

    d_hat: np.ndarray      # (horizon, n_demand)
    alpha_hat: np.ndarray  # (horizon, n_price)

    def __post_init__(self) -> None:
        self.d_hat = np.atleast_2d(np.asarray(self.d_hat, float))
        self.alpha_hat = np.atleast_2d(np.asarray(self.alpha_hat, float))
        if self.d_hat.shape[0] != self.alpha_hat.shape[0]:
            raise ValueError(f"demand and price forecasts disagree on horizon: "
                             f"{self.d_hat.shape[0]} vs {self.alpha_hat.shape[0]}")
        if self.d_hat.size == 0:
            raise ValueError("dHat must not be empty")
        if self.alpha_hat.size == 0:
            raise ValueError("alphaHat must not be empty")
        if np.any(self.d_hat < 0):
            raise ValueError("dHat must be nonnegative")

    @property
    def horizon(self) -> int:
        return self.d_hat.shape[0]

    @property
    def n_demand(self) -> int:
        return self.d_hat.shape[1]

    @property
    def n_price(self) -> int:
        return self.alpha_hat.shape[1]
