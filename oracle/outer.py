"""NumPy restatement of the reference outer optimizers -- TEST INFRASTRUCTURE
ONLY (see oracle/__init__.py). Follows /root/reference/pkg/src/churncomm/
algos.py:75-105 (PlainSGD, NesterovOuter) and :334 (pseudo-gradient)."""

from __future__ import annotations

import numpy as np


def pseudo_gradient(global_params: np.ndarray, local_params: np.ndarray) -> np.ndarray:
    out = np.empty_like(global_params)
    np.subtract(global_params, local_params, out=out)  # algos.py:334
    return out


def sgd_step(params: np.ndarray, grad: np.ndarray, lr: float) -> None:
    params -= np.float32(lr) * grad  # algos.py:83-84


def nesterov_step(params: np.ndarray, delta: np.ndarray, velocity: np.ndarray, lr: float, momentum: float) -> None:
    lr, mu = np.float32(lr), np.float32(momentum)  # algos.py:93-95
    np.multiply(velocity, mu, out=velocity)  # :98
    velocity += delta  # :99
    params -= lr * (delta + mu * velocity)  # :100
