"""Outer optimizers of the DiLoCo loops on the GPU (algos.py:75-105).

The step on either side of the all-reduce: the
pseudo-gradient ``delta = global - local`` (algos.py:236, :334) and the
outer update, with the reference's NumPy rounding sequence kept exactly
(no fused multiply-add), so parameters stay bit-identical to a CPU peer.
"""

from __future__ import annotations

import torch

from ._native import check, lib
from .collective import UsageError


def _f32(t: torch.Tensor, what: str, like: torch.Tensor | None = None) -> None:
    """Checked before any launch (a host, short or other-device tensor is a
    UsageError, never a device fault); `like`: same size and device."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
        raise UsageError(f"{what} must be a contiguous float32 CUDA tensor")
    if like is not None and (t.numel() != like.numel() or t.device != like.device):
        raise UsageError(f"{what} must match {tuple(like.shape)} on {like.device}")


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def pseudo_gradient(global_params: torch.Tensor, local_params: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """delta = global - local (np.subtract, algos.py:334)."""
    _f32(global_params, "global_params")
    _f32(local_params, "local_params", global_params)
    out = torch.empty_like(global_params) if out is None else out
    _f32(out, "out", global_params)
    with torch.cuda.device(out.device):
        check(lib().pcclb_pseudo_gradient_f32(out.data_ptr(), global_params.data_ptr(), local_params.data_ptr(),
                                              out.numel(), _stream()), "pseudo_gradient")
    return out


class PlainSGD:
    """algos.py:75-87: params -= lr * grad."""

    def __init__(self, lr: float = 2.0**-6):
        self.lr = float(torch.tensor(lr, dtype=torch.float32))

    def step(self, params: torch.Tensor, grad: torch.Tensor) -> None:
        _f32(params, "params")
        _f32(grad, "grad", params)
        with torch.cuda.device(params.device):
            check(lib().pcclb_outer_sgd_f32(params.data_ptr(), grad.data_ptr(), params.numel(), self.lr, _stream()),
                  "outer_sgd")


class NesterovOuter:
    """algos.py:90-105: v = v*mu; v += delta; params -= lr * (delta + mu*v)."""

    def __init__(self, dim: int, lr: float = 0.5, momentum: float = 0.9, device=None):
        self.lr = float(torch.tensor(lr, dtype=torch.float32))
        self.momentum = float(torch.tensor(momentum, dtype=torch.float32))
        self.velocity = torch.zeros(dim, dtype=torch.float32, device=device or "cuda")

    def step(self, params: torch.Tensor, delta: torch.Tensor) -> None:
        _f32(params, "params", self.velocity)
        _f32(delta, "delta", self.velocity)
        with torch.cuda.device(params.device):
            check(lib().pcclb_outer_nesterov_f32(params.data_ptr(), delta.data_ptr(), self.velocity.data_ptr(),
                                                 params.numel(), self.lr, self.momentum, _stream()), "outer_nesterov")

    def state_entries(self, prefix: str = ""):
        from .sharedstate import DType, SharedStateEntry

        return [SharedStateEntry(prefix + "outer_momentum", DType.F32, self.velocity)]
