"""SPO+ layer: the differentiable LP layer of PAPER.md §2.2
(Eq. spo+ loss P:76-78, Eq. spo+ gradient P:80-82) in the form of the listing of
P:198-215 -- a custom autograd function whose forward solves the batch of inner
LPs min_{x in S} (2c^ - c)'x and whose backward returns 2 (x*(c) - x*(2c^ - c)).

Thin binding: the inner solves, the loss and the subgradient are computed by
lp_spo_plus (CUDA); torch only averages over the batch and scales by the
incoming gradient."""
from __future__ import annotations

import torch

from .lp import BatchSolver


class SPOPlus(torch.autograd.Function):
    """loss = mean_b SPO+(c^_b, c_b); d loss / d c^ = 2 (x*(c) - x*(2c^ - c)) / B."""

    @staticmethod
    def forward(ctx, pred_cost, true_cost, true_sol, true_obj, solver: BatchSolver, warm: bool, opts: dict):
        loss, grad, res = solver.spo_plus(pred_cost.detach(), true_cost, true_sol, true_obj, warm=warm, **opts)
        ctx.save_for_backward(grad)
        ctx.results = res
        return loss.mean()

    @staticmethod
    def backward(ctx, g):
        (grad,) = ctx.saved_tensors
        return grad * (g / grad.shape[0]), None, None, None, None, None, None


def spo_plus_loss(pred_cost, true_cost, true_sol, true_obj, solver: BatchSolver, warm: bool = False, **opts):
    """Batch-mean SPO+ loss with the subgradient of Eq. (spo+ gradient) as its backward."""
    return SPOPlus.apply(pred_cost, true_cost, true_sol, true_obj, solver, warm, opts)
