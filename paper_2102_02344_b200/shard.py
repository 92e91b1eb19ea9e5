"""Model-array sharding across GPUs.

The fused array of B_total models splits into disjoint contiguous blocks, one
per rank (the paper: fusion "can be performed for both single-accelerator and
distributed training"; models are independent, App. C Eq. 2:
the cross-model gradient is zero).  No collective is on the step's
data path; the only communication is one all-gather of the per-model losses
(C1), padded with a NaN sentinel when B_total is not a multiple of the world
size.  Works with any torch.distributed backend (nccl on GPUs, gloo in the CPU
tests).
"""
import math

import torch


def model_range(rank, world, B_total):
    """Contiguous block [lo, hi) of global model indices owned by `rank`."""
    per = math.ceil(B_total / world)
    lo = min(rank * per, B_total)
    return lo, min(lo + per, B_total)


def slice_hparams(hp, lo, hi):
    return {k: v[lo:hi] for k, v in hp.items()}


def gather_losses(loss_local, B_total, world, group=None):
    """All-gather per-model losses into global model order ([B_total], rank-major)."""
    import torch.distributed as dist
    per = math.ceil(B_total / world)
    buf = torch.full((per,), float("nan"), dtype=torch.float32, device=loss_local.device)
    buf[:loss_local.numel()] = loss_local.reshape(-1)
    out = torch.empty(per * world, dtype=torch.float32, device=loss_local.device)
    if world > 1:
        dist.all_gather_into_tensor(out, buf, group=group)
    else:
        out.copy_(buf)
    return out[:B_total]
