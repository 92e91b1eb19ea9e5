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


class LossGather:
    """The per-model loss gather (C1) off the step's critical path (SURVEY
    8(e)): the compute stream copies loss[B_g] into one of two staging
    buffers and records an event; a side stream waits on it and all-gathers
    the staged copy while the compute stream runs the next step.  A staging
    buffer is reused only after the gather that read it has finished (event
    wait on the compute stream).  On CPU tensors (gloo tests) the gather is
    synchronous."""

    def __init__(self, B_total, world, device, group=None):
        import torch.distributed as dist  # noqa: F401  (the caller initialised the process group)
        self.B_total, self.world, self.group = B_total, world, group
        self.per = math.ceil(B_total / world)
        dev = torch.device(device)
        self.cuda = dev.type == "cuda"
        self.stage = [torch.full((self.per,), float("nan"), dtype=torch.float32, device=dev) for _ in range(2)]
        self.out = [torch.empty(self.per * world, dtype=torch.float32, device=dev) for _ in range(2)]
        self.i = 0
        if self.cuda:
            self.side = torch.cuda.Stream(device=dev)
            self.staged = [torch.cuda.Event() for _ in range(2)]
            self.done = [None, None]

    def launch(self, loss_local):
        """Enqueue the gather of this step's losses; returns the [B_total] output tensor
        (valid after `wait()` / on the side stream)."""
        import torch.distributed as dist
        j = self.i % 2
        self.i += 1
        cur = torch.cuda.current_stream() if self.cuda else None
        if self.cuda and self.done[j] is not None:
            cur.wait_event(self.done[j])              # the gather that read this buffer has finished
        self.stage[j][:loss_local.numel()].copy_(loss_local.reshape(-1))
        if not self.cuda:
            if self.world > 1:
                dist.all_gather_into_tensor(self.out[j], self.stage[j], group=self.group)
            else:
                self.out[j].copy_(self.stage[j])
            return self.out[j][:self.B_total]
        self.staged[j].record(cur)
        with torch.cuda.stream(self.side):
            self.side.wait_event(self.staged[j])
            if self.world > 1:
                dist.all_gather_into_tensor(self.out[j], self.stage[j], group=self.group)
            else:
                self.out[j].copy_(self.stage[j])
            ev = torch.cuda.Event()
            ev.record(self.side)
            self.done[j] = ev
        return self.out[j][:self.B_total]

    def wait(self):
        if self.cuda:
            torch.cuda.current_stream().wait_stream(self.side)
