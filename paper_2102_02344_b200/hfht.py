"""HFHT: horizontally fused hyper-parameter tuning (App. E, Alg. 1 P:L1406-1429;
P:L949-985).

A tuning algorithm (random search or Hyperband) proposes a batch H of
hyper-parameter sets.  `partition_and_fuse` groups the sets that share the
values of every *infusible* hyper-parameter (batch size, feature transform,
architecture: they change operator types or shapes) into partitions
whose members differ only in *fusible* ones (learning rate, Adam betas,
weight decay, LR-decay factor and period); each partition is ONE
fused job of B models (a `FusedPointNet` array on one GPU here).
`Scheduler.schedule_and_run` runs the jobs -- on G GPUs it assigns the fused
arrays longest-first to the least-loaded device -- and `unfuse_and_reorder`
scatters the per-model results back into the order of H.  The algorithms only
ever see (H, R) pairs, so fusing changes the cost, never the result
(P:L923): the serial scheduler (one job per set) and the HFTA scheduler
return the same best set for a deterministic evaluator.

Host-side control logic only (no arithmetic of the training step): the fused
step itself is libhfta's.
"""
import math
from dataclasses import dataclass, field

import numpy as np


# ---------------------------------------------------------- search space ----

@dataclass(frozen=True)
class HP:
    """One hyper-parameter: continuous [lo, hi] (log-uniform if log) or a
    discrete set of values; fusible = may differ inside one fused job."""
    name: str
    fusible: bool
    lo: float = None
    hi: float = None
    values: tuple = None
    log: bool = False

    def sample(self, rng):
        if self.values is not None:
            return self.values[int(rng.integers(len(self.values)))]
        if self.log:
            return float(math.exp(rng.uniform(math.log(self.lo), math.log(self.hi))))
        return float(rng.uniform(self.lo, self.hi))

    def check(self, v, where=""):
        if self.values is not None:
            ok = v in self.values
        else:
            ok = self.lo <= v <= self.hi
        if not ok:
            raise ValueError("%s: %s = %r outside its domain" % (where, self.name, v))


def pointnet_space():
    """The PointNet classification tuning space of the paper's HFHT table
    (P:L968-985): six fusible and two infusible hyper-parameters."""
    return [HP("lr", True, 1e-4, 1e-2, log=True),
            HP("beta1", True, 0.001, 0.999),
            HP("beta2", True, 0.001, 0.999),
            HP("wd", True, 0.0, 0.5),
            HP("gamma", True, 0.1, 0.9),                      # LR decay factor (StepLR)
            HP("step_size", True, values=(5, 10, 20, 40)),    # LR decay period (epochs)
            HP("batch_size", False, values=(8, 16, 32)),
            HP("feature_transform", False, values=(True, False))]


def sample_sets(space, n, rng):
    return [{h.name: h.sample(rng) for h in space} for _ in range(n)]


# ------------------------------------------------------------ partitions ----

@dataclass
class Partition:
    key: tuple                    # the infusible values shared by every member
    members: list                 # [(original_index, set), ...] in proposal order

    @property
    def B(self):
        return len(self.members)


def partition_and_fuse(sets, space, max_B=None):
    """Alg. 1 partition_and_fuse: group by the tuple of infusible values
    (first-seen order), split groups larger than max_B into ceil(n / max_B)
    partitions preserving order.  Every set lands in exactly one partition."""
    infusible = [h.name for h in space if not h.fusible]
    for i, hs in enumerate(sets):
        for h in space:
            if h.name not in hs:
                raise ValueError("set %d: missing %s" % (i, h.name))
            h.check(hs[h.name], "set %d" % i)
    groups = {}
    for i, hs in enumerate(sets):
        groups.setdefault(tuple(hs[k] for k in infusible), []).append((i, hs))
    parts = []
    for key, mem in groups.items():
        step = len(mem) if not max_B else int(max_B)
        for j in range(0, len(mem), step):
            parts.append(Partition(key, mem[j:j + step]))
    return parts


def unfuse_and_reorder(results):
    """results: [(partition, per-member records)] -> records in original order.
    Raises on a missing or duplicated original index."""
    out = {}
    for part, recs in results:
        if len(recs) != part.B:
            raise ValueError("partition %r returned %d records for %d members" % (part.key, len(recs), part.B))
        for (i, _), r in zip(part.members, recs):
            if i in out:
                raise ValueError("original index %d returned twice" % i)
            out[i] = r
    n = len(out)
    if sorted(out) != list(range(n)):
        missing = sorted(set(range(max(out) + 1 if out else 0)) - set(out))
        raise ValueError("original indices missing: %s" % missing)
    return [out[i] for i in range(n)]


# -------------------------------------------------------------- schedule ----

@dataclass
class JobResult:
    metrics: list                 # per member, higher is better
    cost: float                   # device-seconds of the job


class Scheduler:
    """Runs one batch of proposals.  kind 'hfta': one fused job per partition
    (max_B models each); 'serial': one job per set.  Jobs are assigned
    longest-first to the least-loaded of `devices` (LPT), the model array of a
    job stays on one device (models are independent)."""

    def __init__(self, space, runner, kind="hfta", max_B=None, devices=1):
        assert kind in ("hfta", "serial")
        self.space, self.runner, self.kind, self.max_B, self.devices = space, runner, kind, max_B, devices
        self.total_cost = 0.0
        self.jobs = 0
        self.placements = []      # (device, partition key, B) per job, for inspection

    def run(self, sets, epochs):
        parts = partition_and_fuse(sets, self.space, 1 if self.kind == "serial" else self.max_B)
        est = [self.runner.estimate(p, epochs) for p in parts]
        load = [0.0] * self.devices
        order = sorted(range(len(parts)), key=lambda j: -est[j])
        dev_of = {}
        for j in order:
            d = min(range(self.devices), key=lambda k: load[k])
            dev_of[j] = d
            load[d] += est[j]
        results = []
        for j, p in enumerate(parts):
            r = self.runner.run(p, epochs, device=dev_of[j])
            self.total_cost += r.cost
            self.jobs += 1
            self.placements.append((dev_of[j], p.key, p.B))
            results.append((p, r.metrics))
        return unfuse_and_reorder(results)


# ------------------------------------------------------------- algorithms ----

def _argmax_first(metrics):
    best = 0
    for i, m in enumerate(metrics):
        if m > metrics[best]:
            best = i
    return best


def random_search(space, total_sets, epochs, scheduler, rng):
    """Random search: total_sets sets drawn from the space, each
    trained `epochs` epochs; best = argmax (ties: lowest index)."""
    H = sample_sets(space, total_sets, rng)
    R = scheduler.run(H, epochs)
    b = _argmax_first(R)
    return dict(best=H[b], best_metric=R[b], history=[(h, r, epochs) for h, r in zip(H, R)])


def hyperband_brackets(R, eta, skip_last=0):
    """The Hyperband schedule (Li et al.; P:L953-960 settings R, eta, skip):
    for s = s_max .. 0: n = ceil((s_max + 1) / (s + 1) * eta^s) sets, rounds
    i = 0 .. s with n_i = floor(n eta^-i) sets trained r_i = R eta^(i - s)
    epochs; the last `skip_last` rounds of every bracket are omitted (a bracket
    keeps at least its first round)."""
    if R < 1 or eta < 2 or skip_last < 0:
        raise ValueError("hyperband: need R >= 1, eta >= 2, skip_last >= 0")
    s_max = 0
    while eta ** (s_max + 1) <= R + 1e-9:
        s_max += 1
    out = []
    for s in range(s_max, -1, -1):
        n = int(math.ceil((s_max + 1) / (s + 1) * eta ** s))
        rounds = []
        for i in range(s + 1):
            n_i = int(math.floor(n * eta ** (-i)))
            r_i = R * eta ** (i - s)
            rounds.append((n_i, r_i))
        keep = max(1, len(rounds) - skip_last)
        out.append((s, rounds[:keep]))
    return out


def hyperband(space, R, eta, skip_last, scheduler, rng):
    """Successive halving per bracket: every round's survivors (top n_{i+1}
    by metric, ties by proposal order) are re-trained with the next budget."""
    history, best, best_metric = [], None, -math.inf
    for s, rounds in hyperband_brackets(R, eta, skip_last):
        T = sample_sets(space, rounds[0][0], rng)
        for i, (n_i, r_i) in enumerate(rounds):
            T = T[:n_i]
            epochs = max(1, int(round(r_i)))
            L = scheduler.run(T, epochs)
            history += [(h, m, epochs) for h, m in zip(T, L)]
            for h, m in zip(T, L):
                if m > best_metric:
                    best, best_metric = h, m
            if i + 1 < len(rounds):
                order = sorted(range(len(T)), key=lambda j: (-L[j], j))
                T = [T[j] for j in order[:rounds[i + 1][0]]]
    return dict(best=best, best_metric=best_metric, history=history)


def tune(algorithm, scheduler, space, rng, **kw):
    """Alg. 1: propose -> partition_and_fuse -> schedule_and_run ->
    unfuse_and_reorder -> select_best -> update (the algorithms above run the
    loop internally); returns the best set, metric, history and the device
    cost the scheduler accrued."""
    if algorithm == "random_search":
        res = random_search(space, kw["total_sets"], kw["epochs"], scheduler, rng)
    elif algorithm == "hyperband":
        res = hyperband(space, kw["R"], kw["eta"], kw.get("skip_last", 0), scheduler, rng)
    else:
        raise ValueError(algorithm)
    res["cost"] = scheduler.total_cost
    res["jobs"] = scheduler.jobs
    return res


# ------------------------------------------------------ the GPU runner ----

class PointNetRunner:
    """Trains one partition as ONE fused PointNet-cls array (FusedPointNet)
    on synthetic ModelNet-shaped data: per member its own lr, betas, weight
    decay and StepLR(gamma, step_size); the partition's infusible batch size
    is the fused job's N.  An "epoch" is `steps_per_epoch` fused steps.
    metric = -(final training loss) of each model (higher is better); cost =
    the job's device time (CUDA events) in seconds.  The infusible feature-
    transform switch selects the STNkd variant (FusedPointNet feature_transform,
    P:L981)."""

    def __init__(self, L=256, k=40, steps_per_epoch=2, dtype="bf16", seed=0, device_ids=None):
        self.L, self.k, self.spe, self.dtype, self.seed = L, k, steps_per_epoch, dtype, seed
        self.device_ids = device_ids

    def estimate(self, part, epochs):
        return float(part.key[0]) * self.L * epochs * (1.0 + 0.02 * part.B)   # ~ fused step cost

    def run(self, part, epochs, device=0):
        import torch
        import synth
        from .pointnet import FusedPointNet
        from . import hfta as H
        dev = "cuda:%d" % (self.device_ids[device] if self.device_ids else 0)
        N = int(part.key[0])
        ft = bool(part.key[1]) if len(part.key) > 1 else False
        sets = [m[1] for m in part.members]
        B = len(sets)
        hp = {k: np.array([s_[k] for s_ in sets], dtype=np.float64) for k in ("lr", "beta1", "beta2", "wd")}
        hp["eps"] = np.full(B, 1e-8)
        specs = [(n, s) for n, s, _ in synth.param_specs("pointnet_cls", self.k, None, ft)]
        Ps = [synth.init_params("pointnet_cls", 1000 + m[0], self.k, None, ft) for m in part.members]
        with torch.cuda.device(dev):
            # each set's dropout masks keyed by its own id: results independent of the partitioning
            net = FusedPointNet(B, specs, Ps, hp, task="cls", dtype=self.dtype, N=N, L=self.L, k=self.k, device=dev,
                                feature_transform=ft, model_ids=[m[0] for m in part.members])
            gam = torch.tensor([s_["gamma"] for s_ in sets], dtype=torch.float32, device=dev)
            per = torch.tensor([s_["step_size"] for s_ in sets], dtype=torch.int32, device=dev)
            lr0 = net.hv.t["lr"].clone()
            x, y = synth.points_cls(self.seed, N=N, L=self.L, k=self.k)
            xd = torch.tensor(x.reshape(-1, 3), dtype=torch.float32, device=dev)
            yd = torch.tensor(y, dtype=torch.int32, device=dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            loss = None
            for ep in range(epochs):
                H.hfta_steplr(B, H.ptr(lr0), H.ptr(gam), H.ptr(per), ep, H.ptr(net.hv.t["lr"]),
                              H.stream_ptr(None))
                for _ in range(self.spe):
                    loss = net.step(xd, yd)
            e1.record()
            torch.cuda.synchronize()
            cost = e0.elapsed_time(e1) / 1e3
            metrics = [-float(v) for v in loss.cpu().numpy()]
        return JobResult(metrics, cost)
