"""BJ configs[0]: B=2 fused shared MLPs (Conv1d k=1 3->64->64, BN, ReLU, MSE),
one fwd+bwd+per-model Adam step through the C ABI vs the per-model oracle.
EVERY gradient tensor is gated normwise: fp32 at 1e-4; bf16 at
max(2e-2, 2 x the AMP witness), where the witness is the error that bf16
rounding at the stored tensors alone causes in fp64 arithmetic
(tools/cfg1_conditioning.py: c1.W 4.9e-2, c2.W 2.9e-2 -- above 2e-2 for any
bf16 implementation)."""
import numpy as np
import pytest
import torch

import synth
from oracle import models as OM
from tests._cmp import TOL, relerr

import importlib.util
import os
_spec = importlib.util.spec_from_file_location(
    "cfg1_cond", os.path.join(os.path.dirname(__file__), "..", "tools", "cfg1_conditioning.py"))

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _init():
    import paper_2102_02344_b200.hfta as H
    H.hfta_init(0)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_cfg1_step(dtype):
    from paper_2102_02344_b200.mlp import FusedMLP
    B = 2
    specs = [(n, s) for n, s, _ in synth.param_specs("mlp_cfg1")]
    Ps = [synth.init_params("mlp_cfg1", 1000 + b) for b in range(B)]
    hp = synth.hparams_cfg1()
    x, T = synth.mlp_cfg1_batch(0)
    net = FusedMLP(B, specs, Ps, hp, rows=x.shape[0], dtype=dtype)
    loss = net.step(torch.tensor(x, dtype=torch.float32, device="cuda"),
                    torch.tensor(T, dtype=torch.float32, device="cuda")).cpu().numpy()
    res, ref, Lf = OM.fused_step_oracle("mlp_cfg1", Ps, [{}] * B, [{}] * B, (x, T), 1, hp)
    tol = TOL[dtype]
    witness = [None] * B
    if dtype == "bf16":
        import sys
        sys.argv = ["cfg1_conditioning"]
        w = _load_witness()
        witness = [w.run(Ps[b], x, T, True) for b in range(B)]
        exact = [w.run(Ps[b], x, T, False) for b in range(B)]
    for b in range(B):
        assert abs(loss[b] - ref[b]) <= tol * abs(ref[b])
        G = net.grads(b)
        gmax = max(np.linalg.norm(v) for v in res[b]["grads"].values())
        for n, r in res[b]["grads"].items():
            if n in ("c1.b", "c2.b"):             # BN-absorbed: identically zero
                assert np.linalg.norm(G[n]) == 0.0 and np.linalg.norm(r) < 1e-9 * gmax
                continue
            t_n = tol
            if witness[b] is not None:
                t_n = max(tol, 2 * relerr(witness[b][n], exact[b][n]))
            assert relerr(G[n], r) <= t_n, (b, n, relerr(G[n], r), t_n)
        m = net.arena.host_tensor("m", "c2.W")[b]        # m = (1 - beta1) g at t = 1: same gate as g
        t_m = tol if witness[b] is None else max(tol, 2 * relerr(witness[b]["c2.W"], exact[b]["c2.W"]))
        assert relerr(m, res[b]["opt"]["c2.W"][0]) <= t_m
        lr = hp["lr"][b]
        pb = net.params(b)
        for n in res[b]["params"]:
            assert np.max(np.abs(pb[n] - res[b]["params"][n])) <= 2 * lr * (1 + 1e-3) + 1e-7, n
        for name in ("bn1", "bn2"):
            assert relerr(net.running[name][0][b].cpu().numpy(), res[b]["stats"][name + ".rm"]) <= tol
            assert relerr(net.running[name][1][b].cpu().numpy(), res[b]["stats"][name + ".rv"]) <= tol


def _load_witness():
    """tools/cfg1_conditioning.py without running its report (functions only)."""
    import types
    src = open(_spec.origin).read()
    mod = types.ModuleType("cfg1_cond")
    exec(compile(src, _spec.origin, "exec"), mod.__dict__)
    return mod
