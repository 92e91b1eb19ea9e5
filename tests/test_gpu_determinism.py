"""Bitwise reproducibility (SURVEY §4 test plan (v); hfta.h "Determinism"):
the same fused step run twice from the same state gives identical bits."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _init():
    import paper_2102_02344_b200.hfta as H
    H.hfta_init(0)


def _dcgan_once(dtype):
    from paper_2102_02344_b200.dcgan import FusedDCGAN
    B, N = 2, 4
    gs = [(n, s) for n, s, _ in synth.param_specs("dcgan_g")]
    ds = [(n, s) for n, s, _ in synth.param_specs("dcgan_d")]
    PG = [synth.init_params("dcgan_g", 1000 + b) for b in range(B)]
    PD = [synth.init_params("dcgan_d", 2000 + b) for b in range(B)]
    net = FusedDCGAN(B, gs, ds, PG, PD, synth.hparams_dcgan(3, B), N=N, dtype=dtype)
    real = synth.images(0, N=N)
    zs = np.stack([synth.noise(0, b, 1, N=N) for b in range(B)])
    net.set_inputs(torch.tensor(real.transpose(0, 2, 3, 1), dtype=torch.float32, device="cuda"),
                   torch.tensor(zs, dtype=torch.float32, device="cuda"))
    net.step()
    torch.cuda.synchronize()
    return (net.G.arena.g.cpu().numpy(), net.D.arena.g.cpu().numpy(), net.G.arena.p.cpu().numpy(),
            net.fake.float().cpu().numpy())


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_dcgan_bitwise(dtype):
    a, b = _dcgan_once(dtype), _dcgan_once(dtype)
    for x, y, what in zip(a, b, ("G grads", "D grads", "G params", "fake")):
        diff = np.flatnonzero(x.ravel() != y.ravel())
        assert diff.size == 0, "%s differ at %d elements (first %s)" % (what, diff.size, diff[:5])


def _pointnet_once(dtype):
    from paper_2102_02344_b200.pointnet import FusedPointNet
    B, N, L, k = 3, 8, 500, 40
    specs = [(n, s) for n, s, _ in synth.param_specs("pointnet_cls", k)]
    Ps = [synth.init_params("pointnet_cls", 1000 + b, k) for b in range(B)]
    net = FusedPointNet(B, specs, Ps, synth.hparams_pointnet(7, B), task="cls", dtype=dtype, N=N, L=L, k=k)
    x, y = synth.points_cls(0, N=N, L=L, k=k)
    net.step(torch.tensor(x.reshape(-1, 3), dtype=torch.float32, device="cuda"),
             torch.tensor(y, dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    return net.arena.g.cpu().numpy(), net.arena.p.cpu().numpy()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_pointnet_bitwise(dtype):
    a, b = _pointnet_once(dtype), _pointnet_once(dtype)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
