"""Diagnostic: per-tensor normwise errors of the fused PointNet step vs the
decision-matched oracle, plus the gradient arriving at every BN layer
(GPU buffer vs the oracle's value captured from its backward)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import models as OM
from tests.test_gpu_pointnet import run_pair
from tests._cmp import relerr
import paper_2102_02344_b200.hfta as H

H.hfta_init(0)
CAP = {}
_orig = OM._conv_bn_act_bwd


def _cap(P, G, da, cache, need_dx=True):
    CAP.setdefault(cache["bnn"], []).append(da)
    return _orig(P, G, da, cache, need_dx)


OM._conv_bn_act_bwd = _cap
task, dtype, B, N, L, k = sys.argv[1], sys.argv[2], 1, int(sys.argv[3]), int(sys.argv[4]), 40
net, out = run_pair(task, dtype, B, N, L, k, witness=False)
loss, ref, grads, res = out[0]
print(dtype, "loss", loss, ref)
errs = [(relerr(grads[0][n], res[0]["grads"][n]), n, np.linalg.norm(res[0]["grads"][n])) for n in res[0]["grads"]]
print(" ".join("%s:%.1e(|%.0e|)" % (n, e, nr) for e, n, nr in errs))
S = net.S
gpu_da = {"stn.bn2": S["d.c2a"], "feat.bn2": S["d.c2a"]}
# the last-captured call of each name is the decision-matched pass
for name, lst in CAP.items():
    print(name, "captured", len(lst), "shape", lst[-1].shape)
if "stn.bn2" in CAP:
    da = CAP["stn.bn2"][-1]
    g = S["d.c2a"][0].float().cpu().numpy()
    print("stn.bn2 incoming grad rel err:", relerr(g, da), "norm", np.linalg.norm(da))
    y2 = S["stn.y2"][0].float().cpu().numpy() if "stn.y2" in S else None
