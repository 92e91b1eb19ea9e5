"""Diagnostic: per-tensor normwise errors of the fused PointNet step vs the oracle."""
import sys
import numpy as np
sys.path.insert(0, ".")
from tests.test_gpu_pointnet import run_pair
from tests._cmp import relerr
import paper_2102_02344_b200.hfta as H
H.hfta_init(0)
for dtype, B, N, L, k, steps in [("f32", 2, 4, 200, 10, 2), ("bf16", 3, 4, 300, 40, 1)]:
    net, out = run_pair("cls", dtype, B, N, L, k, steps=steps)
    for t, (loss, ref, grads, res) in enumerate(out):
        print(dtype, "step", t + 1, "loss", loss, ref)
        for b in range(B):
            errs = [(relerr(grads[b][n], res[b]["grads"][n]), n, np.linalg.norm(res[b]["grads"][n])) for n in res[b]["grads"]]
            print("  model", b, " ".join("%s:%.1e(|%.0e|)" % (n, e, nr) for e, n, nr in errs))
    pe = [(n, relerr(net.params(0)[n], res[0]["params"][n])) for n in res[0]["params"]]
    print(" params after last step, model 0:", " ".join("%s:%.1e" % x for x in pe))
