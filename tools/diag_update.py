import sys
import numpy as np
sys.path.insert(0, ".")
from tests.test_gpu_pointnet import run_pair
import paper_2102_02344_b200.hfta as H
H.hfta_init(0)
net, out = run_pair("cls", "f32", 3, 32, 50, 40)
loss, ref, grads, res = out[0]
b = 0
n = "head.fc2.W"
g_ref = res[b]["grads"][n]; g_gpu = grads[b][n]
p0 = res[b]["p_before"][n]; pr = res[b]["params"][n]; pg = res[b]["p_gpu_after"][n]
hp = {k: float(net.hv.t[k][b].item()) for k in net.hv.t}
print("hp", hp)
d = np.abs((pg - p0) - (pr - p0))
idx = np.argsort(-d.ravel())[:8]
for i in idx:
    print("elem", np.unravel_index(i, d.shape), "g_ref %.3e g_gpu %.3e p0 %.3e upd_ref %.3e upd_gpu %.3e" % (
        g_ref.ravel()[i], g_gpu.ravel()[i], p0.ravel()[i], (pr - p0).ravel()[i], (pg - p0).ravel()[i]))
print("grad relerr", np.linalg.norm(g_gpu - g_ref) / np.linalg.norm(g_ref))
m_gpu = net.arena.host_tensor("m", n)[b]; v_gpu = net.arena.host_tensor("v", n)[b]
m_ref, v_ref = res[b]["opt"][n]
print("m relerr", np.linalg.norm(m_gpu - m_ref) / np.linalg.norm(m_ref), "v relerr", np.linalg.norm(v_gpu - v_ref) / np.linalg.norm(v_ref))
