import os, subprocess, sys, numpy as np
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2104_04726_b200 import _lib as L
rng = np.random.default_rng(0)
n, k = 1080, 270
q, _ = np.linalg.qr(rng.standard_normal((n, n)))
lam = 1e3 * np.exp(-np.linspace(0, 20, n))
g = (q * lam) @ q.T; g = 0.5 * (g + g.T)
gd = L.dev_f64(g); vecs = L.empty_f64(n * k); vals = L.empty_f64(k); h = L.ctx()
L.check(L.LIB.tmb_leading_eigvecs(h, L.ptr(gd), n, k, L.ptr(vecs), L.ptr(vals)), h)
torch.cuda.synchronize()
np.save(sys.argv[1], np.concatenate([vecs.cpu().numpy().ravel(), vals.cpu().numpy().ravel()]))
'''
open("/tmp/tc.py", "w").write(code)
for t in ("0", "128"):
    env = dict(os.environ, TMB_SYTRD_TAIL1=t)
    subprocess.run([sys.executable, "/tmp/tc.py", f"/tmp/tc_{t}.npy"], env=env, check=True)
a, b = np.load("/tmp/tc_0.npy"), np.load("/tmp/tc_128.npy")
print("max abs diff", np.abs(a - b).max(), "identical", np.array_equal(a, b))
