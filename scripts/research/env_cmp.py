"""Research check: leading_eigvecs output with an A/B environment switch on
and off must be bitwise identical (or report the difference).
  python scripts/research/env_cmp.py VAR=value [n k]"""
import os
import subprocess
import sys

import numpy as np

var, val = sys.argv[1].split("=", 1)
n, k = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (1920, 480)
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2104_04726_b200 import _lib as L
rng = np.random.default_rng(0)
n, k = int(sys.argv[2]), int(sys.argv[3])
q, _ = np.linalg.qr(rng.standard_normal((n, n)))
lam = 1e3 * np.exp(-np.linspace(0, 20, n))
g = (q * lam) @ q.T; g = 0.5 * (g + g.T)
gd = L.dev_f64(g); vecs = L.empty_f64(n * k); vals = L.empty_f64(k); h = L.ctx()
L.check(L.LIB.tmb_leading_eigvecs(h, L.ptr(gd), n, k, L.ptr(vecs), L.ptr(vals)), h)
torch.cuda.synchronize()
np.save(sys.argv[1], np.concatenate([vecs.cpu().numpy().ravel(), vals.cpu().numpy().ravel()]))
'''
open("/tmp/env_cmp_run.py", "w").write(code)
out = {}
for tag, env in (("off", {k_: v for k_, v in os.environ.items() if k_ != var}), ("on", dict(os.environ, **{var: val}))):
    subprocess.run([sys.executable, "/tmp/env_cmp_run.py", f"/tmp/env_cmp_{tag}.npy", str(n), str(k)], env=env,
                   check=True, timeout=120)
    out[tag] = np.load(f"/tmp/env_cmp_{tag}.npy")
print(f"{var}={val} n={n} k={k}: identical {np.array_equal(out['on'], out['off'])}, "
      f"max abs diff {float(np.abs(out['on'] - out['off']).max()):.3e}")
