"""Bitwise A/B of the register-private Khatri-Rao moment kernel (BCG_MOMENT_PRIV=1)
against the shared-build kernel: packed raw moments of several shapes in two
subprocesses (the knob is read once per process)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import paper_1701_05420_b200 as bcg
out = {}
for i, (t, n, m, b) in enumerate([(5000, 12, 2, 3), (40000, 20, 3, 4), (33333, 24, 4, 4), (20000, 16, 5, 4),
                                  (50001, 18, 6, 3), (3000, 36, 6, 6), (9000, 11, 4, 3), (700, 300, 2, 7)]):
    rng = np.random.default_rng(100 + i)
    x = rng.standard_normal((t, n)) + rng.exponential(1.0, (t, n))
    out[f"s{i}"] = bcg.moment(x, m, b=b).packed_host()
np.savez(sys.argv[1], **out)
"""
res = {}
for name, env in (("shared", {}), ("priv", {"BCG_MOMENT_PRIV": "1"})):
    path = f"/tmp/ab_priv_{name}.npz"
    subprocess.check_call([sys.executable, "-c", CODE % ROOT, path], env=dict(os.environ, **env))
    res[name] = np.load(path)
bad = 0
for k in res["shared"].files:
    a, b = res["shared"][k], res["priv"][k]
    d = int((a != b).sum())
    bad += d
    print(k, a.size, "differ:", d, "max abs", float(np.max(np.abs(a - b))) if d else 0.0)
print("BITWISE OK" if bad == 0 else "MISMATCH")
