"""v7 vs v2 on one b = 6 shape in two subprocesses (BCG_RF_VARIANT), report
the differing elements (debug helper for the streamed recursion)."""
import os
import subprocess
import sys

import numpy as np

CODE = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import paper_1701_05420_b200 as bcg
n, t = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(2002)
x = rng.exponential(1.0, size=(t, n)) + rng.standard_normal((t, n))
np.save(sys.argv[3], bcg.cumulants_upto(x, 6, b=6)[6].packed_host())
"""
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n, t = int(sys.argv[1]), int(sys.argv[2])
out = {}
for name, env in (("v2", {"BCG_RF_VARIANT": "2"}), ("v7", {})):
    e = dict(os.environ, **env)
    path = f"/tmp/rs_{name}.npy"
    subprocess.check_call([sys.executable, "-c", CODE % root, str(n), str(t), path], env=e)
    out[name] = np.load(path)
d = out["v2"] != out["v7"]
print(f"n={n} tile={os.environ.get('BCG_RS_TILE', '0')}: {int(d.sum())} of {d.size} differ",
      (np.nonzero(d)[0][:10] // 46656).tolist(), float(np.max(np.abs(out['v2'] - out['v7']))))
