import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_1701_05420_b200 as bcg
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
rng = np.random.default_rng(1)
x = rng.exponential(1.0, size=(300, n)) + rng.standard_normal((300, n))
cs = bcg.cumulants_upto(x, 6, b=6)
print("ok", float(np.abs(cs[6].packed_host()).sum()))
