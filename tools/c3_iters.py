import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1310_6736_b200 as sx
from tests import phantoms
vol, _ = sx.make_phantom(phantoms.config_c3())
sel, seeds, visits = sx.detect_records(vol, "shift", 16.0, [8.0, 12.0], 20, 5.0, 0, 64, 64, per_seed=True)
it = seeds["iterations"]; sc = np.sqrt(seeds["H"][:, 0])
for s in (8, 12):
    m = sc == s
    print(s, "n", m.sum(), "iters mean", it[m].mean(), "p50", np.median(it[m]), "p99", np.percentile(it[m], 99), "max", it[m].max(), "n50", (it[m] == 50).sum(), "degenerate", ((seeds["flags"][m] & 2) > 0).sum())
print("visits", visits)
