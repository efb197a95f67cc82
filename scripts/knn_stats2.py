"""Selection counters of one xmap table build (needs a CMB_STATS=1 build):
python scripts/knn_stats2.py [N]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2105_12301_b200 as P
from paper_2105_12301_b200 import _native as nat

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
X = P.mixed_dataset(N, 1450, seed=2105)
est, _ = P.edim(X.T.astype(np.float64), 20, 1, 1)
out = np.zeros(8, dtype=np.int64)
nat.call("cmb_diagnostics", 0, nat.ptr(out), 8)
print("edim rows", out[1], "pool/rowE %.2f rounds/rowE %.3f hits/rowE %.2f overflows/rowE %.4f fallback %d" % (out[3] / out[1], out[4] / out[1], out[5] / out[1], out[6] / out[1], out[0]))
t0 = time.time()
P.xmap(X.T, est, layout=P.LAYOUT_TGT_MAJOR, dtype=np.float32)
nat.call("cmb_diagnostics", 0, nat.ptr(out), 8)
print("xmap rows", out[1], "pool/rowE %.2f rounds/rowE %.3f hits/rowE %.2f overflows/rowE %.4f fallback %d" % (out[3] / out[1], out[4] / out[1], out[5] / out[1], out[6] / out[1], out[0]), time.time() - t0)
