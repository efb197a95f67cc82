"""Selection statistics of the kNN sweep (hits, compactions) for one xmap."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2105_12301_b200 as P
from paper_2105_12301_b200 import _native as nat

N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
X = P.mixed_dataset(N, 1450, seed=2105)
est, _ = P.edim(X.T.astype(np.float64), 20, 1, 1)
out = np.zeros(8, dtype=np.int64)
nat.call("cmb_diagnostics", 0, nat.ptr(out), 8)
print("edim:", out.tolist())
for kind in ("all", "noise-only", "logistic-only"):
    if kind == "all":
        Xs = X
    elif kind == "noise-only":
        Xs = X[[i for i in range(N) if i % 20 in (14, 15, 16, 17)]]
    else:
        Xs = X[[i for i in range(N) if i % 20 < 8]]
    e = est[: len(Xs)] * 0 + est.max()
    e[:] = np.arange(len(Xs)) % 20 + 1
    P.xmap(Xs.T, e, layout=P.LAYOUT_TGT_MAJOR, dtype=np.float32)
    nat.call("cmb_diagnostics", 0, nat.ptr(out), 8)
    rows = out[1]
    print(kind, "rowsE", rows, "hits/rowE %.1f" % (out[3] / rows), "compactions/rowE %.2f" % (out[4] / rows),
          "events/rowE %.2f" % (out[5] / rows), "fallback", out[0])
