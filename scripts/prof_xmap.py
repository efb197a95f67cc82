"""Small xmap + edim run for ncu captures: python scripts/prof_xmap.py [N] [T]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2105_12301_b200 as P

N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1450
X = P.mixed_dataset(N, T, seed=2105)
est, _ = P.edim(X.T.astype(np.float64), 20, 1, 1)
rho = P.xmap(X.T, est, layout=P.LAYOUT_TGT_MAJOR, dtype=np.float32)
print("ok", N, T, np.bincount(est).tolist(), float(np.nanmean(rho)))
