"""Config 5 (BASELINE configs[4]): ccm convergence sweep -- library sizes 100..1,400
(step 100), 100 random library samples per size, all ordered pairs of a
256-series batch (T = 1,450, E from GPU edim).  GPU wall time vs the oracle
restatement on a bounded sample (pairs x sizes x samples), extrapolated.
python scripts/bench_ccm.py [N_series] [samples]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import numpy as np

import crossmap_oracle as O
import paper_2105_12301_b200 as P

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
S = int(sys.argv[2]) if len(sys.argv) > 2 else 100
T = 1450
sizes = list(range(100, 1401, 100))
X = P.mixed_dataset(N, T, seed=2105)
est, _ = P.edim(X.T, 20, 1, 1)
E = np.where(est > 0, est, 1).astype(np.int32)
P.ccm_sweep(X[:4].T, E[:4], sizes[:2], samples=2)  # warm-up
t0 = time.perf_counter()
rho = P.ccm_sweep(X.T, E, sizes, samples=S, seed=7)
el = time.perf_counter() - t0
units = N * N * len(sizes) * S  # (pair, size, sample) skills
# oracle: 2 pairs x 2 sizes x 3 samples
t0 = time.perf_counter()
cnt = 0
for (l, t) in [(0, 1), (5, 9)]:
    O.ccm_convergence(X[l], X[t], int(E[t]), 1, [100, 1400], 3, 7)
    cnt += 2 * 3
el_o = time.perf_counter() - t0
print(json.dumps({"config": f"ccm convergence N={N} T={T} sizes 100..1400 x {S} samples, all pairs",
                  "gpu_seconds": el, "skills_per_s": units / el, "units": units,
                  "oracle_skills_per_s": cnt / el_o, "speedup": (units / el) / (cnt / el_o),
                  "finite_fraction": float(np.isfinite(rho).mean())}))
