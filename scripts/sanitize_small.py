"""Small end-to-end run of every device path, for compute-sanitizer:
    compute-sanitizer --tool memcheck python scripts/sanitize_small.py"""
import os
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_2105_12301_b200 as P

rng = np.random.default_rng(3)
X = P.mixed_dataset(40, 300, seed=5)
est, curves = P.edim(X.T, 12, 1, 1)                       # EDIM tile kernel
e = np.where(est > 0, est, 1)
rho = P.xmap(X.T, e, dtype=np.float32)                    # TABLE tile kernel + resident lookup
os.environ["CMB_LOOKUP_FP16"] = "1"
rho16 = P.xmap(X.T, e, dtype=np.float32)                  # fp16-target lookup
os.environ.pop("CMB_LOOKUP_FP16")
Xl = P.mixed_dataset(6, 7000, seed=6)                     # long series: non-resident lookup
rl = P.xmap(Xl.T, [1, 2, 3, 2, 1, 4], dtype=np.float32)  # (target-block-major work items)
os.environ["CMB_LOOKUP_TMAJOR"] = "0"                     # library-major order, same kernel
rl0 = P.xmap(Xl.T, [1, 2, 3, 2, 1, 4], dtype=np.float32)
os.environ.pop("CMB_LOOKUP_TMAJOR")
assert np.array_equal(np.nan_to_num(rl), np.nan_to_num(rl0))
t = P.build_knn_table(X[3], P.EmbeddingSpec(5, 1))        # RAW tile kernel
t2 = P.build_knn_table(X[3], P.EmbeddingSpec(3, 2))       # RAW v4 (tau = 2)
cv = P.ccm_sweep(X[:5].T, e[:5], [20, 80], samples=3)     # convergence tables + lookup
cv2 = P.ccm_sweep(X[:3].T, e[:3], [30], samples=2, tau=2) # generic restricted tables
# round 2 paths: rotated lookup with every (library, block) queued for the fp64
# fixup, float64 inputs with an offset (cmb_xmap64), predictions from the xmap
# tables (cmb_xmap_predict), the NCCL rank path with one rank (cmb_xmap_multi)
os.environ["CMB_FIX_RATIO"] = "2"
rfix = P.xmap(X.T, e, dtype=np.float32)
os.environ.pop("CMB_FIX_RATIO")
r64 = P.xmap((300.0 + 1e-3 * X).T, e)
data = P.Dataset(tuple(P.TimeSeries(X[i], f"s{i}") for i in range(12)))
mp = P.ccm_pairwise(data, P.CcmConfig(e_max=8, emit_predictions=True))
from paper_2105_12301_b200.distributed import xmap_multi
rm = xmap_multi(X.astype(np.float32), e, [0])
with tempfile.TemporaryDirectory() as d:
    m = P.SkillMatrix([f"s{i}" for i in range(40)], np.nan_to_num(rho.astype(np.float64), nan=0.5))
    P.write_skill_matrix(m, Path(d) / "m.csv")           # GPU CSV formatter
    back = P.read_skill_matrix(Path(d) / "m.csv")
print("ok", float(np.nanmean(rho)), float(np.nanmean(rho16)), float(np.nanmean(rl)), t.indices.shape,
      t2.indices.shape, cv.shape, cv2.shape, back.rho.shape, float(np.nanmax(np.abs(rfix - rho))),
      float(np.nanmean(r64)), len(mp.predictions), float(np.nanmax(np.abs(rm - rho))))
