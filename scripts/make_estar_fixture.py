"""Regenerate tests/golden/estar_config3.npz: E* of the config-3 dataset
(mixed recipe, N = 53,053, T = 1,450, seed 2105; float32 samples) from the GPU
edim (E_max = 20, Tp = 1).  bench.py's reference arm reads it so that it never
loads libcmb200; tests/test_gpu_scale.py checks 64 sampled entries against the
oracle's optimal_embedding.  Run on a GPU box:  python scripts/make_estar_fixture.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import paper_2105_12301_b200 as P
    n, t, seed = 53053, 1450, 2105
    X = P.mixed_dataset(n, t, seed=seed, dtype=np.float32)
    est, rho = P.edim(X.T.astype(np.float64), 20, 1, 1)
    out = ROOT / "tests" / "golden" / "estar_config3.npz"
    np.savez(out, estar=est.astype(np.int8), n=n, t=t, seed=seed)
    ties = P.near_ties(rho, est)
    print(f"wrote {out}: E* histogram {np.bincount(est, minlength=21).tolist()}, "
          f"{len(ties)} series with a best/runner-up gap < 1e-4")


if __name__ == "__main__":
    main()
