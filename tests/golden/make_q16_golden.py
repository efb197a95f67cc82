"""Oracle rho for the 16-bit target-lookup case (tests/test_gpu_parity.py::test_q16_target_mode).

160 series of the mixed recipe at T = 700 (seed 31), series 5 replaced by a
constant, E* from the oracle edim (E_max = 20, Tp = 1; undefined -> 1), rho
from the oracle xmap (fp64).  Writes xmap_mixed160_t700_const5.npz (~1 min).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
import crossmap_oracle as O  # noqa: E402
from paper_2105_12301_b200.synthetic import mixed_dataset  # noqa: E402


def main():
    X = mixed_dataset(160, 700, seed=31).astype(np.float64)
    X[5, :] = 0.25
    est = np.array([O.edim(x, 20, 1, 1)[0] or 1 for x in X], dtype=np.int32)
    rho, _ = O.xmap(list(X), est)
    np.savez_compressed(os.path.join(HERE, "xmap_mixed160_t700_const5.npz"), rho=rho, est=est)


if __name__ == "__main__":
    main()
