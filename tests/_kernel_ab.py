"""Helper for test_tile_kernel_matches_v4: run the cross-map pipeline pieces on
fixed inputs and save everything to an .npz (run once per kNN kernel choice;
the library reads CMB_KNN_V4 once per process)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2105_12301_b200 as P  # noqa: E402


def cases():
    rng = np.random.default_rng(7)
    mixed = P.mixed_dataset(24, 900, seed=2105)
    yield "mixed", mixed
    ints = rng.integers(0, 5, size=(6, 700)).astype(np.float64)          # heavy exact ties
    yield "ints", ints
    per = np.tile(np.sin(np.arange(12) * 0.7), 60)[None, :].repeat(3, 0)   # exactly periodic
    per[1, 300:340] = 0.25                                                 # constant stretch
    yield "periodic", per
    yield "short", rng.random((5, 60))                                     # L < one tile
    yield "tiny", rng.random((4, 26))                                      # fewer candidates than lanes
    const = rng.random((4, 400))
    const[1] = 0.3                                                         # constant series
    const[2, :200] = 0.7                                                   # constant half
    yield "constant", const
    yield "float64", rng.standard_normal((5, 500)) * 1e3 + 1e-7 * rng.random((5, 500))  # not fp32-representable
    yield "long", P.mixed_dataset(4, 3000, seed=11)                       # several tiles


def main(out):
    res = {}
    for name, X in cases():
        emax = 20 if X.shape[1] >= 60 else 4
        est, curves = P.edim(X.T, emax, 1, 1)
        res[f"{name}_est"] = est
        res[f"{name}_curves"] = curves
        e = np.where(est > 0, est, 1)
        res[f"{name}_rho"] = P.xmap(X.T, e, dtype=np.float32)
        for E in (1, 3, 8, 20) if X.shape[1] >= 60 else (1, 2, 4):
            if X.shape[1] - (E - 1) < E + 2:
                continue
            t = P.build_knn_table(X[0], P.EmbeddingSpec(E, 1))
            res[f"{name}_idx{E}"] = t.indices
            res[f"{name}_w{E}"] = t.weights
    np.savez(out, **res)


if __name__ == "__main__":
    main(sys.argv[1])
