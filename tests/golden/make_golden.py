"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package (pkg/src/crossmap,
pkg/binding/src/crossmap_binding and the brute-force oracle
pkg/tests/bruteforce.py) read-only, evaluates it on seeded inputs that are
rounded to float32 first (the B200 path computes on float32 samples, so the
reference is fed the identical values), and writes compressed .npz files.
The GPU box never needs /root/reference: the tests read only these fixtures.
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "binding" / "src"), str(REF / "tests")]

import numpy as np  # noqa: E402

import crossmap as ref  # noqa: E402
import bruteforce  # noqa: E402
from crossmap_binding import ccm_matrix as ref_ccm_matrix  # noqa: E402

OUT = Path(__file__).resolve().parent


def f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def make_mixed(length, seed):
    """pkg/tests/conftest.py:7-23 (the reference's own 20-series fixture)."""
    rng = np.random.default_rng(seed)
    cols, names = [], []
    for i, r in enumerate((3.58, 3.62, 3.7, 3.74, 3.82, 3.87, 3.92, 3.99)):
        cols.append(ref.logistic_map(length, seed=seed + i, r=r).values)
        names.append(f"log{i}")
    for i, beta in enumerate((0.25, 0.35, 0.5)):
        pair = ref.coupled_logistic(length, seed=seed + 50 + i, beta=beta)
        cols += [pair[0].values, pair[1].values]
        names += [f"drv{i}", f"rsp{i}"]
    for i in range(4):
        cols.append(ref.uniform_noise(length, seed=seed + 90 + i).values)
        names.append(f"noise{i}")
    steps = np.arange(length)
    for i, period in enumerate((47.0, 131.0)):
        cols.append(np.sin(2 * np.pi * steps / period) + 0.05 * rng.standard_normal(length))
        names.append(f"sine{i}")
    return np.stack(cols), names


def knn_inputs():
    rng = np.random.default_rng(4242)
    cases = {
        "noise": f32(ref.uniform_noise(300, seed=1).values),
        "logistic": f32(ref.logistic_map(300, seed=2, r=3.8).values),
        "r4tail": f32(ref.logistic_map(120, r=4.0, v0=0.5).values),   # constant tail: zero distances
        "ties": rng.integers(0, 3, 200).astype(np.float64),            # heavy exact ties
        "sine": f32(np.sin(np.linspace(0, 40 * np.pi, 500))),
        "constant": np.full(50, 2.5),
    }
    return cases


def main():
    out = {}
    # ---------------- synthetic generators (for the package's vectorised copies)
    out["syn_logistic"] = ref.logistic_map(100, seed=7, r=3.7).values
    pair = ref.coupled_logistic(64, seed=3, beta=0.4)
    out["syn_coupled"] = np.stack([pair[0].values, pair[1].values])
    out["syn_noise"] = ref.uniform_noise(40, seed=5).values
    mixed60, _ = make_mixed(60, 1234)
    out["syn_mixed60"] = mixed60
    np.savez_compressed(OUT / "synthetic.npz", **out)

    # ---------------- kNN tables + lookups (knn.py:205-217, prediction.py:122-161)
    out = {}
    case_list = []
    for name, x in knn_inputs().items():
        for E, tau in ((1, 1), (2, 1), (3, 2), (5, 1), (5, 2), (20, 1)):
            spec = ref.EmbeddingSpec(E, tau)
            try:
                table = ref.build_knn_table(x, spec, workers=1)
            except ref.SeriesTooShortError:
                continue
            key = f"{name}_E{E}_t{tau}"
            case_list.append(key)
            out[f"{key}_x"] = x
            out[f"{key}_idx"] = table.indices.astype(np.int32)
            out[f"{key}_w"] = table.weights
            # sorted squared distances too (pairwise_distances + partial_sort_topk)
            top_d, _ = ref.partial_sort_topk(ref.pairwise_distances(x, spec, workers=1), E + 1, workers=1)
            out[f"{key}_d"] = top_d
            # cross-map lookups of three targets through this table (Tp = 0)
            trg = [f32(ref.uniform_noise(x.size, seed=77).values), x,
                   f32(np.cos(np.arange(x.size) / 7.0))]
            res = ref.lookup_batch(table, trg, want_predictions=True, workers=1)
            out[f"{key}_targets"] = np.stack(trg)
            out[f"{key}_rho"] = np.array([np.nan if r.rho is None else r.rho for r in res])
            out[f"{key}_pred"] = np.stack([r.predicted for r in res])
    out["cases"] = np.array(case_list)
    np.savez_compressed(OUT / "knn_lookup.npz", **out)

    # ---------------- edim curves / simplex (prediction.py:164-262)
    out = {}
    series = {
        "logistic": f32(ref.logistic_map(400, seed=27, r=3.85).values),
        "noise": f32(ref.uniform_noise(300, seed=28).values),
        "period2": np.tile([0.2, 0.8], 100).astype(np.float32).astype(np.float64),
        "sine": f32(np.sin(np.linspace(0, 40 * np.pi, 500))),
        "coupled": f32(ref.coupled_logistic(600, seed=6, beta=0.3)[1].values),
    }
    names = []
    for name, x in series.items():
        for E_max, tau, Tp in ((20, 1, 1), (6, 2, 2), (8, 1, 3)):
            res = ref.optimal_embedding(x, e_max=E_max, tau=tau, tp=Tp, workers=1)
            key = f"{name}_M{E_max}_t{tau}_p{Tp}"
            names.append(key)
            out[f"{key}_x"] = x
            out[f"{key}_curve"] = np.array([res.rho_by_e[e] for e in range(1, E_max + 1)])
            out[f"{key}_estar"] = np.array(res.e_star)
            out[f"{key}_simplex3"] = np.array(ref.simplex_self_predict(x, ref.EmbeddingSpec(3, tau), tp=Tp, workers=1))
    out["cases"] = np.array(names)
    np.savez_compressed(OUT / "edim.npz", **out)

    # ---------------- config 1: coupled logistic T=1000 (SURVEY.md section 7 goldens)
    out = {}
    pair = ref.coupled_logistic(1000, seed=3, beta=0.4)
    x64 = np.stack([pair[0].values, pair[1].values])
    for tag, X in (("f64", x64), ("f32", f32(x64))):
        data = ref.Dataset((ref.TimeSeries(X[0], "driver"), ref.TimeSeries(X[1], "response")))
        m = ref.ccm_pairwise(data, ref.CcmConfig(), workers=1)
        stars = [ref.optimal_embedding(X[i], 20, 1, 1, workers=1) for i in range(2)]
        out[f"{tag}_x"] = X
        out[f"{tag}_rho"] = m.rho
        out[f"{tag}_estar"] = np.array([s.e_star for s in stars])
        out[f"{tag}_curves"] = np.stack([[s.rho_by_e[e] for e in range(1, 21)] for s in stars])
        out[f"{tag}_tables_built"] = np.array(m.stats.tables_built)
        fixed = ref.ccm_pairwise(data, ref.CcmConfig(), e_star=[2, 2], workers=1)
        out[f"{tag}_rho_e22"] = fixed.rho
        out[f"{tag}_brute_e22"] = bruteforce.ccm_matrix([X[0], X[1]], [2, 2])
    np.savez_compressed(OUT / "config1.npz", **out)

    # ---------------- 20-series mixed pipeline (pkg/tests/conftest.py fixture), float32-rounded
    X, names = make_mixed(2000, 1234)
    X = f32(X)
    bound = ref_ccm_matrix(X.T, names, workers=8)
    stars = [ref.optimal_embedding(X[i], 20, 1, 1, workers=8) for i in range(len(names))]
    np.savez_compressed(OUT / "mixed20.npz", x=X, names=np.array(names), rho=bound.skill,
                        estar=np.array([s.e_star for s in stars]),
                        curves=np.stack([[s.rho_by_e[e] for e in range(1, 21)] for s in stars]))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
