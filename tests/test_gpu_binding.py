"""The drop-in surfaces on the GPU: the binding's contract tests
(pkg/binding/tests/test_binding.py:23-60 -- binding vs CLI, no mutation of the
caller's arrays across dtypes) and materialised predictions from the cross
map's own tables (ccm.py:130, 148-149, prediction.py:145-153)."""

import numpy as np
import pytest

import crossmap_oracle as O
import paper_2105_12301_b200 as P
from paper_2105_12301_b200.cli import run_ccm

pytestmark = pytest.mark.gpu


def _write_csv(names, cols, path):
    lines = [",".join(names)] + [",".join(repr(float(c[t])) for c in cols) for t in range(len(cols[0]))]
    path.write_text("\n".join(lines) + "\n")


def test_binding_parity_with_cli(tmp_path):
    """ccm_matrix equals the CLI's in-memory result (the same device path) to
    1e-12 and the caller's array is not mutated (test_binding.py:23-40)."""
    X = P.mixed_dataset(20, 600, seed=2105)
    names = [f"s{i}" for i in range(20)]
    src, dst = tmp_path / "m.csv", tmp_path / "o.csv"
    _write_csv(names, list(X), src)
    cli_matrix, _ = run_ccm(str(src), str(dst), P.CcmConfig(), workers=2)
    values = np.ascontiguousarray(X.T)
    snapshot = values.copy()
    bound = P.ccm_matrix(values, names, workers=2)
    assert bound.names == cli_matrix.names
    assert np.array_equal(np.isnan(bound.skill), np.isnan(cli_matrix.rho))
    assert np.nanmax(np.abs(bound.skill - cli_matrix.rho)) <= 1e-12
    assert np.array_equal(values, snapshot)


def test_inputs_never_mutated_across_dtypes():
    """test_binding.py:54-60: C, Fortran and integer arrays come back untouched."""
    rng = np.random.default_rng(0)
    base = rng.random((300, 2))
    for candidate in (base, np.asfortranarray(base), (base * 100).astype(np.int64)):
        snapshot = candidate.copy()
        P.ccm_matrix(candidate, ["a", "b"], e_max=3, workers=1)
        assert np.array_equal(candidate, snapshot)
    x = rng.random(200)
    snap = x.copy()
    P.binding.simplex(x, 3)
    P.binding.optimal_embedding(x, E_max=5)
    assert np.array_equal(x, snap)


def test_emit_predictions_from_the_cross_map_tables():
    """ccm_pairwise(emit_predictions=True): every defined (library, target) pair's
    prediction series, in the reference's order, against the oracle's
    lookup(want_predictions=True) on the same data (fp32 lookup path: 1e-4)."""
    X = P.mixed_dataset(12, 400, seed=31)
    X[4] = 0.5  # a constant series: no row or column
    data = P.Dataset(tuple(P.TimeSeries(X[i], f"s{i}") for i in range(12)))
    m = P.ccm_pairwise(data, P.CcmConfig(e_max=8, emit_predictions=True))
    est, _ = P.edim(X.T, 8, 1, 1)
    defined = [i for i in range(12) if est[i] > 0]
    assert 4 not in defined
    groups = {}
    for t in defined:
        groups.setdefault(int(est[t]), []).append(t)
    want_order = [(l, t) for l in defined for e in sorted(groups) for t in groups[e]]
    assert list(m.predictions) == want_order
    worst = 0.0
    for lib in defined:
        for e, ts in groups.items():
            idx, w = O.knn_table(X[lib], e, 1)
            rr, preds = O.lookup(idx, w, e, 1, [X[t] for t in ts], want_predictions=True)
            for t, r, pr in zip(ts, rr, preds):
                got = m.predictions[(lib, t)]
                assert got.shape == pr.shape
                worst = max(worst, float(np.max(np.abs(got - pr))))
                if r is not None:
                    assert abs(m.rho[lib, t] - r) <= 1e-4
    assert worst <= 1e-4, worst
