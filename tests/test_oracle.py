"""Pin the CPU oracle (oracle/crossmap_oracle.py) before trusting it.

Known-answer vectors are the ones frozen in the reference's own tests; the
golden fixtures are outputs of the reference itself (tests/golden/make_golden.py).
"""

import numpy as np
import pytest

import crossmap_oracle as O
from conftest import parse_case, parse_edim_case

# pkg/tests/test_knn.py:19-22
WEIGHTS_1_4_9 = [0.6652409557748219, 0.24472847105479767, 0.09003057317038046]
WEIGHTS_0_0_4 = [0.4223187982515182, 0.4223187982515182, 0.15536240349696362]
# pkg/tests/test_prediction.py:23-25
HAND_PREDICTIONS = [2.25, 1.5, 1.25]
HAND_RHO = -0.9607689228305228


def test_distance_kats():
    # pkg/tests/test_knn.py:26-37
    assert np.array_equal(O.squared_distances([7.0] * 4, 1, 1), np.zeros((4, 4)))
    assert O.squared_distances([0.0, 3.0], 1, 1).tolist() == [[0.0, 9.0], [9.0, 0.0]]
    assert O.squared_distances([0.0, 1.0, 3.0], 2, 1).tolist() == [[0.0, 5.0], [5.0, 0.0]]


def test_topk_kats():
    # pkg/tests/test_knn.py:66-76
    m = np.array([[5.0, 1, 3, 2], [1, 0, 2, 3], [3, 2, 0, 1], [2, 3, 1, 0]])
    d, i = O.select_k(m, 2)
    assert i[0].tolist() == [1, 3] and d[0].tolist() == [1.0, 2.0]
    m = np.ones((4, 4)) - np.eye(4)
    m[0] = [0.0, 1.0, 1.0, 1.0]
    assert O.select_k(m, 2)[1][0].tolist() == [1, 2]


def test_topk_matches_full_sort_with_ties():
    rng = np.random.default_rng(0)
    for trial in range(40):
        n = int(rng.integers(4, 40))
        m = rng.integers(0, 4, size=(n, n)).astype(float) if trial % 2 else rng.random((n, n))
        np.fill_diagonal(m, 0.0)
        k = int(rng.integers(1, n))
        d, idx = O.select_k(m, k)
        for r in range(n):
            row = m[r].copy()
            row[r] = np.inf
            order = np.lexsort((np.arange(n), row))[:k]
            assert idx[r].tolist() == order.tolist()


def test_weight_kats():
    assert np.allclose(O.simplex_weights(np.array([[1.0, 4.0, 9.0]]))[0], WEIGHTS_1_4_9, atol=1e-12)
    assert np.allclose(O.simplex_weights(np.array([[0.0, 0.0, 4.0]]))[0], WEIGHTS_0_0_4, atol=1e-12)
    assert np.allclose(O.simplex_weights(np.zeros((2, 4))), 0.25, atol=1e-15)


def test_hand_lookup_kat():
    idx = np.array([[1, 2], [0, 2], [0, 1]])
    w = np.array([[0.75, 0.25]] * 3)
    rho, pred = O.lookup(idx, w, 1, 1, [np.array([1.0, 2.0, 3.0])], want_predictions=True)
    assert pred[0].tolist() == HAND_PREDICTIONS
    assert abs(rho[0] - HAND_RHO) <= 1e-12


def test_knn_and_lookup_match_reference_goldens(golden):
    g = golden("knn_lookup")
    for key in g["cases"]:
        E, tau = parse_case(key)
        idx, w = O.knn_table(g[f"{key}_x"], E, tau, workers=2)
        assert np.array_equal(idx, g[f"{key}_idx"]), key
        assert np.max(np.abs(w - g[f"{key}_w"])) <= 1e-15, key
        rho, pred = O.lookup(idx, w, E, tau, list(g[f"{key}_targets"]), want_predictions=True)
        rho = np.array([np.nan if r is None else r for r in rho])
        assert np.array_equal(rho, g[f"{key}_rho"], equal_nan=True), key
        assert np.array_equal(np.stack(pred), g[f"{key}_pred"]), key


def test_edim_matches_reference_goldens(golden):
    g = golden("edim")
    for key in g["cases"]:
        E_max, tau, Tp = parse_edim_case(key)
        star, curve = O.edim(g[f"{key}_x"], E_max, tau, Tp, workers=2)
        assert star == int(g[f"{key}_estar"]), key
        assert np.array_equal(np.array([curve[e] for e in range(1, E_max + 1)]), g[f"{key}_curve"]), key
        assert O.simplex(g[f"{key}_x"], 3, tau, Tp) == float(g[f"{key}_simplex3"]), key


@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_config1_matches_reference(golden, tag):
    g = golden("config1")
    X = g[f"{tag}_x"]
    rho, stars = O.ccm_pairwise([X[0], X[1]], 20, 1, 1, workers=1)
    assert stars == g[f"{tag}_estar"].tolist()
    assert np.array_equal(rho, g[f"{tag}_rho"], equal_nan=True)
    fixed, tables = O.xmap([X[0], X[1]], [2, 2], 1)
    assert np.array_equal(fixed, g[f"{tag}_rho_e22"])
    assert np.max(np.abs(fixed - g[f"{tag}_brute_e22"])) <= 1e-9


def test_config1_survey_values(golden):
    # SURVEY.md section 7 (computed by the reference on float64 inputs)
    g = golden("config1")
    assert g["f64_estar"].tolist() == [1, 2]
    assert np.allclose(g["f64_rho"], [[0.9999979235921396, 0.42920905645039803],
                                      [0.1810567198762813, 0.999840242842384]], atol=1e-15)


def test_mixed20_pipeline_matches_reference(golden):
    g = golden("mixed20")
    X = g["x"]
    rho, stars = O.ccm_pairwise(list(X), 20, 1, 1, workers=4)
    assert stars == g["estar"].tolist()
    assert np.array_equal(rho, g["rho"], equal_nan=True)


def test_pearson_merge_invariance():
    rng = np.random.default_rng(3)
    a, b = rng.standard_normal(400), rng.standard_normal(400)
    whole = O.agg_rho(O.agg_from_arrays(a, b))
    parts = [O.agg_from_arrays(a[lo:hi], b[lo:hi]) for lo, hi in ((0, 37), (37, 200), (200, 400))]
    left = O.agg_merge(O.agg_merge(parts[0], parts[1]), parts[2])
    right = O.agg_merge(parts[0], O.agg_merge(parts[1], parts[2]))
    assert abs(O.agg_rho(left) - whole) <= 1e-12 and abs(O.agg_rho(right) - whole) <= 1e-12


def test_convergence_sampling_is_seeded_and_sorted():
    a = O.sample_libraries(100, [10, 50], 3, seed=5)
    b = O.sample_libraries(100, [10, 50], 3, seed=5)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    assert all(np.all(np.diff(blk, axis=1) > 0) for blk in a)


def test_convergence_full_library_equals_xmap():
    # with the whole point set as the library, every sample is the plain cross map
    rng = np.random.default_rng(9)
    x = rng.random(120)
    y = np.roll(x, 1) * 0.5 + rng.random(120) * 0.1
    n = O.valid_count(120, 3, 1)
    means, per = O.ccm_convergence(x, y, 3, 1, [n], 2, seed=1)
    idx, w = O.knn_table(x, 3, 1)
    direct = O.lookup(idx, w, 3, 1, [y])[0][0]
    assert np.allclose(per, direct, atol=1e-15)
