"""CPU-side checks of the drop-in boundary (no GPU needed)."""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_2105_12301_b200 as P
from paper_2105_12301_b200 import _native

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "cmb200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(cmb_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert "cmb_xmap" in syms and "cmb_knn_table" in syms and "cmb_edim" in syms
    assert set(syms) == set(_native.EXPORTS)


def test_library_loads_and_exports_every_declared_symbol():
    lib = _native.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.cmb_version() == 100
    assert P.__version__ == "0.1.0" and P.binding.__version__ == P.__version__


def test_no_cpu_fallback_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(P.DeviceError):
        P.simplex(np.random.default_rng(0).random(100), 2)


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(P.DeviceError, match="not built"):
        _native.load(tmp_path / "libcmb200.so")


def test_host_validation_matches_reference_messages():
    with pytest.raises(P.ParameterError, match="names"):
        P.ccm_matrix(np.random.default_rng(1).random((100, 2)), [])
    with pytest.raises(P.ParameterError, match="2-D"):
        P.ccm_matrix(np.zeros(10), ["a"])
    bad = np.ones((60, 2))
    bad[3, 1] = np.nan
    with pytest.raises(P.ParameterError, match="non-finite"):
        P.ccm_matrix(bad, ["a", "b"], e_max=2)
    with pytest.raises(P.ParameterError, match="own neighbor"):
        P.NeighborTable(np.array([[0, 1], [0, 2], [0, 1]]), np.array([[0.6, 0.4]] * 3), P.EmbeddingSpec(1, 1))
    idx = np.array([[1, 2], [0, 2], [0, 1]])
    with pytest.raises(P.ParameterError, match="sum"):
        P.NeighborTable(idx, np.array([[0.6, 0.3]] * 3), P.EmbeddingSpec(1, 1))
    with pytest.raises(P.ParameterError, match="non-increasing"):
        P.NeighborTable(idx, np.array([[0.4, 0.6]] * 3), P.EmbeddingSpec(1, 1))
    with pytest.raises(P.ParameterError, match="distinct"):
        P.NeighborTable(np.array([[1, 1], [0, 2], [0, 1]]), np.array([[0.6, 0.4]] * 3), P.EmbeddingSpec(1, 1))
    with pytest.raises(P.ParameterError):
        P.EmbeddingSpec(21, 1)
    assert P.EmbeddingSpec(25, 1, e_max=30).E == 25
    with pytest.raises(P.SeriesTooShortError):
        P.valid_count(5, P.EmbeddingSpec(3, 2))
    assert P.valid_count(100, P.EmbeddingSpec(3, 2)) == 96
    with pytest.raises(P.ParameterError, match="lengths differ"):
        P.Dataset((P.TimeSeries([1, 2], "a"), P.TimeSeries([1, 2, 3], "b")))
    with pytest.raises(P.ParameterError, match="duplicate"):
        P.Dataset((P.TimeSeries([1, 2], "a"), P.TimeSeries([3, 4], "a")))
    with pytest.raises(P.ParameterError, match="position 1"):
        P.TimeSeries([1.0, np.nan, 2.0])
    for kw in ({"e_max": 0}, {"tau": 0}, {"tp_search": 0}):
        with pytest.raises(P.ParameterError):
            P.CcmConfig(**kw)


def test_group_by_optimal_e():
    embs = [P.OptimalEmbedding(2, {2: 0.5}), P.OptimalEmbedding(2, {2: 0.4}), P.OptimalEmbedding(5, {5: 0.9})]
    assert P.group_by_optimal_e(embs) == {2: [0, 1], 5: [2]}
    assert P.group_by_optimal_e([]) == {}


def test_pearson_merge_is_host_logic():
    a = P.PearsonAggregate(3, 1.0, 2.0, 2.0, 2.0, 1.0)
    assert a.merge(P.PearsonAggregate.empty()) == a
    assert P.PearsonAggregate.empty().merge(a) == a


def test_synthetic_generators_bit_identical_to_reference(golden):
    g = golden("synthetic")
    assert np.array_equal(P.logistic_map(100, seed=7, r=3.7).values, g["syn_logistic"])
    pair = P.coupled_logistic(64, seed=3, beta=0.4)
    assert np.array_equal(np.stack([pair[0].values, pair[1].values]), g["syn_coupled"])
    assert np.array_equal(P.uniform_noise(40, seed=5).values, g["syn_noise"])
    assert np.array_equal(P.mixed_dataset(20, 60, seed=1234, dtype=np.float64), g["syn_mixed60"])
    tiled = P.mixed_dataset(45, 60, seed=1234, dtype=np.float64)
    assert np.array_equal(tiled[:20], g["syn_mixed60"]) and tiled.shape == (45, 60)


def test_convergence_sampling_matches_oracle_rule():
    import crossmap_oracle as O
    from paper_2105_12301_b200.convergence import sample_libraries
    a = sample_libraries(500, [10, 100, 500], 4, seed=21)
    b = O.sample_libraries(500, [10, 100, 500], 4, seed=21)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    with pytest.raises(P.ParameterError):
        sample_libraries(50, [60], 1, seed=0)


def test_bench_roofline_models():
    """bench.py's algorithmic byte and shared-memory wavefront models (K3)
    on a hand-countable workload: 2 libraries, targets E* = [1, 1, 2], T = 10."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    estar = np.array([1, 1, 2], dtype=np.int32)
    T, libs = 10, 2
    # E=1: N_E=2, n_E=10, k=2; E=2: N_E=1, n_E=9, k=3  (B_pair = 4 n + 8 n k / N_E + 4)
    want = libs * (2 * (4 * 10 + 4) + 8 * 10 * 2) + libs * (1 * (4 * 9 + 4) + 8 * 9 * 3)
    assert bench.lookup_alg_bytes(estar, libs, T) == want
    # one 32-target block per E group; per point and 32 pairs k gathers + the observed
    # value + R/64 record loads (two-target path: k=2 records 8 B, k=3 16 B)
    assert bench.lookup_alg_wavefronts(estar, libs, T) == libs * (10 * (2 + 1 + 8 / 64) + 9 * (3 + 1 + 16 / 64))
    assert bench.rec_bytes(2) == 8 and bench.rec_bytes(4) == 48 and bench.rec_bytes(21) == 144
