"""Data formats: load_csv / read_skill_matrix / write_skill_matrix
against the reference's own outputs (tests/golden/io_cases.json, produced by
tests/golden/make_io_golden.py from /root/reference) and the oracle restatement.

CPU tests cover the native host reader (libcmb200's cmb_csv_header /
cmb_csv_body, loaded without a device); the GPU tests cover the formatter kernel."""

import json
from pathlib import Path

import numpy as np
import pytest

import crossmap_oracle as O
import paper_2105_12301_b200 as P
from paper_2105_12301_b200 import io as pio

CASES = json.loads((Path(__file__).parent / "golden" / "io_cases.json").read_text(encoding="utf-8"))


def _hex(rows):
    return [[float.fromhex(v) for v in r] for r in rows]


def _check(outcome, fn, text, tmp_path):
    p = tmp_path / "case.csv"
    p.write_bytes(text.encode("utf-8"))
    if "error" in outcome:
        with pytest.raises(P.CsvFormatError) as exc:
            fn(p)
        assert str(exc.value) == outcome["error"].replace("{path}", str(p))
        return None
    return fn(p)


@pytest.mark.parametrize("case", sorted(CASES["load_csv"]))
def test_load_csv_matches_reference(case, tmp_path):
    g = CASES["load_csv"][case]
    ds = _check(g, P.load_csv, g["text"], tmp_path)
    if ds is None:
        return
    assert ds.names == g["names"]
    want = np.array(_hex(g["values"]))
    got = np.array([s.values for s in ds])
    assert got.tobytes() == want.tobytes()  # bit-exact (std::from_chars vs float())


@pytest.mark.parametrize("case", sorted(CASES["read_skill_matrix"]))
def test_read_skill_matrix_matches_reference(case, tmp_path):
    g = CASES["read_skill_matrix"][case]
    m = _check(g, P.read_skill_matrix, g["text"], tmp_path)
    if m is None:
        return
    assert m.names == g["names"]
    want = np.array(_hex(g["rho"]))
    assert np.array_equal(np.isnan(m.rho), np.isnan(want))
    assert np.array_equal(np.nan_to_num(m.rho, nan=7.0), np.nan_to_num(want, nan=7.0))


def test_no_reference_code_in_the_reader():
    """The input side is the native reader (cmb_csv_header / cmb_csv_body); there
    is no restated reference algorithm to fall back to."""
    assert not any(hasattr(pio, n) for n in ("_load_csv_reference", "_read_skill_matrix_reference"))
    rng = np.random.default_rng(0)
    X = rng.standard_normal((300, 4)) * 10.0 ** rng.integers(-8, 8, (300, 4))
    ds = None
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "d.csv"
        p.write_text("a,b,c,d\n" + "".join(",".join(repr(float(v)) for v in row) + "\n" for row in X))
        ds = P.load_csv(p)
    assert np.array_equal(np.array([s.values for s in ds]).T, X)


def _fuzz_cell(rng, numeric_only=False, unit=False):
    kinds = ["num", "num", "num", "ws", "under", "exp", "inf", "nan", "quoted", "bad", "empty", "nbsp"]
    k = kinds[int(rng.integers(len(kinds)))] if not numeric_only else "num"
    v = float(rng.uniform(-1, 1)) if unit else float(rng.standard_normal() * 10.0 ** int(rng.integers(-5, 5)))
    if k == "num":
        return repr(v)
    if k == "ws":
        return " \t" + repr(v) + " "
    if k == "under":
        return ["1_000", "1__0", "_1", "1_", "1_0.2_5", "1e1_0", "1._5"][int(rng.integers(7))]
    if k == "exp":
        return ["1e400", "-1e-400", "2.5E-3", "+.5", "5.", ".", "1e", "e5"][int(rng.integers(8))]
    if k == "inf":
        return ["inf", "-Infinity", "+INF", "infinit"][int(rng.integers(4))]
    if k == "nan":
        return ["nan", "-NaN", "nan(1)", "NA"][int(rng.integers(4))]
    if k == "quoted":
        return '"' + repr(v) + '"' if rng.random() < 0.7 else '"1,5"'
    if k == "bad":
        return ["x", "0x10", "1 2", "--1", "(1)"][int(rng.integers(5))]
    if k == "nbsp":
        return "\u00a0" + repr(v) if rng.random() < 0.5 else "\u0661\u0662"
    return ""


def _fuzz_text(rng, label):
    ncol = int(rng.integers(1, 5))
    names = [f"c{j}" for j in range(ncol)]
    lines = [("," if label else "") + ",".join(names)]
    nrow = ncol if label else int(rng.integers(0, 6))
    for r in range(nrow):
        cells = [_fuzz_cell(rng, numeric_only=rng.random() < 0.6, unit=label) for _ in range(ncol)]
        if rng.random() < 0.1:
            cells = cells[:-1]
        lines.append(((names[r] + ",") if label else "") + ",".join(cells))
    if rng.random() < 0.1:
        lines.insert(int(rng.integers(1, len(lines) + 1)), "")
    eol = ["\n", "\r\n", "\r"][int(rng.integers(3))]
    return eol.join(lines) + (eol if rng.random() < 0.8 else "")


@pytest.mark.parametrize("label", [False, True])
def test_native_reader_matches_reference_semantics(label, tmp_path):
    """Fuzz of the grammar (quoting, blank lines, \\r / \\r\\n records, '_'
    separators, exponents, inf/nan spellings, Unicode digits and blanks, ragged
    rows) against the csv-module restatement of the reference readers."""
    rng = np.random.default_rng(11 + label)
    p = tmp_path / "f.csv"
    for case in range(400):
        text = _fuzz_text(rng, label)
        p.write_bytes(text.encode("utf-8"))
        oracle = O.read_skill_matrix_rows if label else O.load_csv_rows
        try:
            want = oracle(p)
            err = None
        except (O.CsvOracleError, O.OracleError, IndexError) as exc:
            want, err = None, (type(exc), str(exc))
        kinds = {P.CsvFormatError: O.CsvOracleError, P.ParameterError: O.OracleError, IndexError: IndexError}
        try:
            got = P.read_skill_matrix(p) if label else P.load_csv(p)
            gerr = None
        except tuple(kinds) as exc:
            got, gerr = None, (next(v for k, v in kinds.items() if isinstance(exc, k)), str(exc))
        assert gerr == err, (case, repr(text))
        if err is None:
            if label:
                assert got.names == want[0]
                assert np.array_equal(np.isnan(got.rho), np.isnan(want[1]))
                assert np.array_equal(np.nan_to_num(got.rho), np.nan_to_num(want[1])), (case, repr(text))
            else:
                assert got.names == want[0]
                vals = np.array([s.values for s in got]).T
                assert vals.tobytes() == np.array(want[1], dtype=np.float64).reshape(vals.shape).tobytes(), repr(text)


def test_npz_round_trip(tmp_path):
    rho = np.array([[1.0, -0.25], [np.nan, 0.5]])
    P.write_skill_matrix_npz(P.SkillMatrix(["x", "y"], rho), tmp_path / "m.npz")
    back = P.read_skill_matrix_npz(tmp_path / "m.npz")
    assert back.names == ["x", "y"] and np.array_equal(np.nan_to_num(back.rho), np.nan_to_num(rho))


def test_oracle_writer_pinned_to_reference_bytes():
    for g in CASES["write_skill_matrix"].values():
        assert O.skill_matrix_csv_bytes(g["names"], np.array(_hex(g["rho"]))) == g["bytes"].encode("utf-8")


# ---------------------------------------------------------------- GPU formatter
@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(CASES["write_skill_matrix"]))
def test_write_skill_matrix_bytes_match_reference(case, tmp_path):
    g = CASES["write_skill_matrix"][case]
    p = tmp_path / "m.csv"
    P.write_skill_matrix(P.SkillMatrix(g["names"], np.array(_hex(g["rho"]))), p)
    assert p.read_bytes() == g["bytes"].encode("utf-8")


@pytest.mark.gpu
def test_write_read_write_is_byte_stable_and_batched(tmp_path, monkeypatch):
    rng = np.random.default_rng(5)
    n = 700
    rho = rng.uniform(-1, 1, (n, n))
    rho[rng.random((n, n)) < 0.05] = np.nan
    rho[3, :] = rng.integers(-8, 9, n) / 16.0          # exact binary fractions: round-half-even ties
    rho[4, :] = -rng.uniform(0, 5e-7, n)              # "-0.000000"
    names = [f"n{i}" if i % 7 else f'odd,"{i}"' for i in range(n)]
    monkeypatch.setattr(pio, "_BATCH_BYTES", 64 * 1024)  # many formatting batches
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    P.write_skill_matrix(P.SkillMatrix(names, rho), a)
    assert a.read_bytes() == O.skill_matrix_csv_bytes(names, rho)
    P.write_skill_matrix(P.read_skill_matrix(a), b)
    assert a.read_bytes() == b.read_bytes()


@pytest.mark.gpu
def test_write_from_device_buffer(tmp_path):
    import torch
    rng = np.random.default_rng(9)
    n = 257
    rho32 = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    rho32[0, :5] = np.nan
    names = [f"s{i}" for i in range(n)]
    dev = torch.from_numpy(rho32).cuda()
    p = tmp_path / "d.csv"
    P.write_skill_matrix_device(dev.data_ptr(), n, n, names, p, float32=True)
    assert p.read_bytes() == O.skill_matrix_csv_bytes(names, rho32.astype(np.float64))
    d64 = torch.from_numpy(rho32.astype(np.float64)).cuda()
    q = tmp_path / "e.csv"
    P.write_skill_matrix_device(d64.data_ptr(), n, n, names, q, float32=False)
    assert q.read_bytes() == p.read_bytes()
