"""CSV ingestion and skill-matrix serialization (reference pkg/src/crossmap/io.py).

Same functions, layouts and CsvFormatError messages as the reference:

* ``load_csv`` (io.py:25-61): header row of unique column names, one time
  step per row, every column a series.
* ``write_skill_matrix`` (io.py:70-78): target names across the header,
  library names down the first column, cells f"{v:.6f}" or "NA", csv.writer's
  "\\r\\n" terminator -- a write/read/write cycle is byte-stable.
* ``read_skill_matrix`` (io.py:81-110): the inverse at six-decimal precision.

B200 path.  The cell text of a skill matrix is produced on the GPU
(``cmb_format_skill_csv``: exact round-half-even "%.6f" from the float64
bits, csrc/io.cu) in row batches, from host arrays or straight from a device
buffer (``write_skill_matrix_device``, e.g. the target-major output of the
sharded cross map), so at N = 53,053 the 28 GB of text is formatted where
rho already lives.  Numeric CSV bodies are parsed in C++ (``std::from_chars``,
correctly rounded like Python's float).  The reference's own csv-module
algorithm (restated below) handles text outside that fast grammar -- quoted
fields, '_' digit separators -- and every invalid file, so errors carry the
reference's exact messages.  ``write_skill_matrix_npz`` / ``read_skill_matrix_npz``
add the binary path for matrices too large for text.
"""

from __future__ import annotations

import csv
import io as _io
import math
from pathlib import Path

import numpy as np

from . import _native as nat
from .embedding import Dataset, TimeSeries
from .errors import CsvFormatError
from .pairwise import SkillMatrix

_NA = "NA"
_BATCH_BYTES = 1 << 30  # text per GPU formatting batch


# ---------------------------------------------------------------- reference algorithm
def _load_csv_reference(path: Path) -> Dataset:
    """io.py:25-61 restated: the csv-module parse with the reference's checks."""
    with path.open(newline="", encoding="utf-8") as handle:
        reader = csv.reader(handle)
        try:
            header = next(reader)
        except StopIteration:
            raise CsvFormatError(f"{path}: empty file") from None
        names = [cell.strip() for cell in header]
        if any(not name for name in names):
            raise CsvFormatError(f"{path}: blank column name in header")
        duplicates = {n for n in names if names.count(n) > 1}
        if duplicates:
            raise CsvFormatError(f"{path}: duplicate column names: {sorted(duplicates)}")
        columns: list[list[float]] = [[] for _ in names]
        for row_number, row in enumerate(reader, start=2):
            if len(row) != len(names):
                raise CsvFormatError(
                    f"{path}: row {row_number} has {len(row)} cells, expected {len(names)}")
            for col, cell in enumerate(row):
                try:
                    value = float(cell)
                except ValueError:
                    raise CsvFormatError(
                        f"{path}: row {row_number}, column {names[col]!r}: "
                        f"not numeric: {cell.strip()!r}") from None
                if not math.isfinite(value):
                    raise CsvFormatError(
                        f"{path}: row {row_number}, column {names[col]!r}: "
                        f"non-finite value {cell.strip()!r}")
                columns[col].append(value)
    if not columns[0]:
        raise CsvFormatError(f"{path}: no data rows")
    return Dataset(tuple(TimeSeries(column, name) for column, name in zip(columns, names)))


def _read_skill_matrix_reference(path: Path) -> SkillMatrix:
    """io.py:81-110 restated."""
    with path.open(newline="", encoding="utf-8") as handle:
        reader = csv.reader(handle)
        try:
            header = next(reader)
        except StopIteration:
            raise CsvFormatError(f"{path}: empty file") from None
        names = header[1:]
        if not names:
            raise CsvFormatError(f"{path}: no target columns in header")
        rho = np.full((len(names), len(names)), np.nan)
        row_names = []
        for row_number, row in enumerate(reader, start=2):
            if len(row) != len(names) + 1:
                raise CsvFormatError(
                    f"{path}: row {row_number} has {len(row)} cells, expected {len(names) + 1}")
            row_names.append(row[0])
            for col, cell in enumerate(row[1:]):
                if cell == _NA:
                    continue
                try:
                    rho[row_number - 2, col] = float(cell)
                except (ValueError, IndexError):
                    raise CsvFormatError(
                        f"{path}: row {row_number}, column {names[col]!r}: bad cell {cell!r}") from None
    if row_names != names:
        raise CsvFormatError(f"{path}: library rows do not match target columns")
    return SkillMatrix(names, rho)


# ---------------------------------------------------------------- fast paths
def _split_header(raw: bytes):
    """(header cells, body offset) when the header needs no csv quoting, else None."""
    nl = raw.find(b"\n")
    if nl < 0:
        return None
    line = raw[:nl]
    if line.endswith(b"\r"):
        line = line[:-1]
    if b'"' in line or b"\r" in line:
        return None
    try:
        cells = line.decode("utf-8").split(",")
    except UnicodeDecodeError:
        return None
    return cells, nl + 1


def _parse_body(raw: bytes, start: int, ncols: int, label: bool, allow_na: bool, check_finite: bool,
                cap_rows: int | None = None):
    body = np.frombuffer(raw, dtype=np.uint8)[start:]
    cap = cap_rows if cap_rows is not None else int(np.count_nonzero(body == 10)) + 1
    out = np.empty((max(cap, 1), ncols), dtype=np.float64)
    labels = np.zeros((max(cap, 1), 2), dtype=np.int64) if label else None
    nrows = np.zeros(1, dtype=np.int64)
    body = np.ascontiguousarray(body)
    rc = nat.load().cmb_parse_numeric_csv(nat.ptr(body), body.size, ncols, int(label), int(allow_na),
                                          int(check_finite), nat.ptr(out), cap, nat.ptr(nrows),
                                          nat.ptr(labels))
    if rc != 0:
        return None
    n = int(nrows[0])
    return out[:n], (labels[:n] if label else None), body


def load_csv(path) -> Dataset:
    """Parse a columns-as-series CSV into a Dataset (io.py:25-61)."""
    path = Path(path)
    raw = path.read_bytes()
    head = _split_header(raw)
    if head is not None:
        names = [c.strip() for c in head[0]]
        if names and all(names) and len(set(names)) == len(names):
            parsed = _parse_body(raw, head[1], len(names), False, False, True)
            if parsed is not None and parsed[0].shape[0] > 0:
                values = parsed[0]
                return Dataset(tuple(TimeSeries(values[:, j], name) for j, name in enumerate(names)))
    return _load_csv_reference(path)  # quoting, '_' separators, or an invalid file


def _name_fields(names) -> list[bytes]:
    """Each name as csv.writer renders it inside a multi-field row."""
    out = []
    for s in names:
        buf = _io.StringIO()
        csv.writer(buf, lineterminator="").writerow([s, ""])
        out.append(buf.getvalue()[:-1].encode("utf-8"))
    return out


def _header_bytes(names) -> bytes:
    buf = _io.StringIO()
    csv.writer(buf, lineterminator="\r\n").writerow([""] + list(names))
    return buf.getvalue().encode("utf-8")


def _write_rows(handle, rho, on_device: bool, is_f32: bool, n: int, ld: int, names) -> int:
    fields = _name_fields(names)
    blob = np.frombuffer(b"".join(fields) or b"\0", dtype=np.uint8).copy()
    off = np.zeros(n + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(f) for f in fields])
    per_row_max = 10 * n + 2
    rows_per = max(1, _BATCH_BYTES // max(per_row_max, 1))
    esz = 4 if is_f32 else 8
    written = 0
    out_len = np.zeros(1, dtype=np.int64)
    for r0 in range(0, n, rows_per):
        nr = min(rows_per, n - r0)
        cap = int(nr * per_row_max + (off[r0 + nr] - off[r0]))
        out = np.empty(cap, dtype=np.uint8)
        base = (rho + r0 * ld * esz) if on_device else nat.ptr(rho[r0:])
        nat.call("cmb_format_skill_csv", nat.device(), base, int(on_device), int(is_f32), n, ld, r0, nr,
                 nat.ptr(blob), nat.ptr(off), nat.ptr(out), cap, nat.ptr(out_len))
        handle.write(memoryview(out)[: int(out_len[0])])
        written += int(out_len[0])
    return written


def write_skill_matrix(matrix: SkillMatrix, path) -> None:
    """Serialize a skill matrix (io.py:70-78); cells are formatted on the GPU."""
    path = Path(path)
    names = list(matrix.names)
    rho = np.ascontiguousarray(np.asarray(matrix.rho, dtype=np.float64))
    with path.open("wb") as handle:
        handle.write(_header_bytes(names))
        _write_rows(handle, rho, False, False, len(names), rho.shape[1], names)


def write_skill_matrix_device(rho_ptr: int, n: int, ld: int, names, path, float32: bool = True) -> None:
    """write_skill_matrix from a device buffer: rho[lib, tgt] (row = library, leading
    dimension ld elements, float32 or float64) at device address ``rho_ptr`` on the
    current CMB_DEVICE -- e.g. a library-major cross-map result -- without staging
    the matrix through host memory; only the text crosses PCIe."""
    path = Path(path)
    names = list(names)
    if len(names) != n:
        raise CsvFormatError(f"{len(names)} names for a {n}-row matrix")
    with path.open("wb") as handle:
        handle.write(_header_bytes(names))
        _write_rows(handle, int(rho_ptr), True, float32, n, ld, names)


def read_skill_matrix(path) -> SkillMatrix:
    """Inverse of write_skill_matrix, at six-decimal precision (io.py:81-110)."""
    path = Path(path)
    raw = path.read_bytes()
    head = _split_header(raw)
    if head is not None and len(head[0]) > 1:
        names = head[0][1:]
        parsed = _parse_body(raw, head[1], len(names), True, True, False, cap_rows=len(names))
        if parsed is not None:
            values, spans, body = parsed
            try:
                row_names = [bytes(body[a:a + b]).decode("utf-8") for a, b in spans]
            except UnicodeDecodeError:
                row_names = None
            if row_names is not None:
                if row_names != names:
                    raise CsvFormatError(f"{path}: library rows do not match target columns")
                rho = np.full((len(names), len(names)), np.nan)
                rho[: values.shape[0]] = values
                return SkillMatrix(names, rho)
    return _read_skill_matrix_reference(path)


# ---------------------------------------------------------------- binary path
def write_skill_matrix_npz(matrix: SkillMatrix, path) -> None:
    """Binary companion of write_skill_matrix: names and float64 rho in an .npz."""
    np.savez(Path(path), names=np.array(list(matrix.names), dtype=object),
             rho=np.asarray(matrix.rho, dtype=np.float64))


def read_skill_matrix_npz(path) -> SkillMatrix:
    with np.load(Path(path), allow_pickle=True) as z:
        return SkillMatrix([str(s) for s in z["names"]], np.array(z["rho"]))
