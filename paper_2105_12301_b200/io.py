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
rho already lives.  Input files are read by libcmb200's host CSV reader
(``cmb_csv_header`` / ``cmb_csv_body``): the csv module's excel dialect and
float()'s grammar in C++ (``std::from_chars``, correctly rounded like float()),
returning the position and text of the first invalid record or cell, from
which the reference's exact CsvFormatError messages are built here.
``write_skill_matrix_npz`` / ``read_skill_matrix_npz`` add the binary path for
matrices too large for text.
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


# ---------------------------------------------------------------- input (native reader)
_FIELD_LIMIT = 131072  # csv.field_size_limit() default, enforced by cmb_csv_*
_CSV_EMPTY, _CSV_WIDTH, _CSV_NOT_NUMERIC, _CSV_NON_FINITE, _CSV_BAD_CELL, _CSV_FIELD_LIMIT = 1, 2, 3, 4, 5, 6


def _raw(path: Path) -> bytes:
    """The file image; non-ASCII content must be valid UTF-8 (the reference opens
    with encoding="utf-8", so an invalid byte raises UnicodeDecodeError there too)."""
    raw = path.read_bytes()
    if np.count_nonzero(np.frombuffer(raw, dtype=np.uint8) >= 0x80):
        raw.decode("utf-8")
    return raw


def _header(raw: bytes, path: Path) -> tuple[list[str], int]:
    """Unquoted cells of the first record and the offset of the second
    (cmb_csv_header; the csv module's excel dialect).  Buffers are sized from a
    window that starts at the first line and doubles when the record (a quoted
    field with line breaks) runs past it, never from the whole file."""
    full = np.frombuffer(raw, dtype=np.uint8)
    nl = raw.find(b"\n")
    win = len(raw) if nl < 0 else nl + 1
    while True:
        view = full[:win] if win < full.size else full
        max_cells = int(np.count_nonzero(view == 44)) + 1
        text = np.empty(max(view.size, 1), dtype=np.uint8)
        spans = np.empty(2 * max_cells, dtype=np.int64)
        ncells, body = np.zeros(1, np.int64), np.zeros(1, np.int64)
        rc = nat.load().cmb_csv_header(nat.ptr(full if full.size else np.zeros(1, np.uint8)), len(raw),
                                       nat.ptr(text), text.size, nat.ptr(spans), max_cells, nat.ptr(ncells),
                                       nat.ptr(body))
        if rc != 7 or win >= full.size:  # 7 = CMB_CSV_CAPACITY: widen the window
            break
        win = min(full.size, 2 * win)
    if rc == _CSV_EMPTY:
        raise CsvFormatError(f"{path}: empty file")
    _raise_field_limit(rc)
    t = text.tobytes()
    cells = [t[spans[2 * c]:spans[2 * c] + spans[2 * c + 1]].decode("utf-8") for c in range(int(ncells[0]))]
    return cells, int(body[0])


def _raise_field_limit(rc: int) -> None:
    if rc == _CSV_FIELD_LIMIT:
        import csv
        raise csv.Error(f"field larger than field limit ({_FIELD_LIMIT})")
    if rc not in (0, _CSV_EMPTY, _CSV_WIDTH, _CSV_NOT_NUMERIC, _CSV_NON_FINITE, _CSV_BAD_CELL):
        raise CsvFormatError(f"CSV reader failed with status {rc}")


class _Body:
    """Records after the header through cmb_csv_body: values, row labels (mode 1),
    the cells left for Python's float() (non-ASCII), and the first error."""

    def __init__(self, raw: bytes, off: int, mode: int, ncols: int, cap_rows: int | None):
        buf = np.ascontiguousarray(np.frombuffer(raw, dtype=np.uint8)[off:])
        records = int(np.count_nonzero(buf == 10) + np.count_nonzero(buf == 13)) + 1
        cap = records if cap_rows is None else cap_rows
        self.values = np.full((max(cap, 1), max(ncols, 1)), np.nan)
        lspans = np.zeros((max(cap, 1) if mode == 1 else 1, 2), dtype=np.int64)
        ndef_cap = int(np.count_nonzero(buf >= 0x80)) + 1
        defer = np.zeros((ndef_cap, 4), dtype=np.int64)
        err = np.zeros(8, dtype=np.int64)
        err_text = np.empty(_FIELD_LIMIT + 1, dtype=np.uint8)
        nrows, ndef = np.zeros(1, np.int64), np.zeros(1, np.int64)
        bptr = nat.ptr(buf) if buf.size else nat.ptr(np.zeros(1, np.uint8))
        # row labels (mode 1) and the text of non-ASCII cells: small buffers that
        # grow (the pass is re-run) only if a file needs more
        lab_cap = min(buf.size, 1 << 22) if mode == 1 else 1
        txt_cap = min(buf.size, 1 << 20) if ndef_cap > 1 else 1
        while True:
            labels = np.empty(max(lab_cap, 1), dtype=np.uint8)
            dtext = np.empty(max(txt_cap, 1), dtype=np.uint8)
            self.rc = nat.load().cmb_csv_body(bptr, buf.size, mode, ncols, nat.ptr(self.values), cap,
                                              nat.ptr(nrows), nat.ptr(labels), labels.size, nat.ptr(lspans),
                                              nat.ptr(defer), ndef_cap, nat.ptr(dtext), dtext.size, nat.ptr(ndef),
                                              nat.ptr(err_text), err_text.size, nat.ptr(err))
            if self.rc != 7 or (lab_cap >= buf.size and txt_cap >= buf.size):  # 7: a buffer was too small
                break
            lab_cap = min(buf.size, 4 * lab_cap) if mode == 1 else 1
            txt_cap = min(buf.size, 4 * txt_cap) if ndef_cap > 1 else 1
        _raise_field_limit(self.rc)
        self.nrows = int(nrows[0])
        self.err_row, self.err_col, self.err_cells = int(err[1]), int(err[2]), int(err[3])
        self.err_text = err_text[: int(err[4])].tobytes().decode("utf-8", errors="surrogateescape")
        dt = dtext.tobytes() if int(ndef[0]) else b""
        self.deferred = [(int(r), int(c)) for r, c, _, _ in defer[: int(ndef[0])]]
        self.deferred_text = [dt[o:o + n].decode("utf-8") for _, _, o, n in defer[: int(ndef[0])]]
        lb = labels.tobytes() if mode == 1 else b""
        self.labels = [lb[a:a + b].decode("utf-8") for a, b in lspans[: min(self.nrows, cap)]] if mode == 1 else []


def load_csv(path) -> Dataset:
    """Parse a columns-as-series CSV into a Dataset (io.py:25-61): the native
    reader tokenises and converts, errors carry the reference's messages."""
    path = Path(path)
    raw = _raw(path)
    cells, off = _header(raw, path)
    names = [c.strip() for c in cells]
    if any(not n for n in names):
        raise CsvFormatError(f"{path}: blank column name in header")
    seen: dict[str, int] = {}
    for n in names:
        seen[n] = seen.get(n, 0) + 1
    dup = sorted(n for n, c in seen.items() if c > 1)
    if dup:
        raise CsvFormatError(f"{path}: duplicate column names: {dup}")
    b = _Body(raw, off, 0, len(names), None)
    for (r, c), text in zip(b.deferred, b.deferred_text):
        where = f"{path}: row {r + 2}, column {names[c]!r}"
        try:
            v = float(text)
        except ValueError:
            raise CsvFormatError(f"{where}: not numeric: {text.strip()!r}") from None
        if not math.isfinite(v):
            raise CsvFormatError(f"{where}: non-finite value {text.strip()!r}")
        b.values[r, c] = v
    if b.rc == _CSV_WIDTH:
        raise CsvFormatError(f"{path}: row {b.err_row + 2} has {b.err_cells} cells, expected {len(names)}")
    if b.rc in (_CSV_NOT_NUMERIC, _CSV_NON_FINITE):
        what = "not numeric:" if b.rc == _CSV_NOT_NUMERIC else "non-finite value"
        raise CsvFormatError(f"{path}: row {b.err_row + 2}, column {names[b.err_col]!r}: "
                             f"{what} {b.err_text.strip()!r}")
    if not names:
        raise IndexError("list index out of range")  # the reference indexes columns[0] of none
    if b.nrows == 0:
        raise CsvFormatError(f"{path}: no data rows")
    values = b.values[: b.nrows]
    return Dataset(tuple(TimeSeries(values[:, j], name) for j, name in enumerate(names)))


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
    """Inverse of write_skill_matrix, at six-decimal precision (io.py:81-110),
    through the native reader."""
    path = Path(path)
    raw = _raw(path)
    header, off = _header(raw, path)
    names = header[1:]
    if not names:
        raise CsvFormatError(f"{path}: no target columns in header")
    n = len(names)
    b = _Body(raw, off, 1, n, n)
    for (r, c), text in zip(b.deferred, b.deferred_text):
        try:
            v = float(text)
        except ValueError:
            raise CsvFormatError(f"{path}: row {r + 2}, column {names[c]!r}: bad cell {text!r}") from None
        b.values[r, c] = v
    if b.rc == _CSV_WIDTH:
        raise CsvFormatError(f"{path}: row {b.err_row + 2} has {b.err_cells} cells, expected {n + 1}")
    if b.rc == _CSV_BAD_CELL:
        raise CsvFormatError(f"{path}: row {b.err_row + 2}, column {names[b.err_col]!r}: bad cell {b.err_text!r}")
    if b.nrows != n or b.labels != names:
        raise CsvFormatError(f"{path}: library rows do not match target columns")
    return SkillMatrix(names, b.values[:n, :n].copy())


# ---------------------------------------------------------------- binary path
def write_skill_matrix_npz(matrix: SkillMatrix, path) -> None:
    """Binary companion of write_skill_matrix: names and float64 rho in an .npz."""
    np.savez(Path(path), names=np.array(list(matrix.names), dtype=object),
             rho=np.asarray(matrix.rho, dtype=np.float64))


def read_skill_matrix_npz(path) -> SkillMatrix:
    with np.load(Path(path), allow_pickle=True) as z:
        return SkillMatrix([str(s) for s in z["names"]], np.array(z["rho"]))
