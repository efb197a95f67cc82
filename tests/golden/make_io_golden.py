"""Golden vectors for the data formats, produced by the
reference itself (/root/reference/pkg, importable in the build container):
load_csv / read_skill_matrix outcomes (values bit-exact as float.hex, or the
CsvFormatError message with the path replaced by {path}) and the exact bytes of
write_skill_matrix.  Run from the repo root:  python tests/golden/make_io_golden.py"""
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from crossmap import CsvFormatError, SkillMatrix, load_csv, read_skill_matrix, write_skill_matrix  # noqa: E402

LOAD = {
    "basic": "a,b\n1,2\n3,4\n",
    "single_column": "only\n1\n2\n3\n",
    "crlf": "x,y\r\n0.5,-1e-3\r\n2.25,1E5\r\n",
    "no_final_newline": "a,b\n1,2\n3,4",
    "spaces_signs": "a, b ,c\n +1.5 , -2 ,.5\n 7. ,+0, -0.0\n",
    "exponents_digits": "p,q\n1.0000000000000002,2.2250738585072014e-308\n123456789012345678,4.9e-324\n",
    "quoted": 'a,"b,c"\n"1",2\n3,"4"\n',
    "underscore": "a\n1_000\n2\n",
    "unicode_names": "tempér,δ\n1,2\n",
    "ragged": "a,b\n1,2\n3\n",
    "too_many": "a,b\n1,2,3\n",
    "blank_line": "a,b\n1,2\n\n3,4\n",
    "not_numeric": "a,b\n1,2\n3,oops\n",
    "nan_cell": "a,b\n1,2\nNaN,4\n",
    "inf_cell": "a,b\n1,inf\n",
    "duplicate": "a,a\n1,2\n",
    "blank_name": "a, \n1,2\n",
    "empty": "",
    "header_only": "a,b\n",
    "nan_paren": "a\nnan(1)\n",
}

READ = {
    "layout": ",a,b\r\na,1.000000,-0.123457\r\nb,NA,0.500000\r\n",
    "lf": ",a,b\na,0.1,0.2\nb,0.3,0.4\n",
    "mismatch": ",a,b\nb,0.1,0.2\na,0.3,0.4\n",
    "bad_cell": ",a,b\na,0.1,what\nb,0.3,0.4\n",
    "spaced_na": ",a,b\na, NA,0.2\nb,0.3,0.4\n",
    "short": ",a,b\na,0.1,0.2\n",
    "extra_row": ",a\na,0.5\nb,0.25\n",
    "no_targets": "x\n",
    "quoted_names": ',"a,1",b\n"a,1",0.5,NA\nb,-0.25,1.000000\n',
    "ragged": ",a,b\na,0.1\n",
}


def outcome(fn, text, tmp):
    p = Path(tmp) / "case.csv"
    p.write_bytes(text.encode("utf-8"))
    try:
        r = fn(p)
    except CsvFormatError as exc:
        return {"error": str(exc).replace(str(p), "{path}")}
    if hasattr(r, "series"):
        return {"names": r.names, "values": [[float(v).hex() for v in s.values] for s in r]}
    return {"names": r.names, "rho": [[float(v).hex() for v in row] for row in r.rho]}


def matrices():
    rng = np.random.default_rng(2105)
    ties = [2.0 ** -7, 3 * 2.0 ** -7, 2.0 ** -8, 2.0 ** -9, -(2.0 ** -7), 0.5, -0.5, 0.0625, 2.0 ** -20]
    special = [0.0, -0.0, 1.0, -1.0, -1e-9, 1e-9, 4.9e-324, -4.9e-324, 0.9999995, -0.9999995, 0.1234565,
               float("nan"), float("inf"), -float("inf"), 0.999999999, 5e-7, -5e-7, 1.5e-6]
    vals = np.array(ties + special + list(rng.uniform(-1, 1, 37)), dtype=np.float64)
    n = 8
    a = vals[: n * n].reshape(n, n)
    f32 = rng.uniform(-1, 1, (5, 5)).astype(np.float32).astype(np.float64)
    f32[1, 2] = np.nan
    yield "tricky", [f"s{i}" for i in range(n)], a
    yield "float32_widened", ["a", "b,c", 'q"uote', "", "δ"], f32
    yield "single", ["only"], np.array([[float("nan")]])


def main():
    out = {"load_csv": {}, "read_skill_matrix": {}, "write_skill_matrix": {}}
    with tempfile.TemporaryDirectory() as tmp:
        for k, t in LOAD.items():
            out["load_csv"][k] = {"text": t, **outcome(load_csv, t, tmp)}
        for k, t in READ.items():
            out["read_skill_matrix"][k] = {"text": t, **outcome(read_skill_matrix, t, tmp)}
        for k, names, rho in matrices():
            p = Path(tmp) / "m.csv"
            write_skill_matrix(SkillMatrix(names, rho), p)
            out["write_skill_matrix"][k] = {"names": names, "rho": [[float(v).hex() for v in r] for r in rho],
                                            "bytes": p.read_bytes().decode("utf-8")}
    Path(__file__).with_name("io_cases.json").write_text(json.dumps(out, indent=1, ensure_ascii=False))
    print("wrote", Path(__file__).with_name("io_cases.json"))


if __name__ == "__main__":
    main()
