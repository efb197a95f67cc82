"""Data-format throughput: GPU skill-matrix CSV writer vs the
reference algorithm (csv module + f"{v:.6f}", restated in the oracle) and the
native CSV parser vs the csv-module parse.  python scripts/bench_io.py [N]"""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import numpy as np
import torch

import crossmap_oracle as O
import paper_2105_12301_b200 as P
from paper_2105_12301_b200 import io as pio

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
rng = np.random.default_rng(0)
rho = torch.empty((N, N), dtype=torch.float32, device="cuda").uniform_(-1, 1)
names = [f"s{i}" for i in range(N)]
with open(os.devnull, "wb") as fh:
    pio._write_rows(fh, rho.data_ptr(), True, True, 1024, N, names[:1024])  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nbytes = pio._write_rows(fh, rho.data_ptr(), True, True, N, N, names)
    el = time.perf_counter() - t0
cells = N * N
sample = rho[:64].cpu().numpy().astype(np.float64)
t0 = time.perf_counter()
O.skill_matrix_csv_bytes(names[:64], np.pad(sample, ((0, 0), (0, 0)))[:, :N]) if False else None
import csv, io as _io, math  # noqa: E401
buf = _io.StringIO(newline="")
w = csv.writer(buf)
for i in range(64):
    w.writerow([names[i]] + ["NA" if not math.isfinite(v) else f"{v:.6f}" for v in sample[i]])
el_ref = time.perf_counter() - t0
# parser: 1,024 series x 1,450 samples
X = P.mixed_dataset(1024, 1450, seed=2105)
with tempfile.TemporaryDirectory() as d:
    p = Path(d) / "x.csv"
    p.write_text(",".join(f"s{i}" for i in range(1024)) + "\n" +
                 "".join(",".join(repr(float(v)) for v in row) + "\n" for row in X.T))
    t0 = time.perf_counter(); P.load_csv(p); el_parse = time.perf_counter() - t0
    # the reference algorithm, as restated in the oracle (csv module + float())
    t0 = time.perf_counter(); O.load_csv_rows(p); el_parse_ref = time.perf_counter() - t0
    mb = p.stat().st_size / 1e6
print(json.dumps({
    "write_skill_matrix": {"N": N, "cells_per_s": cells / el, "text_GB_per_s": nbytes / el / 1e9,
                           "text_bytes": nbytes, "reference_cells_per_s": 64 * N / el_ref,
                           "speedup": (cells / el) / (64 * N / el_ref)},
    "load_csv": {"MB": mb, "native_MB_per_s": mb / el_parse, "reference_MB_per_s": mb / el_parse_ref,
                 "speedup": el_parse_ref / el_parse},
}))
