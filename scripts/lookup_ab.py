"""A/B of the cross-map lookup modes on one GPU (config-3-shaped data by default).

    python scripts/lookup_ab.py [N] [T] [modes...]

For each CMB_LOOKUP_ROT mode: one warm-up xmap, then two timed ones (tables /
lookup seconds from the library's CUDA events, fixup count); rho of every mode
is compared with the first mode's, and a few whole library rows with the CPU
oracle (the checker, oracle/crossmap_oracle.py).  Prints one JSON line.
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def main():
    import torch

    import paper_2105_12301_b200 as P
    from paper_2105_12301_b200 import _native as nat
    from paper_2105_12301_b200.distributed import xmap_sharded

    N = int(sys.argv[1]) if len(sys.argv) > 1 else 53053
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 1450
    modes = sys.argv[3:] or ["0", "1"]
    n_oracle = int(os.environ.get("AB_ORACLE_ROWS", "2"))
    X = P.mixed_dataset(N, T, seed=2105, dtype=np.float32)
    dev = torch.device("cuda", 0)
    Xd = torch.from_numpy(X).to(dev)
    rho_e = torch.empty((N, 20), dtype=torch.float64, device=dev)
    est_d = torch.empty(N, dtype=torch.int32, device=dev)
    nat.call("cmb_edim_dev", 0, Xd.data_ptr(), N, T, T, 20, 1, 1, rho_e.data_ptr(), est_d.data_ptr(),
             torch.cuda.current_stream().cuda_stream)
    estar = est_d.cpu().numpy().astype(np.int32)
    out = {"N": N, "T": T, "modes": {}}
    ref = None
    for m in modes:
        # mode "R" or "R:F": CMB_LOOKUP_ROT=R, CMB_FIX_RATIO=F
        rot, _, fr = m.partition(":")
        os.environ["CMB_LOOKUP_ROT"] = rot
        if fr:
            os.environ["CMB_FIX_RATIO"] = fr
        else:
            os.environ.pop("CMB_FIX_RATIO", None)
        st = np.zeros(8)
        xmap_sharded(Xd, estar, 1, stats=st)
        torch.cuda.synchronize()
        times = []
        for _ in range(2):
            t0 = time.perf_counter()
            rho = xmap_sharded(Xd, estar, 1, stats=st)
            torch.cuda.synchronize()
            times.append((time.perf_counter() - t0, st[0], st[1], st[6]))
        rec = {"wall_s": min(t[0] for t in times), "tables_s": min(t[1] for t in times),
               "lookup_s": min(t[2] for t in times), "fixups": times[-1][3]}
        if ref is None:
            ref = rho
        else:
            same_nan = bool(torch.equal(torch.isnan(ref), torch.isnan(rho)))
            d = torch.nan_to_num(torch.abs(ref - rho), nan=0.0)
            rec["max_abs_diff_vs_first"] = float(d.max())
            rec["nan_equal_vs_first"] = same_nan
            del d
        # oracle rows (rho_T[tgt][lib] slab: column = library)
        import crossmap_oracle as O
        if n_oracle == 0:
            out["modes"][m] = rec
            del rho
            print(json.dumps(out), flush=True)
            continue
        rng = np.random.default_rng(5)
        valid = np.flatnonzero(estar > 0)
        libs = [int(x) for x in rng.choice(valid, n_oracle, replace=False)]
        series = [X[i].astype(np.float64) for i in range(N)]
        t0 = time.perf_counter()
        orc = O.xmap_rows(series, [int(e) for e in estar], libs, 1, workers=os.cpu_count() or 1)
        worst = 0.0
        for r, lib in enumerate(libs):
            got = rho[:N, lib].cpu().numpy().astype(np.float64)
            exp = orc[r]
            ok = np.isnan(got) == np.isnan(exp)
            rec.setdefault("oracle_nan_equal", True)
            rec["oracle_nan_equal"] &= bool(ok.all())
            worst = max(worst, float(np.nanmax(np.abs(got - exp))))
        rec["oracle_rows"] = libs
        rec["oracle_max_abs"] = worst
        rec["oracle_s"] = time.perf_counter() - t0
        out["modes"][m] = rec
        del rho
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
