"""Lookup efficiency per neighbour count k: every target at one E*, N series of
the mixed recipe at T = 1,450, lookup seconds (library CUDA events) against the
shared-memory wavefront model of bench.py (lookup_alg_wavefronts).

    python scripts/lookup_per_k.py [N] [E ...]
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    import paper_2105_12301_b200 as P
    from paper_2105_12301_b200.distributed import xmap_sharded

    N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    Es = [int(e) for e in sys.argv[2:]] or [1, 2, 3, 4, 6, 8, 10, 12, 13, 16, 20]
    T = 1450
    X = P.mixed_dataset(N, T, seed=2105, dtype=np.float32)
    Xd = torch.from_numpy(X).cuda()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    ghz = 1.965
    out = []
    for E in Es:
        est = np.full(N, E, dtype=np.int32)
        st = np.zeros(8)
        xmap_sharded(Xd, est, 1, stats=st)
        xmap_sharded(Xd, est, 1, stats=st)
        t = float(st[1])
        wf = bench.lookup_alg_wavefronts(est, N, T)
        pp = float(N) * N * (T - E + 1)
        out.append({"E": E, "k": E + 1, "lookup_s": t, "point_pairs_per_s": pp / t,
                    "wavefront_frac": wf / t / (sms * ghz * 1e9), "fixups": float(st[6])})
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
