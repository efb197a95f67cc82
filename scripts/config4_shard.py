"""Config 4 (BASELINE configs[3]): N = 100,000 x T = 10,000 all-to-all xmap
sharded over 8 B200.  One GPU runs rank 0's shard -- libraries [0, N/8) x all
N targets -- which is exactly one rank's work in the 8-GPU job (library-row
sharding, per-rank work identical up to the remainder).  Also times edim over
all N series (in the 8-GPU job each rank runs N/8 of them) and checks sampled
pairs against the CPU oracle.

python scripts/config4_shard.py [N] [T] [G]   ->  gpurun_out/config4_shard.json
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np
import torch

import paper_2105_12301_b200 as P
from paper_2105_12301_b200 import _native as nat
from paper_2105_12301_b200.distributed import native_shard, shard_bounds

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
T = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000
G = int(sys.argv[3]) if len(sys.argv) > 3 else 8

t0 = time.perf_counter()
X = P.mixed_dataset(N, T, seed=2105, dtype=np.float32)
t_gen = time.perf_counter() - t0
Xd = torch.from_numpy(X).cuda()
s = torch.cuda.current_stream().cuda_stream
rho_e = torch.empty((N, 20), dtype=torch.float64, device="cuda")
est_d = torch.empty(N, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
nat.call("cmb_edim_dev", 0, Xd.data_ptr(), N, T, T, 20, 1, 1, rho_e.data_ptr(), est_d.data_ptr(), s)
torch.cuda.synchronize()
t_edim = time.perf_counter() - t0
estar = est_d.cpu().numpy().astype(np.int32)
del rho_e

lo, hi = shard_bounds(N, G, 0)
slab = torch.empty((N, hi - lo), dtype=torch.float32, device="cuda")
stats = np.zeros(8)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
ev0.record()
native_shard(Xd, estar, 1, lo, hi, slab, stats, 0, s)
ev1.record()
torch.cuda.synchronize()
t_shard = ev0.elapsed_time(ev1) * 1e-3
valid = int(np.sum(estar > 0))
libs_valid = int(np.sum(estar[lo:hi] > 0))
pairs = libs_valid * valid

# oracle check: one library, one target per distinct E* (fp64 CPU oracle)
import crossmap_oracle as O  # noqa: E402
rng = np.random.default_rng(4)
lib = int(rng.choice(np.flatnonzero(estar[lo:hi] > 0))) + lo
tg = []
for e in np.unique(estar[estar > 0]):
    tg.append(int(rng.choice(np.flatnonzero(estar == e))))
series = {i: X[i].astype(np.float64) for i in [lib] + tg}
t0 = time.perf_counter()
sub = [series[i] for i in [lib] + tg]
sub_est = [int(estar[i]) for i in [lib] + tg]
ref, _ = O.xmap(sub, sub_est, 1, libraries=[0], workers=os.cpu_count())
t_oracle = time.perf_counter() - t0
got = slab[tg, lib - lo].cpu().numpy().astype(np.float64)
want = ref[0, 1:]
dev = float(np.nanmax(np.abs(got - want)))
out = {
    "workload": f"config 4 shard: xmap libraries [{lo}, {hi}) of N={N} x all targets, T={T} (rank 0 of {G})",
    "n_series": N, "T": T, "gpus_emulated": G, "data_gen_s": t_gen,
    "edim_all_series_s": t_edim, "edim_series_per_s": N / t_edim,
    "shard_s": t_shard, "tables_s": float(stats[0]), "lookup_s": float(stats[1]),
    "shard_pairs": pairs, "pairs_per_s_per_gpu": pairs / t_shard,
    "projected_8gpu_pairs_per_s": pairs / t_shard * G,
    "projected_8gpu_job_s": t_edim / G + t_shard,
    "estar_hist": np.bincount(estar, minlength=21).tolist(),
    "oracle_check": {"library": lib, "targets": tg, "E": [int(estar[i]) for i in tg],
                     "max_abs_rho_diff": dev, "nan_equal": bool(np.array_equal(np.isnan(got), np.isnan(want))),
                     "oracle_s": t_oracle},
}
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/config4_shard.json").write_text(json.dumps(out, indent=1))
print(json.dumps(out))
