"""Multi-rank functional check under torchrun: sharded xmap (broadcast of X,
library-row shards, gather of rho slabs) equals the single-process result.
    CMB_DIST_BACKEND=gloo python -m torch.distributed.run --nproc-per-node 2 \\
        --master-addr 127.0.0.1 --master-port 29561 scripts/dist_check.py [N] [T]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import torch.distributed as dist

import paper_2105_12301_b200 as P
from paper_2105_12301_b200.distributed import assemble, xmap_sharded

N = int(sys.argv[1]) if len(sys.argv) > 1 else 300
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1450
backend = os.environ.get("CMB_DIST_BACKEND", "nccl")
local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
torch.cuda.set_device(local)
os.environ["CMB_DEVICE"] = str(local)
dist.init_process_group(backend)
rank, world = dist.get_rank(), dist.get_world_size()
X = P.mixed_dataset(N, T, seed=2105, dtype=np.float32)
est, _ = P.edim(X.T.astype(np.float64), 20, 1, 1)
Xd = torch.from_numpy(X).cuda() if rank == 0 else torch.zeros((N, T), dtype=torch.float32, device="cuda")
res = xmap_sharded(Xd, est, 1)
if rank == 0:
    rho = assemble(res, N, world)
    ref = P.xmap(X.T, est, dtype=np.float32)
    same_nan = np.array_equal(np.isnan(rho), np.isnan(ref))
    diff = float(np.nanmax(np.abs(rho - ref)))
    print(f"dist_check world={world} backend={backend} N={N}: nan pattern equal {same_nan}, max|diff| {diff:.3e}")
    assert same_nan and diff == 0.0
dist.destroy_process_group()
