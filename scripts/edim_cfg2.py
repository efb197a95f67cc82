"""Config 2 timing: edim E=1..20 on N synthetic series x T=10,000 (default N=1,024).
python scripts/edim_cfg2.py [N] [T]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2105_12301_b200 as P
from paper_2105_12301_b200 import _native as nat

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
T = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
X = P.mixed_dataset(N, T, seed=2105, dtype=np.float32)
Xd = torch.from_numpy(X).cuda()
rho = torch.empty((N, 20), dtype=torch.float64, device="cuda")
est = torch.empty(N, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def run():
    nat.call("cmb_edim_dev", 0, Xd.data_ptr(), N, T, T, 20, 1, 1, rho.data_ptr(), est.data_ptr(), s)
    torch.cuda.synchronize()
run()
t0 = time.perf_counter(); run(); el = time.perf_counter() - t0
e = est.cpu().numpy()
print(f"edim N={N} T={T}: {el:.3f} s  {N / el:.1f} series/s  E* hist {np.bincount(e, minlength=21).tolist()}")
