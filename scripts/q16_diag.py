"""Dump fp32 / fp16 / q16 lookup rho for the q16 parity case (analysis input)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_12301_b200 as P

est = np.load(sys.argv[1])["est"]
X = P.mixed_dataset(160, 700, seed=31)
X[5, :] = 0.25
out = {}
for mode in ("0", "1", "2"):
    os.environ["CMB_LOOKUP_FP16"] = mode
    out["m" + mode] = P.xmap(X.T, est, dtype=np.float32)
np.savez("gpurun_out/q16_diag.npz", **out)
print("ok")
