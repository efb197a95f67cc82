"""Benchmark: all-to-all xmap cross-map pairs/s on synthetic zebrafish-shaped data.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], the metric's config): N = 53,053 series x
T = 1,450 samples, the reference's 20-series mix tiled (seed 2105, float32),
per-series E* from GPU edim (E_max = 20, Tp = 1), then the N x N cross map
(Tp = 0).  One step = one full xmap over every ordered pair with X resident in
HBM (tables + lookup; for N > 1 also the NCCL broadcast of X and the gather of
rho slabs to rank 0).  X (308 MB) and rho (11.3 GB) exceed the 126 MB L2, so
no flush is needed between steps.

``--impl reference`` times the CPU oracle (oracle/crossmap_oracle.py, a
restatement of the reference's numpy algorithm; the reference is pure Python
and cannot ship to the GPU box) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "xmap cross-map pairs/sec (N×N, T=1450) at 1/2/4/8 B200; lookup HBM GB/s"
UNIT = "pairs/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--series", dest="n", type=int, default=53053)
    p.add_argument("--length", dest="t", type=int, default=1450)
    p.add_argument("--seed", type=int, default=2105)
    p.add_argument("--e-max", type=int, default=20)
    p.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU baseline sample budget")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--lookup-fp16", nargs="?", const="1", default=None,
                   help="also time the opt-in 16-bit-target lookup modes (CMB_LOOKUP_FP16=1 fp16, =2 q16 "
                        "fixed point; comma list) and report their rho deviation")
    return p.parse_args()


# ---------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def sm_clock_ghz(clk) -> float:
    """Median SM clock sampled during the timed region (GHz), else the max clock."""
    sm = clk.summary().get("sm_mhz") or clk.summary().get("sm_max_mhz") or 1965.0
    return float(sm) / 1e3


def measured_peak_hbm():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        return float(json.loads(f.read_text())["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def profiled_traffic():
    """dram bytes per lookup launch from the committed ncu --set full summary."""
    f = ROOT / "profiles" / "lookup_traffic.json"
    if f.exists():
        d = json.loads(f.read_text())
        return d.get("dram_bytes_per_launch"), d.get("alg_bytes_per_launch")
    return None, None


def lookup_alg_bytes(estar: np.ndarray, n_libs: int, T: int, tau: int = 1) -> float:
    """B_pair = 4 n_E + 8 n_E k / N_E + 4 per pair, summed over the
    pairs of one step on this rank (n_libs libraries x all defined targets)."""
    tot = 0.0
    for E in np.unique(estar[estar > 0]):
        NE = int(np.sum(estar == E))
        nE = T - (int(E) - 1) * tau
        k = int(E) + 1
        tot += n_libs * NE * (4.0 * nE + 4.0) + n_libs * 8.0 * nE * k
    return tot


def lookup_alg_wavefronts(estar: np.ndarray, n_libs: int, T: int, tau: int = 1) -> float:
    """Shared-memory wavefronts the lookup issues per step on this rank (the
    binding resource, K3): per embedded point of a (library, 32-target
    block) pair k gathers + the record's 8-byte broadcast loads (ceil(k/2) weight +
    ceil(k/4) row loads; one load in all for k = 2) + the observed-value load,
    shared by the two libraries a warp runs in lockstep (1/2 per pair).  The
    one-library form matched ncu l1tex__data_pipe_lsu_wavefronts_mem_shared
    within 2% (profiles/r01_lookup_ncu_summary.txt)."""
    tot = 0.0
    for E in np.unique(estar[estar > 0]):
        NE = int(np.sum(estar == E))
        nE = T - (int(E) - 1) * tau
        k = int(E) + 1
        # record broadcasts: k <= 3 stores k - 1 weights (cmb_common.cuh rec_*)
        rec = 1 if k == 2 else ((k - 1 if k == 3 else k) + 1) // 2 + (k + 3) // 4
        tot += n_libs * ((NE + 31) // 32) * nE * (k + rec + 0.5)
    return tot


def make_data(n, t, seed):
    from paper_2105_12301_b200.synthetic import mixed_dataset
    return mixed_dataset(n, t, seed=seed, dtype=np.float32)


# ---------------------------------------------------------------- CPU arm
def cpu_sample(X: np.ndarray, estar: np.ndarray, budget_s: float, workers: int):
    """Oracle xmap on whole library rows (all targets) until the budget is spent."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import crossmap_oracle as O
    series = [X[i].astype(np.float64) for i in range(X.shape[0])]
    valid = np.flatnonzero(estar > 0)
    rng = np.random.default_rng(0)
    libs = rng.permutation(valid)
    done_pairs = 0
    t0 = time.perf_counter()
    n_libs = 0
    for lib in libs:
        O.xmap(series, [int(e) for e in estar], 1, workers=workers, libraries=[int(lib)])
        done_pairs += valid.size
        n_libs += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    el = time.perf_counter() - t0
    return done_pairs / el, f"{n_libs} random libraries x all {valid.size} targets (oracle xmap rows)", el


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    X = make_data(args.n, args.t, args.seed)
    estar = cpu_estar(X, args)
    workers = os.cpu_count() or 1
    vals = []
    samples = ""
    for _ in range(args.warmup):
        cpu_sample(X, estar, min(3.0, args.cpu_seconds), workers)
    for _ in range(args.steps):
        v, samples, _ = cpu_sample(X, estar, args.cpu_seconds / max(1, args.steps), workers)
        vals.append(v)
    v = float(np.mean(vals))
    n_pairs = float(np.sum(estar > 0)) ** 2
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": n_pairs / v * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"xmap N={args.n} T={args.t} mixed seed {args.seed}, E* from edim",
                       "n_series": args.n, "T": args.t, "tau": 1, "Tp_xmap": 0, "l2": "inputs > L2"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "port",
                             "sample": samples},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_estar(X, args):
    """E* for the CPU arm: the GPU's edim when a device is present (the parity
    rule of SURVEY.md 8c compares xmap under the GPU's E*), else a cheap proxy."""
    try:
        import torch
        if torch.cuda.is_available():
            import paper_2105_12301_b200 as P
            est, _ = P.edim(X.T.astype(np.float64), args.e_max, 1, 1)
            return est
    except Exception:
        pass
    return (np.arange(X.shape[0]) % 5 + 1).astype(np.int32)


# ---------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2105_12301_b200 as P
    from paper_2105_12301_b200 import _native as nat
    from paper_2105_12301_b200.distributed import all_gather_rows, broadcast_, shard_bounds, xmap_sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; CMB_DIST_BACKEND=gloo lets ranks share a GPU (functional runs)
    backend = os.environ.get("CMB_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count() if backend == "gloo" else local
    torch.cuda.set_device(local)
    os.environ["CMB_DEVICE"] = str(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    N, T = args.n, args.t

    # ---- setup (untimed): data on rank 0, E* from device edim
    X_host = make_data(N, T, args.seed) if rank == 0 else np.empty((N, T), np.float32)
    Xd = torch.from_numpy(X_host).to(dev)
    if world > 1:
        broadcast_(Xd, src=0)
    rho_e = torch.empty((N, args.e_max), dtype=torch.float64, device=dev)
    est_d = torch.empty(N, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    # edim shards by series; every rank needs the full E* vector
    lo_s, hi_s = shard_bounds(N, world, rank)
    nat.call("cmb_edim_dev", local, Xd[lo_s:].data_ptr(), hi_s - lo_s, T, T, args.e_max, 1, 1,
             rho_e[lo_s:].data_ptr(), est_d[lo_s:].data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    t_edim = time.perf_counter() - t0
    if world > 1:
        est_d = all_gather_rows(est_d[lo_s:hi_s].contiguous(), N)
    estar = est_d.cpu().numpy().astype(np.int32)
    valid = int(np.sum(estar > 0))
    hist = {int(e): int(c) for e, c in zip(*np.unique(estar, return_counts=True))}

    stats = np.zeros(8)
    lo, hi = shard_bounds(N, world, rank)
    n_sms = torch.cuda.get_device_properties(dev).multi_processor_count

    def step():
        return xmap_sharded(Xd, estar, 1, stats=stats, broadcast=True)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    nat.diagnostics(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    look_s = []
    with ClockSampler(local) as clk:
        e0.record(s)
        for _ in range(args.steps):
            step()
            look_s.append(stats[1])
        e1.record(s)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    t_max = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        if backend == "gloo":
            th = t_max.cpu()
            dist.all_reduce(th, op=dist.ReduceOp.MAX)
            t_max = th
        else:
            dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms = float(t_max.item())
    diag = nat.diagnostics(local)
    pairs = float(valid) * float(valid)
    value = pairs / (ms * 1e-3)

    # roofline of the dominant kernel (lookup) from its CUDA-event time on the launching stream
    libs_rank = int(np.sum(estar[lo:hi] > 0))
    alg = lookup_alg_bytes(estar, libs_rank, T)
    t_look = float(np.median(look_s))
    achieved = alg / t_look / 1e9
    peak, peak_kind = measured_peak_hbm()
    traffic, traffic_alg = profiled_traffic()
    wf = lookup_alg_wavefronts(estar, libs_rank, T)

    # ---- opt-in fp16-target lookup mode: same workload, reported beside the fp32 headline
    t_tables_step, t_lookup_step = float(stats[0]), float(stats[1])
    fp16 = None
    if args.lookup_fp16 and world == 1:
        ref = step()
        fp16 = {}
        notes = {"1": "targets stored as fp16 scaled to [-1,1] (64 per block), fp32 accumulation",
                 "2": "targets stored as 16-bit fixed point v = rint(32767 (y - mid) / half range) (64 per block), "
                      "decoded exactly with PRMT + FADD2, fp32 accumulation about the library's first prediction; "
                      "not parity-valid on forced-E* constant libraries (2e-4, tests/test_gpu_parity.py)"}
        for mode in args.lookup_fp16.split(","):
            os.environ["CMB_LOOKUP_FP16"] = mode
            step()
            torch.cuda.synchronize()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(s)
            look16 = []
            for _ in range(args.steps):
                got = step()
                look16.append(stats[1])
            f1.record(s)
            torch.cuda.synchronize()
            os.environ.pop("CMB_LOOKUP_FP16", None)
            ms16 = f0.elapsed_time(f1) / args.steps
            t16 = float(np.median(look16))
            same_nan = bool(torch.equal(torch.isnan(ref), torch.isnan(got)))
            diff = torch.nan_to_num(torch.abs(ref - got), nan=0.0)
            dmax = float(diff.max())
            n_over = int((diff > 1e-4).sum())
            wt, wl = divmod(int(torch.argmax(diff)), diff.shape[1])  # slab is rho_T[tgt][lib]
            worst = {"lib": wl, "tgt": wt, "rho_fp32": float(ref[wt, wl]), "rho_mode": float(got[wt, wl]),
                     "E_tgt": int(estar[wt]), "E_lib": int(estar[wl])}
            fp16["fp16" if mode == "1" else "q16"] = {
                "env": f"CMB_LOOKUP_FP16={mode}", "value": pairs / (ms16 * 1e-3), "ms_per_step": ms16,
                "lookup_ms_per_step": t16 * 1e3, "roofline_frac_hbm": alg / t16 / 1e9 / peak,
                "max_abs_rho_diff_vs_fp32": dmax, "pairs_over_1e-4": n_over, "nan_pattern_equal": same_nan,
                "worst_pair": worst,
                "note": notes.get(mode, "") + "; opt-in, not the headline"}
            del got, diff
        del ref

    # ---- e2e through the public C ABI with host buffers (rank 0 drives N = 1)
    e2e = None
    if not args.no_e2e and world == 1:
        xp = torch.from_numpy(X_host).pin_memory()
        outp = torch.empty((N, N), dtype=torch.float32).pin_memory()
        st = np.zeros(8)
        est_c = np.ascontiguousarray(estar)

        def e2e_step():
            nat.call("cmb_xmap", local, xp.data_ptr(), N, T, nat.ptr(est_c), 1, outp.data_ptr(),
                     P.LAYOUT_TGT_MAJOR, nat.ptr(st))
            return float(outp[0, 0])

        for _ in range(max(1, args.warmup - 2)):
            e2e_step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        el = (time.perf_counter() - t0) / args.steps
        e2e = {"value": pairs / el, "unit": UNIT, "h2d_bytes_per_step": int(N * T * 4),
               "d2h_bytes_per_step": int(N * N * 4), "layout": "target-major (rho.T view)",
               "ms_per_step": el * 1e3}
        del outp, xp

    # ---- e2e at N > 1: X from pinned host memory on rank 0 (H2D), NCCL broadcast,
    #      sharded cross map, every rank's rho slab copied to its pinned host buffer
    #      (one PCIe link per GPU); wall time per step, max over ranks
    if not args.no_e2e and world > 1:
        xp = torch.from_numpy(X_host).pin_memory() if rank == 0 else None
        Xe = torch.empty((N, T), dtype=torch.float32, device=dev)
        host = {}

        def e2e_step():
            if rank == 0:
                Xe.copy_(xp, non_blocking=True)
            slab = xmap_sharded(Xe, estar, 1, broadcast=True, gather=False)
            if "slab" not in host:
                host["slab"] = torch.empty(slab.shape, dtype=slab.dtype).pin_memory()
            host["slab"].copy_(slab, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            return float(host["slab"][0, 0])

        for _ in range(max(1, args.warmup - 2)):
            e2e_step()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        el = (time.perf_counter() - t0) / args.steps
        dist.barrier()
        el_t = torch.tensor([el], dtype=torch.float64)
        if backend == "gloo":
            dist.all_reduce(el_t, op=dist.ReduceOp.MAX)
        else:
            el_d = el_t.to(dev)
            dist.all_reduce(el_d, op=dist.ReduceOp.MAX)
            el_t = el_d.cpu()
        el = float(el_t.item())
        d2h = int(host["slab"].numel() * 4) * world
        e2e = {"value": pairs / el, "unit": UNIT, "h2d_bytes_per_step": int(N * T * 4),
               "d2h_bytes_per_step": d2h, "layout": "per-rank target-major slabs (library shards)",
               "ms_per_step": el * 1e3}
        del host, Xe, xp

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, sample, el = cpu_sample(X_host, estar, args.cpu_seconds, os.cpu_count() or 1)
        cpu = {"value": v, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "port", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp32 (fp64 selection + skill)", "data": "synthetic",
            "config": {"workload": f"xmap N={N} T={T} (BASELINE configs[2]), mixed seed {args.seed}, "
                                   f"E* from GPU edim E_max={args.e_max} Tp=1",
                       "n_series": N, "T": T, "tau": 1, "Tp_xmap": 0, "parallelism": f"library rows x{world}",
                       "l2": "inputs larger than L2 (X 308 MB, rho 11.3 GB)", "defined_series": valid,
                       "estar_hist": hist},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "lookup_xmap_kernel", "peak_kind": peak_kind,
                         "alg_bytes_per_step": alg, "lookup_ms_per_step": t_look * 1e3},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": diag["kernel_launches"], "fp16_lookup_mode": fp16,
            "clocks": clk.summary(),
            "roofline_smem": {
                "bound": "shared-memory wavefronts (the lookup's binding resource)",
                "achieved": wf / t_look / 1e9, "unit": "G wavefronts/s",
                "peak": n_sms * sm_clock_ghz(clk), "frac": wf / t_look / 1e9 / (n_sms * sm_clock_ghz(clk)),
                "wavefronts_per_step": wf, "model": "1 wavefront/clk/SM; k gathers + record broadcasts + 1/2 "
                                                    "observed load (shared by a library pair) per point and 32 pairs"},
            "extra": {"edim_seconds": t_edim, "edim_series_per_s": N / t_edim,
                      "tables_ms_per_step": t_tables_step * 1e3, "lookup_ms_per_step": t_lookup_step * 1e3,
                      "exact_fallback_rows": diag["exact_fallback_rows"], "rows_checked": diag["rows_checked"]},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
