#!/usr/bin/env python
"""Benchmark: Monte Carlo exp(tA)v entry estimator (BASELINE.json metric:
path transitions/s and solved entries/s, % of the memory roofline).

A "step" is one full pass of the hot path over the configuration: every
requested entry estimated with W walkers (Philox walker, K3), inputs
resident in HBM.  Default workload: BASELINE.json config 5 (BA n=1e7, m=8,
v ~ U[-1,1), beta = 0.02, N = 512, W = 1e3, all 1e7 rows) — the largest
configuration, the one the north star's scaling target names.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5]
  python bench.py --impl reference ...   # the reference CPU path (oracle/_ref)

Multi-GPU (torchrun, one rank per GPU): rows are sharded in contiguous
blocks, every rank holds a full matrix replica, and each step ends with an
NCCL all-gather of the (value, std_error, jumps) slices.  Total work is the
fixed full vector, so scaling is "strong".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="target CPU time of the bounded reference sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ceiling", action="store_true")
    ap.add_argument("--kernel-only", action="store_true",
                    help="only the device timing loop (for ncu launch lists)")
    return ap.parse_args()


# ---------------------------------------------------------------- clocks
class NvmlSampler:
    """SM clock + throttle reasons sampled in-process through NVML during the
    timed region.  Spawning `nvidia-smi -lms 100` perturbed short kernels
    (5-25 ms per step of GPU idle, scripts/diag_steps.py), so sampling is
    in-process and every `interval` s (default 0.25)."""

    def __init__(self, device, interval=0.25):
        import pynvml

        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
        self.interval = interval
        self.samples = []
        self.stop_ev = threading.Event()

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        self.samples.append((sm, mx, rs))

    def _run(self):
        while not self.stop_ev.wait(self.interval):
            self._sample()

    def start(self):
        self._sample()  # NVML initialised and warm before the timed region
        self.samples.clear()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def stop(self):
        self.stop_ev.set()
        self.t.join(timeout=5)
        if not self.samples:
            self._sample()  # short region: one sample right at its end
        nv = self.nv
        names = {nv.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                 nv.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwPowerCap: "sw_power_cap",
                 nv.nvmlClocksEventReasonHwPowerBrakeSlowdown: "hw_power_brake"}
        reasons = sorted({n for _, _, r in self.samples for bit, n in names.items() if r & bit})
        return {"sm_mhz": statistics.median(s for s, _, _ in self.samples),
                "sm_max_mhz": max(m for _, m, _ in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": f"nvml every {self.interval}s"}


def make_sampler(device):
    try:
        return NvmlSampler(device)
    except Exception:
        return ClockSampler(device)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (NVML init) must not fall inside the timed
            # region: wait for its first sample
            t0 = time.time()
            while not self.lines and time.time() - t0 < 10 and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_from_profiles(cfg_idx):
    """dram bytes per launch of the walker kernel from the committed ncu
    --set full summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", f"ncu_full_cfg{cfg_idx}.json")
    try:
        with open(path) as f:
            return float(json.load(f)["dram_bytes_per_launch"])
    except Exception:
        return None


# ------------------------------------------------------- reference (CPU)
def cpu_reference_rate(cfg, seed, target_s, steps=1, warmup=0):
    """The reference's own entry_estimate (oracle/_ref, unmodified sources)
    on bounded row samples, row-parallel on all host cores: each thread calls
    entry_estimate(..., workers=1) on its rows (the faster of the
    two CPU modes).  Returns per-step (seconds, jumps, rows)."""
    import oracle

    ref = oracle.Ref()
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    rm = ref.matrix_from_csr(cfg.csr)
    setup_s = time.perf_counter() - t0
    rows_all = np.arange(cfg.csr.n, dtype=np.uint64) if cfg.rows is None else \
        cfg.rows.astype(np.uint64)
    # calibrate: one row per core
    rng = np.random.default_rng(1234)
    cal = rng.choice(rows_all, size=min(cores, len(rows_all)), replace=False)
    t = time.perf_counter()
    rm.entries(cfg.v, cal, cfg.beta, cfg.n_steps, cfg.walkers, 1, seed, workers=1,
               threads=cores)
    t_cal = max(time.perf_counter() - t, 1e-3)
    per_step = max(len(cal), int(len(cal) * max(1.0, target_s / t_cal)))
    per_step = min(per_step, len(rows_all))
    out = []
    for k in range(warmup + steps):
        sample = np.sort(rng.choice(rows_all, size=per_step, replace=False))
        t = time.perf_counter()
        _, _, j = rm.entries(cfg.v, sample, cfg.beta, cfg.n_steps, cfg.walkers, 1, seed + k,
                             workers=1, threads=cores)
        dt = time.perf_counter() - t
        if k >= warmup:
            out.append((dt, int(j.sum()), per_step))
    return out, cores, setup_s


def run_reference(args, cfg):
    steps, cores, setup_s = cpu_reference_rate(cfg, args.seed, args.cpu_seconds,
                                               steps=args.steps, warmup=args.warmup)
    secs = sum(s for s, _, _ in steps)
    jumps = sum(j for _, j, _ in steps)
    rows = sum(r for _, _, r in steps)
    value = jumps / secs
    sample = (f"{steps[0][2]} uniformly sampled rows per step x {cfg.walkers} walkers, "
              f"N={cfg.n_steps}, row-parallel entry_estimate(workers=1) on {cores} threads")
    line = {
        "impl": "reference", "metric": "path transitions/s", "value": value,
        "unit": "transitions/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / len(steps),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "entries_per_s": rows / secs,
        "config": {"workload": f"cfg{cfg.idx}_{cfg.name}", "n": cfg.csr.n, "nnz": cfg.csr.nnz,
                   "walkers_per_entry": cfg.walkers, "n_steps": cfg.n_steps, "beta": cfg.beta,
                   "splitting": "strang", "parallelism": f"{cores} host threads"},
        "cpu_baseline": {"value": value, "unit": "transitions/s", "cores": cores,
                         "kind": "reference", "sample": sample,
                         "matrix_setup_s": setup_s},
        "e2e": {"value": value, "unit": "transitions/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        import paper_1904_12759_b200 as pb

        lam = None
        if args.config == 2:  # beta = 0.5 / lambda_max from the reference's own stats()
            import oracle

            probe = pb.build_config(2, args.scale, lambda_max=1.0)
            lam = oracle.Ref().matrix_from_csr(probe.csr).lambda_max(100)
        cfg = pb.build_config(args.config, args.scale, lambda_max=lam)
        run_reference(args, cfg)
        return 0

    import torch

    import paper_1904_12759_b200 as pb
    from paper_1904_12759_b200.shard import gather_slices, shard_rows

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    t_setup = time.perf_counter()
    cfg = pb.build_config(args.config, args.scale)
    m = pb.split(cfg.csr, device=local)
    rows_all = np.arange(cfg.csr.n, dtype=np.uint32) if cfg.rows is None else cfg.rows
    rows = shard_rows(rows_all, rank, world)
    nrows = len(rows)
    setup_s = time.perf_counter() - t_setup

    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    v_d = torch.from_numpy(cfg.v).to(dev)
    rows_d = torch.from_numpy(rows.astype(np.int32)).to(dev)
    val = torch.empty(nrows, dtype=torch.float64, device=dev)
    se = torch.empty_like(val)
    jm = torch.empty(nrows, dtype=torch.int64, device=dev)
    jtot = torch.zeros((), dtype=torch.int64, device=dev)
    pb.set_v_device(m, v_d.data_ptr(), cfg.csr.n, sp)

    def params(step):
        return pb.PathParams(cfg.beta, cfg.n_steps, cfg.walkers, pb.Splitting.Strang,
                             args.seed + step, pb.Rng.PHILOX)

    K, Wm = args.steps, args.warmup
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(K)]

    def step(k, timed):
        if timed:
            evs[k][0].record(stream)
        pb.entries_device(m, rows_d.data_ptr(), nrows, params(k), val.data_ptr(),
                          se.data_ptr(), jm.data_ptr(), sp)
        if timed:
            evs[k][1].record(stream)
        jtot.add_(jm.sum())  # warm-up runs it too (lazy module load)
        if world > 1:
            gather_slices(val, se, jm, len(rows_all))

    for k in range(Wm):
        step(K + k, False)
    torch.cuda.synchronize()
    jtot.zero_()
    clocks = make_sampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    launches0 = pb.launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for k in range(K):
        step(k, True)
    t_end.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = pb.launch_count() - launches0
    clk = clocks.stop()
    elapsed_ms = t_start.elapsed_time(t_end)
    kern_ms = sum(a.elapsed_time(b) for a, b in evs) / K
    jumps = int(jtot.item())
    if dist:
        tt = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms = float(tt.item())
        jj = torch.tensor([jumps], dtype=torch.int64, device=dev)
        dist.all_reduce(jj)
        jumps = int(jj.item())
    secs = elapsed_ms / 1e3
    total_entries = len(rows_all) * K
    value = jumps / secs

    # roofline of the walker kernel on this rank (B_alg = 64 J + 48 E)
    j_step_rank = int(jtot.item()) / K
    balg = 64.0 * j_step_rank + 48.0 * nrows
    peak, peak_src = peak_hbm()
    achieved = balg / (kern_ms / 1e3) / 1e9
    traffic = traffic_from_profiles(cfg.idx) if args.scale == 1.0 else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "kernel": "entry_fast_kernel", "kernel_ms": kern_ms,
                "algorithmic_bytes_per_launch": balg,
                "bytes_model": "64 B per jump (neighbour-id sector + landing 32-B row record) "
                               "+ 48 B per entry (start record + value/SE)"}

    line = {
        "metric": "path transitions/s", "value": value, "unit": "transitions/s",
        "n_gpus": world, "steps": K, "warmup": Wm, "ms_per_step": elapsed_ms / K,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, SURVEY §8d)",
        "entries_per_s": total_entries / secs,
        "paths_per_s": total_entries * cfg.walkers / secs,
        # segment-steps (N per path) for comparison with PAPER.md:314
        "segment_steps_per_s": total_entries * cfg.walkers * cfg.n_steps / secs,
        "config": {"workload": f"cfg{cfg.idx}_{cfg.name}", "n": cfg.csr.n, "nnz": cfg.csr.nnz,
                   "entries": len(rows_all), "walkers_per_entry": cfg.walkers,
                   "n_steps": cfg.n_steps, "beta": cfg.beta, "splitting": "strang",
                   "rng": "philox4x32-10", "parallelism": f"rows sharded x{world}",
                   "l2": "inputs larger than L2 (no flush)" if cfg.csr.nnz * 4 + cfg.csr.n * 32 >
                   126e6 else "inputs L2-resident (no flush; cache-resident config)",
                   "setup_s": setup_s},
        "clocks": clk, "gpu_launches": launches, "roofline": roofline,
    }

    if rank == 0 and world == 1 and not args.kernel_only:
        if not args.no_ceiling:
            line["gather_ceiling"] = gather_ceiling(pb, m, cfg, rows_d, nrows, j_step_rank,
                                                    stream, sp)
            line["gather_ceiling"]["frac_of_ceiling"] = \
                (j_step_rank / (kern_ms / 1e3)) / line["gather_ceiling"]["transitions_per_s"]
        if not args.no_e2e:
            line["e2e"] = e2e(pb, m, cfg, rows, args, K, Wm)
        if not args.no_cpu_baseline:
            try:
                st, cores, ref_setup = cpu_reference_rate(cfg, args.seed, args.cpu_seconds)
                s, j, r = st[0]
                line["cpu_baseline"] = {
                    "value": j / s, "unit": "transitions/s", "cores": cores,
                    "kind": "reference",
                    "sample": f"{r} uniformly sampled rows x {cfg.walkers} walkers, "
                              f"row-parallel entry_estimate(workers=1), {s:.1f} s",
                    "entries_per_s": r / s, "matrix_setup_s": ref_setup}
            except Exception as e:  # reference library missing on this box
                line["cpu_baseline"] = {"value": None, "unit": "transitions/s", "cores": 0,
                                        "kind": "reference", "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def gather_ceiling(pb, m, cfg, rows_d, nrows, j_step, stream, sp):
    """K6: memory-only walker with the K3 access pattern and the same number
    of jumps (chains per row x chain length matched to K3's jumpers)."""
    import torch

    rate = pb.inputs.split_d(cfg.csr) - cfg.csr.diag
    rows = cfg.rows if cfg.rows is not None else np.arange(cfg.csr.n)
    jump_frac = float(np.mean(1.0 - np.exp(-rate[rows] * cfg.beta)))
    chains = max(1, int(round(cfg.walkers * jump_frac)))
    length = max(1, int(round(j_step / (nrows * chains))))
    for _ in range(2):
        pb.gather_ceiling_device(m, rows_d.data_ptr(), nrows, chains, length, sp)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    a.record(stream)
    for _ in range(reps):
        pb.gather_ceiling_device(m, rows_d.data_ptr(), nrows, chains, length, sp)
    b.record(stream)
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / reps / 1e3
    jumps = nrows * chains * length
    return {"transitions_per_s": jumps / t, "GBps": (64.0 * jumps + 48.0 * nrows) / t / 1e9,
            "chains_per_row": chains, "chain_len": length, "ms": t * 1e3}


def e2e(pb, m, cfg, rows, args, K, Wm):
    """Same metric through the public host API (C ABI entries call) with
    pinned host buffers: H2D of v (+ rows) and D2H of value/SE/jumps inside
    the timed region."""
    import torch

    n, nrows = cfg.csr.n, len(rows)
    v_h = torch.from_numpy(cfg.v).pin_memory().numpy()
    full = cfg.rows is None and nrows == n
    rows_h = None if full else torch.from_numpy(rows.astype(np.int32)).pin_memory().numpy() \
        .view(np.uint32)
    outs = (torch.empty(nrows, dtype=torch.float64).pin_memory().numpy(),
            torch.empty(nrows, dtype=torch.float64).pin_memory().numpy(),
            torch.empty(nrows, dtype=torch.int64).pin_memory().numpy().view(np.uint64))

    def call(k):
        p = pb.PathParams(cfg.beta, cfg.n_steps, cfg.walkers, pb.Splitting.Strang,
                          args.seed + k, pb.Rng.PHILOX)
        r = pb.entries_estimate(m, v_h, rows_h, p, out=outs)
        return r.total_jumps

    for k in range(Wm):
        call(k)
    torch.cuda.synchronize()
    t = time.perf_counter()
    jumps = 0
    for k in range(K):
        jumps += call(k)
    secs = time.perf_counter() - t
    return {"value": jumps / secs, "unit": "transitions/s",
            "h2d_bytes_per_step": n * 8 + (0 if full else nrows * 4),
            "d2h_bytes_per_step": nrows * 24, "entries_per_s": nrows * K / secs,
            "ms_per_step": 1e3 * secs / K, "api": "expmc_cuda_entries (host buffers, pinned)"}


if __name__ == "__main__":
    sys.exit(main())
