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
def config_dict(idx, name, n, nnz, entries, walkers, n_steps, beta, gpus):
    """The workload description both arms print (identical dicts: the
    driver compares them).  beta is rounded to 10 significant digits so a
    last-bit difference between the two arms' power iterations (config 2)
    cannot split them."""
    big = nnz * 32 + n * 32 > 126e6
    return {"workload": f"cfg{idx}_{name}", "n": int(n), "nnz": int(nnz),
            "entries": int(entries), "walkers_per_entry": int(walkers),
            "n_steps": int(n_steps), "beta": float(f"{beta:.10g}"), "splitting": "strang",
            "parallelism": f"rows sharded x{gpus}",
            "l2": "inputs larger than L2 (no flush)" if big else
                  "inputs L2-resident (no flush; cache-resident config)"}


def cpu_reference_rate(matrix, v, rows_all, walkers, n_steps, beta, seed, target_s, steps=1,
                       warmup=0):
    """The reference's own entry_estimate (oracle/_ref, unmodified sources) on
    bounded row samples, row-parallel on all host cores: each thread calls
    entry_estimate(..., workers=1) on its rows (the faster of the
    two CPU modes).

    Also splits off the reference's O(n) per-call setup (node_factors,
    proj/src/estimator.cpp:41-45, :177-178, plus the thread pool of
    parallel_samples, :50-68): the first sample's rows are re-run with
    samples = 1 on the same threads; that time is the setup the sample paid,
    and jumps / (time - setup) is the path-only rate.  Returns
    (per-step [(seconds, jumps, rows)], cores, split dict)."""
    cores = os.cpu_count() or 1
    rng = np.random.default_rng(1234)
    cal = rng.choice(rows_all, size=min(cores, len(rows_all)), replace=False)
    t = time.perf_counter()
    matrix.entries(v, cal, beta, n_steps, walkers, 1, seed, workers=1, threads=cores)
    t_cal = max(time.perf_counter() - t, 1e-3)
    per_step = max(len(cal), int(len(cal) * max(1.0, target_s / t_cal)))
    per_step = min(per_step, len(rows_all))
    out, first = [], None
    for k in range(warmup + steps):
        sample = np.sort(rng.choice(rows_all, size=per_step, replace=False))
        if first is None:
            first = sample
        t = time.perf_counter()
        _, _, j = matrix.entries(v, sample, beta, n_steps, walkers, 1, seed + k, workers=1,
                                 threads=cores)
        dt = time.perf_counter() - t
        if k >= warmup:
            out.append((dt, int(j.sum()), per_step))
    t = time.perf_counter()
    _, _, j1 = matrix.entries(v, first, beta, n_steps, 1, 1, seed, workers=1, threads=cores)
    setup_s = time.perf_counter() - t
    s0, j0, r0 = out[0]
    # Path-only rate by differencing: the same few rows with samples = 1
    # (setup only) and with samples = F W, F raised until the walkers cost at
    # least half the setup — on config 5 the W = 1e3 walkers of a row are
    # ~0.01% of its call, far below the timing noise of (total - setup).
    # (strided: the sorted sample starts with the low-index hub rows of BA graphs)
    small = first[:: max(1, len(first) // (4 * cores))][: 4 * cores]
    t = time.perf_counter()
    matrix.entries(v, small, beta, n_steps, 1, 1, seed, workers=1, threads=cores)
    t_lo = time.perf_counter() - t
    F, t_hi, j_hi = 1, None, 0
    for F in (16, 256, 4096, 65536):
        t = time.perf_counter()
        _, _, jh = matrix.entries(v, small, beta, n_steps, walkers * F, 1, seed, workers=1,
                                  threads=cores)
        t_hi, j_hi = time.perf_counter() - t, int(jh.sum())
        if t_hi - t_lo >= 0.5 * t_lo or t_hi > 0.5 * target_s:
            break
    path_s = t_hi - t_lo
    ok = path_s > 0.2 * t_hi and j_hi > 0
    split = {"setup_per_call_s": setup_s * cores / r0,
             "setup_share": min(1.0, setup_s / s0),
             "path_only_value": j_hi / path_s if ok else None,
             "path_only_entries_per_s": (len(small) * F / path_s) if ok else None,
             "setup_how": f"same {r0} rows re-run with samples=1 (node_factors O(n) + "
                          f"thread pool per call), row-parallel on {cores} threads",
             "path_only_how": f"{len(small)} rows at samples = {F} x W minus the same rows at "
                              f"samples = 1 ({t_hi:.2f} s - {t_lo:.2f} s); entries/s counts "
                              f"W-walker entries"}
    return out, cores, split


def run_reference(args):
    """bench.py --impl reference: the unmodified reference (oracle/_ref) on
    inputs built by the reference and the oracle only (oracle/inputs.py) —
    the product library is never loaded in this process."""
    from oracle import inputs as oi

    t0 = time.perf_counter()
    rc = oi.build_config(args.config, args.scale)
    setup_s = time.perf_counter() - t0
    rows_all = np.arange(rc.n, dtype=np.uint64) if rc.rows is None else \
        rc.rows.astype(np.uint64)
    # each step a bounded sample, sized so that the whole --steps K --warmup W
    # run stays within a few minutes (~4 min of sampling)
    target_s = min(args.cpu_seconds, 240.0 / max(1, args.steps + args.warmup))
    steps, cores, split = cpu_reference_rate(rc.matrix, rc.v, rows_all, rc.walkers, rc.n_steps,
                                             rc.beta, args.seed, target_s,
                                             steps=args.steps, warmup=args.warmup)
    secs = sum(s for s, _, _ in steps)
    jumps = sum(j for _, j, _ in steps)
    rows = sum(r for _, _, r in steps)
    value = jumps / secs
    sample = (f"{steps[0][2]} uniformly sampled rows per step (of {rc.nrows}) x {rc.walkers} "
              f"walkers, N={rc.n_steps}, row-parallel entry_estimate(workers=1) on {cores} "
              f"threads")
    line = {
        "impl": "reference", "metric": "path transitions/s", "value": value,
        "unit": "transitions/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / len(steps),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, SURVEY §8d)", "entries_per_s": rows / secs,
        "config": config_dict(rc.idx, rc.name, rc.n, rc.nnz, rc.nrows, rc.walkers, rc.n_steps,
                              rc.beta, args.gpus),
        "cpu_baseline": {"value": value, "unit": "transitions/s", "cores": cores,
                         "kind": "reference", "sample": sample, "rng": "pcg32 (reference)",
                         "inputs_setup_s": setup_s,
                         "inputs": "reference generate() (BA) / oracle/inputs_gen.c (FD, WS, "
                                   "vectors, rows); no product library in this process",
                         **split},
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
        run_reference(args)
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
    if dist:
        # ranks share one CSR cache: rank 0 generates (BA 1e7 is sequential,
        # ~8 s), the others load the checksummed file
        os.environ.setdefault("EXPMC_CSR_CACHE", "/tmp/expmc_csr_cache")
        if rank == 0:
            cfg = pb.build_config(args.config, args.scale)
        dist.barrier()
        if rank != 0:
            cfg = pb.build_config(args.config, args.scale)
    else:
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

    contiguous = cfg.rows is None and nrows > 0  # a rank's block of all rows
    K, Wm = args.steps, args.warmup
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(K)]

    def step(k, timed):
        if timed:
            evs[k][0].record(stream)
        if contiguous:  # all rows / a rank's block of them: no row array on the device
            pb.entries_device_range(m, int(rows[0]), nrows, params(k), val.data_ptr(),
                                    se.data_ptr(), jm.data_ptr(), sp)
        else:
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
    roofline = make_roofline(cfg, j_step_rank, nrows, kern_ms, args.scale)

    line = {
        "metric": "path transitions/s", "value": value, "unit": "transitions/s",
        "n_gpus": world, "steps": K, "warmup": Wm, "ms_per_step": elapsed_ms / K,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, SURVEY §8d)",
        "entries_per_s": total_entries / secs,
        "paths_per_s": total_entries * cfg.walkers / secs,
        # segment-steps (N per path) for comparison with PAPER.md:314
        "segment_steps_per_s": total_entries * cfg.walkers * cfg.n_steps / secs,
        "config": config_dict(cfg.idx, cfg.name, cfg.csr.n, cfg.csr.nnz, len(rows_all),
                              cfg.walkers, cfg.n_steps, cfg.beta, world),
        "rng": "philox4x32-10", "setup_s": setup_s,
        "clocks": clk, "gpu_launches": launches, "roofline": roofline,
    }

    if not args.kernel_only:
        if rank == 0 and world == 1 and not args.no_ceiling:
            line["gather_ceiling"] = gather_ceiling(pb, m, cfg, rows_d, nrows, j_step_rank,
                                                    stream, sp)
            line["gather_ceiling"]["frac_of_ceiling"] = \
                (j_step_rank / (kern_ms / 1e3)) / line["gather_ceiling"]["transitions_per_s"]
        if not args.no_e2e:
            line["e2e"] = e2e(pb, m, cfg, rows, args, K, Wm, dist, world, len(rows_all))
        if not args.no_cpu_baseline:
            if rank == 0:
                line["cpu_baseline"] = cpu_baseline_leg(cfg, rows_all, args)
            if dist:
                dist.barrier()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def cpu_baseline_leg(cfg, rows_all, args):
    """The reference's entry_estimate on this box's host cores (rank 0 only),
    on a bounded row sample of the same workload."""
    try:
        import oracle

        t0 = time.perf_counter()
        rm = oracle.Ref().matrix_from_csr(cfg.csr)
        ref_setup = time.perf_counter() - t0
        st, cores, split = cpu_reference_rate(rm, cfg.v, rows_all.astype(np.uint64),
                                              cfg.walkers, cfg.n_steps, cfg.beta, args.seed,
                                              args.cpu_seconds)
        s, j, r = st[0]
        return {"value": j / s, "unit": "transitions/s", "cores": cores, "kind": "reference",
                "sample": f"{r} uniformly sampled rows x {cfg.walkers} walkers, "
                          f"row-parallel entry_estimate(workers=1), {s:.1f} s",
                "entries_per_s": r / s, "matrix_setup_s": ref_setup, **split}
    except Exception as e:  # reference library missing on this box
        return {"value": None, "unit": "transitions/s", "cores": 0, "kind": "reference",
                "sample": f"unavailable: {e}"}


def source_sha():
    """Hash of the kernel sources: ties an ncu capture to the code it measured."""
    import hashlib

    h = hashlib.sha256()
    d = os.path.join(ROOT, "paper_1904_12759_b200", "csrc")
    for f in sorted(os.listdir(d)):
        if f.endswith((".cu", ".cuh", ".cpp", ".h")):
            h.update(f.encode())
            with open(os.path.join(d, f), "rb") as fh:
                h.update(fh.read())
    return h.hexdigest()[:16]


def _load_json(*parts):
    try:
        with open(os.path.join(ROOT, *parts)) as f:
            return json.load(f)
    except Exception:
        return None


def make_roofline(cfg, jumps, entries, kern_ms, scale):
    """Roofline of the walker kernel (K3) for one launch.

    * achieved / frac: SURVEY §8d's algorithmic bytes, 64 B per jump
      (neighbour-id sector + landing row record) + 48 B per entry, over the
      kernel's CUDA-event time.  Config 5's walked set (5 GB) is HBM-bound:
      peak = measured copy bandwidth.  Configs 1-4 are served from L2 (93%+
      hits on config 4, everything on 1-3): peak = the measured L2
      random-gather ceiling (K6 on an L2-resident table, profiles/r02/
      l2_gather_peak.json), counted with the same 64 B per jump.
    * frac_design_bytes: the bytes this design actually has to move (one
      32-B fat Edge sector per jump + 48 B per entry) against HBM.
    * traffic / frac_dram_measured / sector_efficiency: from the committed
      ncu --set full capture of this config (profiles/r02/ncu_cfg<i>.json),
      with the source hash it was taken at (traffic_same_source)."""
    hbm, hbm_src = peak_hbm()
    secs = kern_ms / 1e3
    balg = 64.0 * jumps + 48.0 * entries
    bdes = 32.0 * jumps + 48.0 * entries
    l2 = _load_json("profiles", "r02", "l2_gather_peak.json")
    if cfg.idx == 5 or l2 is None:
        bound, peak, src = "hbm", hbm, hbm_src
    else:
        bound, peak = "l2", float(l2["gbs_model_64B"])
        src = f"measured L2 random-gather ceiling ({l2['how']})"
    achieved = balg / secs / 1e9
    r = {"bound": bound, "achieved": achieved, "peak": peak, "unit": "GB/s",
         "frac": achieved / peak, "peak_source": src, "kernel": "entry_walk_kernel",
         "kernel_ms": kern_ms, "algorithmic_bytes_per_launch": balg,
         "bytes_model": "64 B per jump (neighbour-id sector + landing 32-B row record) "
                        "+ 48 B per entry (start record + value/SE)",
         "design_bytes_per_launch": bdes,
         "frac_design_bytes": bdes / secs / 1e9 / hbm,
         "traffic": None}
    prof = _load_json("profiles", "r02", f"ncu_cfg{cfg.idx}.json") if scale == 1.0 else None
    if prof:
        tr = float(prof["dram_bytes_per_launch"])
        r["traffic"] = tr
        r["frac_dram_measured"] = tr / secs / 1e9 / hbm
        r["traffic_capture"] = prof.get("capture")
        r["traffic_same_source"] = prof.get("source_sha") == source_sha()
        sec = prof.get("l1tex_ld_sectors_per_launch")
        if sec:
            r["sector_efficiency"] = (32.0 * jumps + 40.0 * entries) / (32.0 * float(sec))
            r["sector_efficiency_def"] = ("useful load bytes (32 B Edge per jump + 32 B start "
                                          "record + 8 B rate per entry) / (l1tex global-load "
                                          "sectors x 32)")
        for k in ("l2_hit_rate", "l1_hit_rate", "issue_active", "warp_instructions"):
            if k in prof:
                r["ncu_" + k] = prof[k]
    return r


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


def e2e(pb, m, cfg, rows, args, K, Wm, dist, world, nrows_all):
    """Same metric through the public host API (C ABI entries call) with
    pinned host buffers: H2D of v (+ rows) and D2H of value/SE/jumps inside
    the timed region.  At N > 1 every rank calls it on its row shard (each
    rank writes its slice into its own pinned host buffers); the step time is
    the max over ranks, bracketed by barriers."""
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
    if dist:
        dist.barrier()
    t = time.perf_counter()
    jumps = 0
    for k in range(K):
        jumps += call(k)
    secs = time.perf_counter() - t
    if dist:
        dev = torch.device("cuda", torch.cuda.current_device())
        tt = torch.tensor([secs, float(jumps)], dtype=torch.float64, device=dev)
        mx = tt.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(tt)
        secs, jumps = float(mx[0].item()), int(tt[1].item())
    h2d = world * n * 8 + (0 if full else nrows_all * 4)
    return {"value": jumps / secs, "unit": "transitions/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": nrows_all * 24,
            "entries_per_s": nrows_all * K / secs, "ms_per_step": 1e3 * secs / K,
            "api": "expmc_cuda_entries (host buffers, pinned)" +
                   (f"; one call per rank on its row shard, max over {world} ranks"
                    if world > 1 else "")}


if __name__ == "__main__":
    sys.exit(main())
