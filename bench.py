#!/usr/bin/env python
"""bench.py — events/s of bulk histogram filling on B200 (BASELINE.json metric).

A "step" is one pass of the whole hot path over one batch: reset the histogram,
fill every event of the batch (FindBin, AddBinContent + sumw2, GetStats sums; one
fused kernel per launch), and for N>1 GPUs the exchange step (pack the partial
state, NCCL all-reduce SUM, unpack).  The default workload is BASELINE.json
configs[1] (C2): TH1D with 10,000 variable-width bins, 5e8 Gaussian events with
random weights per GPU (weak scaling: every rank fills its own 5e8-event shard
of the same seeded stream).  Inputs are generated on the host by bhgen (seeded,
synthetic) and copied to HBM before the timed region; they are 8 GB per GPU,
larger than the 126 MB L2, so no L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

Prints ONE JSON line on rank 0 (see DESIGN.md §Measurement for every key).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bhgen  # noqa: E402

METRIC = "events/sec filled at 1/2/4/8 B200 (device-resident & incl. H2D); % of HBM peak"
UNIT = "events/s"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def hbm_peak():
    p = measured_peaks()
    if "hbm_gbs" in p:
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config: str):
    """dram bytes per launch of the fill kernel from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(config)
    except Exception:
        return None


def workload_desc(wl) -> str:
    return {"C1": "C1: TH1D 100 fixed bins [0,1], uniform x, unit weights",
            "C1S": "C1-shape streamed: TH1D 100 fixed bins [0,1], 2^30 uniform events, unit weights",
            "C2": "C2: TH1D 10,000 variable-width bins, 5e8 Gaussian events, random weights",
            "C3": "C3: TH2D 1000x1000 fixed bins, 2e8 uniform events, unit weights",
            "C3W": "C3w: TH2D 1000x1000 fixed bins, 2e8 uniform events, random weights",
            "C4": "C4: TH3D 100^3 with flow, 2e8 Cauchy-peaked events, unit weights",
            "C4W": "C4w: TH3D 100^3 with flow, 2e8 Cauchy-peaked events, random weights"}.get(wl.name, wl.name)


def get_workload(name: str):
    name = name.upper()
    if name == "C1S":
        wl = bhgen.workload("C1", 1 << 30)
        wl.name = "C1S"
        return wl
    return bhgen.workload(name)


# ------------------------------------------------------------------ clocks (NVML, sampled in a thread)
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.ok = False
        self.samples = []
        self.reasons = 0
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.hdl = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.hdl, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.hdl, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.hdl)
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.ok:
            self._stop.clear()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()
            self._t = None

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        reasons = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU oracle timing (reference arm / cpu_baseline)
def time_oracle(wl, sample_events: int, repeats: int = 1):
    """Time the CPU oracle (as it stands, single thread) on events [0, sample) of the workload."""
    import oracle
    hist = wl.hists[0]
    cols = [wl.column(c, 0, sample_events) for c in hist.cols]
    w = wl.column(wl.wcol, 0, sample_events) if hist.weighted else None
    times = []
    for _ in range(repeats):
        h = oracle.OracleHist(oracle.oracle_axes(hist))
        t0 = time.perf_counter()
        h.fill(cols, w)
        times.append(time.perf_counter() - t0)
    return times


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl = get_workload(args.config)
    sample = min(wl.n_events, args.ref_sample)
    times = time_oracle(wl, sample, repeats=args.warmup + args.steps)
    timed = times[args.warmup:]
    sec = float(np.sum(timed))
    value = sample * len(timed) / sec
    cpu = {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
           "sample": f"events [0, {sample}) of the {wl.name} stream per step, single-thread C oracle "
                     f"(Neumaier sums), {len(timed)} timed steps"}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec / len(timed),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (bhgen seeded generator)",
            "config": {"workload": workload_desc(wl), "events_per_step": sample, "host_cores_used": 1},
            "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2401_13310_b200 as pkg
    from paper_2401_13310_b200.dist import allreduce_state

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("for --gpus N>1 launch with torchrun --nproc-per-node N")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    wl = get_workload(args.config)
    hist = wl.hists[0]
    N = wl.n_events
    start = rank * N           # weak scaling: this rank's shard of the seeded stream
    ncol = len(hist.cols) + (1 if hist.weighted else 0)

    # ---- inputs: generated on the host into pinned memory (also the e2e source), copied to HBM once
    host = [torch.empty(N, dtype=torch.float64).pin_memory() for _ in range(ncol)]
    for j, c in enumerate(hist.cols):
        wl.column_ptr(c, start, N, host[j].data_ptr())
    if hist.weighted:
        wl.column_ptr(wl.wcol, start, N, host[-1].data_ptr())
    devc = [t.to(dev, non_blocking=True) for t in host]
    torch.cuda.synchronize()
    coords = devc[:len(hist.cols)]
    w = devc[-1] if hist.weighted else None

    axes = hist.axes_spec()
    H = pkg.Histogram(axes, device=local, strategy={"auto": 0, "priv": 1, "global": 2, "cache": 3}[args.strategy])
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    packed = torch.empty(pkg.bh_packed_size(H.h), dtype=torch.float64, device=dev)
    cptrs = [c.data_ptr() for c in coords]
    wptr = None if w is None else w.data_ptr()
    fill_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]

    def step(i=None):
        pkg.bh_reset(H.h, sh)
        if i is not None:
            fill_ev[i][0].record(stream)
        pkg.bh_fill(H.h, N, cptrs, wptr, sh)
        if i is not None:
            fill_ev[i][1].record(stream)
        if world > 1:
            allreduce_state(H, packed)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = ClockSampler(local)
    clk.start()
    l0 = pkg.bh_launch_count(H.h)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(stream)
    for i in range(args.steps):
        step(i)
    t1.record(stream)
    torch.cuda.synchronize()
    clk.stop()
    launches = pkg.bh_launch_count(H.h) - l0
    ms = t0.elapsed_time(t1)
    fill_ms = [a.elapsed_time(b) for a, b in fill_ev]
    if world > 1:
        m = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        ms = float(m.item())
        dist.barrier()
    total_events = N * world * args.steps
    value = total_events / (ms * 1e-3)

    # ---- end to end through the public API: pinned host columns -> H2D (in the timed region) -> fill -> D2H read
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    host_c = host[:len(hist.cols)]
    host_w = host[-1] if hist.weighted else None

    def e2e_step():
        H.reset()
        H.fill_host(host_c, host_w)
        if world > 1:
            allreduce_state(H, packed)
        return H.read()

    e2e_step()   # warm-up (staging buffers, copy stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk2 = ClockSampler(local)
    clk2.start()
    te = time.perf_counter()
    for _ in range(e2e_steps):
        res = e2e_step()
    e2e_s = time.perf_counter() - te
    clk2.stop()
    if world > 1:
        m = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        e2e_s = float(m.item())
    assert res["entries"] == N * world, res["entries"]
    e2e_value = N * world * e2e_steps / e2e_s
    h2d = 8 * N * ncol
    d2h = 8 * pkg.bh_packed_size(H.h)

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = min(N, args.cpu_sample)
        ts = time_oracle(wl, sample, repeats=1)
        cpu = {"value": sample / ts[0], "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"events [0, {sample}) of the {wl.name} stream, single-thread C oracle (Neumaier sums)"}

    if rank == 0:
        peak, peak_src = hbm_peak()
        bpe = wl.bytes_per_event
        fill_avg = float(np.mean(fill_ms))
        achieved = bpe * N / (fill_avg * 1e-3) / 1e9
        traffic = ncu_traffic(wl.name)
        strat = {0: "auto", 1: "priv", 2: "global", 3: "cache"}[H.strategy(hist.weighted)]
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (bhgen seeded generator, host-generated)",
            "config": {"workload": workload_desc(wl), "events_per_gpu": N, "total_bins": H.nbins_total,
                       "weighted": hist.weighted, "fill_strategy": strat,
                       "l2": f"inputs {bpe * N / 2**30:.1f} GiB/GPU >> 126 MB L2 (no flush needed)",
                       "parallelism": f"dp{world}: events sharded, NCCL all-reduce of packed bins+stats"
                       if world > 1 else "single GPU"},
            "pct_hbm_peak": 100.0 * bpe * value / world / 1e9 / peak,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "kernel": f"k_fill ({strat})", "launch_ms": fill_avg,
                         "algorithmic_bytes_per_launch": bpe * N, "peak_source": peak_src},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps, "pcie_gbs": h2d * world * e2e_steps / e2e_s / 1e9 / world,
                    "clocks": clk2.summary()},
            "gpu_launches": launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    H.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2", help="C1, C1S, C2 (default), C3, C3W, C4, C4W")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--strategy", default="auto", choices=["auto", "priv", "global", "cache"])
    ap.add_argument("--cpu-sample", type=int, default=50_000_000)
    ap.add_argument("--ref-sample", type=int, default=1 << 23)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
