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
            "C4W": "C4w: TH3D 100^3 with flow, 2e8 Cauchy-peaked events, random weights",
            "C1F": "C1-shape streamed in float32: TH1D 100 fixed bins [0,1], 2^30 uniform float32 events",
            "C2F": "C2 in float32: TH1D 10,000 variable-width bins, 5e8 Gaussian float32 events, float32 weights",
            "C5": "C5: 8 histograms (1D/2D mix) from 7 columns, 1.25e8 events/GPU (1e9 over 8 GPUs), "
                  "one bh_fill_multi call"}.get(wl.name, wl.name)


def get_workload(name: str):
    name = name.upper()
    if name == "C1S":
        wl = bhgen.workload("C1", 1 << 30)
        wl.name = "C1S"
        return wl
    if name in ("C1F", "C2F"):   # float32 input columns (NEXT-2)
        wl = get_workload("C1S" if name == "C1F" else "C2")
        wl.name = name
        wl.f32 = True
        return wl
    if name == "C5":             # 1e9 events over 8 GPUs: 1.25e8 per GPU
        return bhgen.workload("C5", 125_000_000)
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
    """Time the CPU oracle (as it stands, single thread) on events [0, sample) of the workload:
    every histogram of the workload is filled from its columns, one after the other."""
    import oracle
    need = sorted({c for h in wl.hists for c in h.cols} | ({wl.wcol} if wl.wcol is not None else set()))
    cols = {c: wl.column(c, 0, sample_events) for c in need}
    times = []
    for _ in range(repeats):
        hs = [oracle.OracleHist(oracle.oracle_axes(h)) for h in wl.hists]
        t0 = time.perf_counter()
        for o, h in zip(hs, wl.hists):
            o.fill([cols[c] for c in h.cols], cols[wl.wcol] if h.weighted else None)
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


_PAR = {}


def _oracle_shard(args):
    """Worker of time_oracle_parallel: the oracle on events [a, b) of the forked columns."""
    import oracle
    a, b = args
    wl, cols = _PAR["wl"], _PAR["cols"]
    for h in wl.hists:
        o = oracle.OracleHist(oracle.oracle_axes(h))
        o.fill([cols[c][a:b] for c in h.cols], cols[wl.wcol][a:b] if h.weighted else None)
    return b - a


def time_oracle_parallel(wl, sample_events: int, threads: int) -> float:
    """Wall time of the same oracle sharded over `threads` forked processes (contiguous
    event ranges, SURVEY.md §8(d)'s T-thread baseline); the merge of the partial states
    (one add per bin) is not included."""
    import multiprocessing as mp
    need = sorted({c for h in wl.hists for c in h.cols} | ({wl.wcol} if wl.wcol is not None else set()))
    _PAR["wl"], _PAR["cols"] = wl, {c: wl.column(c, 0, sample_events) for c in need}
    bounds = [((sample_events * r) // threads, (sample_events * (r + 1)) // threads) for r in range(threads)]
    with mp.get_context("fork").Pool(threads) as pool:
        pool.map(_oracle_shard, [(0, 1)] * threads)            # warm the workers
        t0 = time.perf_counter()
        pool.map(_oracle_shard, bounds)
        dt = time.perf_counter() - t0
    _PAR.clear()
    return dt


# ------------------------------------------------------------------ secondary rows (device-resident only)
def measure_secondary(name: str, steps: int, warmup: int, local: int) -> dict:
    """Device-resident events/s and roofline fraction of another config's fill kernel,
    same protocol as the headline (CUDA events around each bh_fill; inputs >> L2)."""
    import torch
    import paper_2401_13310_b200 as pkg
    name, _, strat_name = name.partition("+")      # e.g. "C3+sort": opt-in strategy
    strategy = {"": pkg.BH_STRATEGY_AUTO, "sort": pkg.BH_STRATEGY_SORT, "cache": pkg.BH_STRATEGY_CACHE,
                "global": pkg.BH_STRATEGY_GLOBAL, "priv": pkg.BH_STRATEGY_PRIV}[strat_name]
    wl = get_workload(name)
    h = wl.hists[0]
    N = wl.n_events
    f32 = getattr(wl, "f32", False)
    host = torch.empty(N, dtype=torch.float64).pin_memory()

    def dev_col(c):
        wl.column_ptr(c, 0, N, host.data_ptr())
        t = host.to(f"cuda:{local}")
        return t.float() if f32 else t
    cols = [dev_col(c) for c in h.cols]
    w = dev_col(wl.wcol) if h.weighted else None
    del host
    H = pkg.Histogram(h.axes_spec(), device=local, strategy=strategy)
    st = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(warmup + steps):
        H.reset()
        if i >= warmup:
            ev[i - warmup][0].record(st)
        if f32:
            H.fill_f32(cols, w)
        else:
            H.fill(cols, w)
        if i >= warmup:
            ev[i - warmup][1].record(st)
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    e2e = None
    if f32:    # end to end through bh_fill_host_f32: pinned host float32 columns, H2D inside
        hc = [c.cpu().pin_memory() for c in cols]
        hw = w.cpu().pin_memory() if w is not None else None
        H.fill_host_f32(hc, hw)
        H.reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        H.fill_host_f32(hc, hw)
        r = H.read()
        dt = time.perf_counter() - t0
        assert r["entries"] == N
        e2e = {"events_per_s": N / dt, "h2d_bytes_per_event": 4 * (len(hc) + (hw is not None)),
               "api": "bh_fill_host_f32"}
        del hc, hw
    peak, _ = hbm_peak()
    bpe = wl.bytes_per_event // (2 if f32 else 1)
    gbs = bpe * N / (ms * 1e-3) / 1e9
    strat = {1: "priv", 2: "global", 3: "cache", 5: "sort"}.get(H.strategy(h.weighted), "?")
    H.close()
    del cols, w
    torch.cuda.empty_cache()
    return {"workload": workload_desc(wl), "events": N, "bytes_per_event": bpe, "events_per_s": N / (ms * 1e-3),
            "fill_ms": ms,
            "achieved_gbs": gbs, "frac": gbs / peak, "fill_strategy": strat, "e2e": e2e}


def measure_bulk_regime(local: int, total: int = 1 << 25, bulk: int = 32768) -> dict:
    """The paper's own benchmark regime: TH1D with 1000 variable bins on
    [0,1] (random widths), uniform float64 events handed over in bulks of 32768 from host
    memory, end to end (H2D inside, steady clock, result read back once at the end,
    PAPER.md:129).  Rows: one bh_fill_host call per bulk from pinned bulk buffers (the
    RDataFrame pattern); the persistent bulk consumer (bh_bulk_fill per bulk, and
    bh_bulk_submit with up to 4 bulks in flight); and one bh_fill_host call over the whole
    array with the library's staging chunk swept (32768 ... 2^22 events)."""
    import torch
    import paper_2401_13310_b200 as pkg
    edges = bhgen.edges_random_widths(bhgen.seed_of(6, 15), 1000)
    host = torch.empty(total, dtype=torch.float64).pin_memory()
    bhgen.fill_ptr(bhgen.UNIFORM, bhgen.seed_of(6, 0), 0, total, 0.0, 1.0, host.data_ptr())
    bulks = [host[i:i + bulk] for i in range(0, total, bulk)]
    H = pkg.Histogram([edges], device=local)
    out = {"workload": f"TH1D 1000 variable bins, {total} uniform float64 events from pinned host memory, "
                       f"bulks of {bulk} (PAPER.md:241)", "events": total}

    def run(fn):
        fn()                                              # warm-up (staging buffers, tables)
        H.reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        r = H.read()
        dt = time.perf_counter() - t0
        assert r["entries"] == total
        return total / dt

    def per_bulk():
        for b in bulks:
            H.fill_host([b])
    pkg.bh_set_chunk(H.h, bulk)
    out["per_bulk_calls_events_per_s"] = run(per_bulk)

    # the persistent bulk consumer (bh_bulk_*): one resident kernel reads each bulk straight
    # from pinned host memory; per bulk no launch and no cudaMemcpy
    def consumer_sync():                                  # bh_bulk_fill: returns when consumed
        H.bulk_begin(False)
        for b in bulks:
            H.bulk_fill([b])
        H.bulk_end()

    def consumer_pipelined():                             # up to 4 bulks in flight
        H.bulk_begin(False)
        t = 0
        for b in bulks:
            t = H.bulk_submit([b])
        H.bulk_wait(t)
        H.bulk_end()
    for key, fn in (("persistent_consumer_per_bulk_events_per_s", consumer_sync),
                    ("persistent_consumer_pipelined_events_per_s", consumer_pipelined)):
        try:
            out[key] = run(fn)
        except pkg.BHistError as e:       # e.g. under a profiler that serializes kernel launches,
            out[key] = f"unavailable: {e}"    # the resident kernel never sees a bulk (times out)
            try:
                H.bulk_end()              # close the abandoned session (reports the timeout again)
            except pkg.BHistError:
                pass
    sweep = {}
    for chunk in (bulk, 1 << 18, 1 << 20, 1 << 22):
        pkg.bh_set_chunk(H.h, chunk)
        sweep[str(chunk)] = run(lambda: H.fill_host([host]))
    out["one_call_chunk_sweep_events_per_s"] = sweep
    H.close()
    return out


# ------------------------------------------------------------------ GPU arm
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2401_13310_b200 as pkg
    from paper_2401_13310_b200.dist import Exchange

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("for --gpus N>1 launch with torchrun --nproc-per-node N")
    local = local % torch.cuda.device_count()     # (tests: several gloo ranks may share one GPU)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.backend)

    wl = get_workload(args.config)
    if args.events:
        wl.n_events = args.events
    N = wl.n_events
    start = rank * N           # weak scaling: this rank's shard of the seeded stream
    hists = wl.hists
    used = sorted({c for h in hists for c in h.cols} | ({wl.wcol} if any(h.weighted for h in hists) else set()))
    slot = {c: j for j, c in enumerate(used)}

    # ---- inputs: generated on the host into pinned memory (also the e2e source), copied to HBM once
    host = [torch.empty(N, dtype=torch.float64).pin_memory() for _ in used]
    for c in used:
        wl.column_ptr(c, start, N, host[slot[c]].data_ptr())
    devc = [t.to(dev, non_blocking=True) for t in host]
    torch.cuda.synchronize()

    strat_code = {"auto": 0, "priv": 1, "global": 2, "cache": 3, "exact": 4, "sort": 5}[args.strategy]
    per_hist = dict(kv.split("=") for kv in args.hist_strategy.split(",") if kv)   # e.g. "6=sort"
    Hs = [pkg.Histogram(h.axes_spec(), device=local,
                        strategy={"auto": 0, "priv": 1, "global": 2, "cache": 3, "exact": 4, "sort": 5}[
                            per_hist.get(str(i), args.strategy)])
          for i, h in enumerate(hists)]
    multi = len(Hs) > 1
    if multi:
        pkg.bh_set_multi_mode(Hs[0].h, {"passes": pkg.BH_MULTI_PASSES, "one-pass": pkg.BH_MULTI_ONE_PASS}[args.multi_mode])
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    # the exchange step (N>1): ONE collective per step over the packed state of every histogram,
    # unit-weight histograms without their sum of w^2; reduce-to-root by default (only rank 0
    # reads the result), --exchange allreduce leaves the total on every rank
    xchg = Exchange(Hs, unit=[not h.weighted for h in hists], op=args.exchange) if world > 1 else None
    fill_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]

    def do_fill(cols):
        if multi:
            pkg.fill_multi(Hs, [[slot[c] for c in h.cols] for h in hists], [h.weighted for h in hists], cols,
                           cols[slot[wl.wcol]] if wl.wcol is not None else None, stream)
        else:
            h = hists[0]
            pkg.bh_fill(Hs[0].h, N, [cols[slot[c]].data_ptr() for c in h.cols],
                        cols[slot[wl.wcol]].data_ptr() if h.weighted else None, sh)

    def step(i=None):
        for H in Hs:
            pkg.bh_reset(H.h, sh)
        if i is not None:
            fill_ev[i][0].record(stream)
        do_fill(devc)
        if i is not None:
            fill_ev[i][1].record(stream)
        if xchg is not None:
            xchg(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = ClockSampler(local)
    clk.start()
    l0 = [pkg.bh_launch_count(H.h) for H in Hs]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(stream)
    for i in range(args.steps):
        step(i)
    t1.record(stream)
    while not t1.query():          # poll (releases the GIL) so the clock sampler keeps sampling
        time.sleep(0.0005)
    torch.cuda.synchronize()
    clk.stop()
    dl = [pkg.bh_launch_count(H.h) - a for H, a in zip(Hs, l0)]
    launches = sum(dl)        # the library counts each kernel launch once (fused passes on their first histogram)
    if world > 1:        # one pack (+ one unpack where the sum lands) per step, counted by the library
        pass
    ms = t0.elapsed_time(t1)
    # the strategy the timed fills ran (AUTO's device-side SORT decision is reset by the e2e leg)
    names = {0: "auto", 1: "priv", 2: "global", 3: "cache", 4: "exact", 5: "sort"}
    strat = f"bh_fill_multi, plan: {args.multi_mode}" if multi else names[Hs[0].strategy(hists[0].weighted)]
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

    def e2e_step():
        for H in Hs:
            H.reset()
        if multi:
            cols = [t.to(dev, non_blocking=True) for t in host]
            do_fill(cols)
        else:
            h = hists[0]
            Hs[0].fill_host([host[slot[c]] for c in h.cols], host[slot[wl.wcol]] if h.weighted else None)
        if xchg is not None:
            xchg(stream)
        return [H.read() for H in Hs]

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
    if rank == 0 or args.exchange == "allreduce":
        assert all(r["entries"] == N * world for r in res), [r["entries"] for r in res]
    if args.dump and rank == 0:          # the reduced states (tests compare them with the oracle)
        np.savez(args.dump, **{f"{k}{i}": r[k] for i, r in enumerate(res) for k in ("content", "sumw2", "stats")},
                 **{f"entries{i}": np.array(r["entries"]) for i, r in enumerate(res)})
    e2e_value = N * world * e2e_steps / e2e_s
    h2d = 8 * N * len(used)
    d2h = 8 * sum(pkg.bh_packed_size(H.h) for H in Hs)      # bh_read of every histogram
    # PCIe roofline of the e2e leg: plain pinned host -> device copy of one input column
    # (up to 1 GiB), timed with CUDA events on this GPU alone
    nb = min(N, 1 << 27)
    dst = torch.empty(nb, dtype=torch.float64, device=dev)
    dst.copy_(host[0][:nb], non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        dst.copy_(host[0][:nb], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    pcie_peak = 3 * 8 * nb / (e0.elapsed_time(e1) * 1e-3) / 1e9
    del dst

    # same-run read ceiling: a plain torch reduction over this step's input columns (measurement
    # only, outside the timed region), the bandwidth a read-only stream of these bytes reaches here
    read_gbs = None
    if rank == 0:
        torch.cuda.synchronize()
        tr = []
        for _ in range(3):
            r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            r0.record()
            for t in devc:
                t.sum()
            r1.record()
            torch.cuda.synchronize()
            tr.append(r0.elapsed_time(r1))
        read_gbs = sum(t.numel() * 8 for t in devc) / (min(tr) * 1e-3) / 1e9

    # ---- secondary rows (rank 0, N=1): e.g. the 1D fixed-bin target of the north star (C1S)
    secondary = {}
    if rank == 0 and world == 1 and args.secondary:
        del devc
        torch.cuda.empty_cache()
        for name in [x for x in args.secondary.split(",") if x]:
            if name == "P32K":
                secondary[name] = measure_bulk_regime(local)
            else:
                secondary[name] = measure_secondary(name, max(3, min(args.steps, 10)), 3, local)

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N=1 only)
    cpu = None
    cpu_par = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = min(N, args.cpu_sample)
        ts = time_oracle(wl, sample, repeats=1)
        cpu = {"value": sample / ts[0], "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"events [0, {sample}) of the {wl.name} stream, single-thread C oracle (Neumaier sums)"}
        threads = os.cpu_count() or 1
        if threads > 1:
            tp = time_oracle_parallel(wl, sample, threads)
            cpu_par = {"value": sample / tp, "unit": UNIT, "cores": threads, "kind": "oracle",
                       "sample": f"the same events sharded over {threads} forked processes (all host cores)"}

    if rank == 0:
        peak, peak_src = hbm_peak()
        bpe = wl.bytes_per_event
        fill_avg = float(np.mean(fill_ms))
        achieved = bpe * N / (fill_avg * 1e-3) / 1e9
        traffic = ncu_traffic(wl.name)
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (bhgen seeded generator, host-generated)",
            "config": {"workload": workload_desc(wl), "events_per_gpu": N,
                       "total_bins": sum(H.nbins_total for H in Hs), "histograms": len(Hs),
                       "weighted": any(h.weighted for h in hists), "fill_strategy": strat,
                       "l2": f"inputs {bpe * N / 2**30:.1f} GiB/GPU >> 126 MB L2 (no flush needed)",
                       "parallelism": f"dp{world}: events sharded, one NCCL {args.exchange} per step of the "
                                      f"packed bins+stats of all histograms ({xchg.nbytes} B)"
                       if world > 1 else "single GPU"},
            "pct_hbm_peak": 100.0 * bpe * value / world / 1e9 / peak,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic,
                         "kernel": ("k_fused (one pass)" if args.multi_mode == "one-pass" else
                                    "k_fill per histogram + k_fill_multi for same-column groups") if multi
                         else ("k_part_scatter + k_part_reduce (sort)"
                                                                  if strat == "sort" else f"k_fill ({strat})"),
                         "launch_ms": fill_avg,
                         "algorithmic_bytes_per_launch": bpe * N, "peak_source": peak_src,
                         "read_ceiling_gbs": read_gbs, "frac_of_read_ceiling": achieved / read_gbs if read_gbs else None,
                         "read_ceiling_source": "torch .sum() over the step's device columns, same run, best of 3"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps, "pcie_gbs": h2d * world * e2e_steps / e2e_s / 1e9 / world,
                    "pcie_peak_gbs": pcie_peak,
                    "pcie_frac": h2d * e2e_steps / e2e_s / 1e9 / pcie_peak,
                    "clocks": clk2.summary()},
            "gpu_launches": launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "cpu_baseline_all_cores": cpu_par,
            "secondary": secondary or None,
        }
        print(json.dumps(line), flush=True)
    for H in Hs:
        H.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2", help="C1, C1S, C2 (default), C3, C3W, C4, C4W, C5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--strategy", default="auto", choices=["auto", "priv", "global", "cache", "exact", "sort"])
    ap.add_argument("--hist-strategy", default="",
                    help="per-histogram strategies of a multi-histogram config, e.g. '6=sort'")
    ap.add_argument("--multi-mode", default="passes", choices=["passes", "one-pass"],
                    help="bh_fill_multi plan for C5 (bh_set_multi_mode)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"], help="process-group backend for N>1")
    ap.add_argument("--exchange", default="reduce", choices=["reduce", "allreduce"],
                    help="N>1: sum the partial states on rank 0 only (reduce) or on every rank")
    ap.add_argument("--dump", default="", help="rank 0 writes the final (reduced) states to this .npz (tests)")
    ap.add_argument("--events", type=int, default=0, help="override events per GPU (tests)")
    ap.add_argument("--secondary", default="C1S,C1F,C2F,C3+sort,P32K",
                    help="comma list of extra configs measured device-resident after the headline ('' = none)")
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
