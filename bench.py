#!/usr/bin/env python
"""Benchmark of the densescan hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl b200|reference]

Workload (BASELINE.json configs[1], the single-GPU config): C2 = 2-D blobs +
10% uniform noise, N=200,000, eps=0.3, MinPts=8, synthetic (seeded generator,
paper_1506_02226_b200.datasets). One step = one full clustering of the N
points (stage 1+2 eps-tile kernel, stage 3 union-find, canonical labels).

  value     points clustered / s, inputs resident in HBM, CUDA-event timed on
            the launching stream, L2 flushed (512 MB write) before every step
  e2e       points clustered / s through the public API run_dbscan() with
            host numpy buffers: H2D of the float64 points and D2H of the int64
            labels inside the timed region (wall clock, synchronous call)
  roofline  the eps-tile kernel against the FP32 pipe: algorithmic FP32 ops =
            pair evaluations x (2d+1), per launch, over its
            CUDA-event duration inside the timed region
  cpu_baseline  the oracle port of the reference CPU path on this host's cores
            on a bounded row sample, extrapolated to the full N (O(N^2) rows
            of uniform cost)

--impl reference prints the reference arm: the same metric for the CPU path
(oracle port, all host threads), rank 0 only.
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

SM_COUNT_DEFAULT = 148
METRIC = "points clustered/sec (end-to-end DBSCAN) with Gpair-evals/sec vs FP32 roofline"
FP32_LANES_PER_SM = 128


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


class ClockSampler:
    """SM clocks + throttle reasons sampled (NVML, every 2 ms) during the timed region.

    Falls back to `nvidia-smi` queries when NVML is unavailable.
    """

    REASONS = {  # nvmlClocksEventReason* bits
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x4: "sw_power_cap",
    }

    def __init__(self, index: int = 0, period_ms: float = 2.0):
        self.index = index
        self.period = period_ms / 1000.0
        self.samples = []  # (sm_mhz, max_mhz, reason_bits)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            nv = self._nvml
            sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            try:
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
            return float(sm), float(mx), int(rs)
        out = subprocess.run(["nvidia-smi", f"--id={self.index}",
                              "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                              "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5)
        sm, mx, act = [p.strip() for p in out.stdout.strip().split(",")]
        return float(sm), float(mx), int(act, 16)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample())
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({name for _, _, bits in self.samples
                          for bit, name in self.REASONS.items() if bits & bit})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def tile_capture(config: str):
    """The eps-tile kernel's entry in the committed ncu capture summary, or {}."""
    for path in (("profiles", "r02", "tile_traffic.json"), ("profiles", "r01_tile_traffic.json")):
        try:
            with open(os.path.join(ROOT, *path)) as fh:
                return json.load(fh)[config]
        except (OSError, KeyError, ValueError):
            continue
    return {}


def tile_traffic(config: str):
    """DRAM bytes per launch of the eps-tile kernel from the committed ncu capture."""
    t = tile_capture(config)
    return t["dram_read_bytes"] + t["dram_write_bytes"] if t else None


def tile_pipes(config: str):
    """FMA / ALU pipe and issue-active percentages of the same ncu capture."""
    t = tile_capture(config)
    keys = ("fma_pipe_pct", "alu_pipe_pct", "issue_active_pct")
    return {k: t[k] for k in keys if k in t} or None


def golden_labels(config: str):
    """The committed labels of a BASELINE config (the reference's own for C1/C2, the
    pinned C oracle's for C3-C5; tests/golden/), or None."""
    path = os.path.join(ROOT, "tests", "golden", f"{config.lower()}.npz")
    if not os.path.exists(path):
        return None
    g = np.load(path)
    key = "labels" if "labels" in g.files else "alg/labels"
    return g[key].astype(np.int64)


def stage3_hbm(stages: dict, n: int, peaks: dict):
    """Stage 3 (union-find merge, borders, canonical labels) against the HBM roofline:
    algorithmic bytes = the adjacency word records read once (8 B per reserved slot,
    stage 1's output) + the O(n) arrays it touches: counts 4, core flag 1, parent
    read + write 8, border minimum 4, root 4, first-appearance flag 4, id scan 4,
    int64 label 8 = 37 B per point."""
    ms = stages.get("merge")
    if not ms:
        return None
    nbytes = 8 * int(stages.get("words_emitted", 0)) + 37 * n
    gbs = nbytes / (ms / 1e3) / 1e9
    peak = peaks.get("hbm_gbs")
    return {"ms": ms, "algorithmic_bytes": nbytes, "achieved_gbs": gbs, "peak_gbs": peak,
            "frac": (gbs / peak) if peak else None,
            "timing": "%globaltimer stamps at the stage boundary (device)"}


def algorithmic_ops_per_pair(d: int, formula: int) -> int:
    # ALGEBRAIC 2d+1, DIRECT 3d-1 separately rounded FP32 ops per pair
    return 2 * d + 1 if formula == 1 else 3 * d - 1


# ---------------------------------------------------------------------------------
def cpu_full_run(points_aos, eps_sq: float, min_pts: int, threads: int):
    """One complete clustering of the workload by the reference's CPU flow (oracle port
    of run_dbscan, pipeline.py:70-92: threaded 256-row blocks materialising the packbits
    neighbourhood matrix, kernels.py:311-337, then the core-core merge, border rule and
    canonical ids, merge.py:116-166 / core.py:116-132). No sampling, no extrapolation.
    Returns (seconds, stage-1+2 seconds, stage-3 seconds, labels)."""
    from oracle import densescan_oracle as oracle
    t0 = time.perf_counter()
    labels, _, s12, s3 = oracle.dbscan_reference_flow(points_aos, eps_sq, min_pts,
                                                      oracle.ALGEBRAIC, threads=threads)
    return time.perf_counter() - t0, s12, s3, labels


def cpu_baseline(points_aos, eps_sq, min_pts, n, runs: int = 1, golden=None):
    threads = os.cpu_count() or 1
    secs, s12, s3 = [], [], []
    equal = None
    for _ in range(runs):
        t, a, b, labels = cpu_full_run(points_aos, eps_sq, min_pts, threads)
        secs.append(t)
        s12.append(a)
        s3.append(b)
        if golden is not None:
            equal = bool(np.array_equal(labels, golden))
    best = min(secs)
    return {"value": n / best, "unit": "points/s", "cores": threads, "kind": "port",
            "sample": (f"full workload: {n} points clustered end to end (stage 1+2 and merge), "
                       f"{runs} run(s), min taken; numpy oracle port of the reference's "
                       f"run_dbscan flow on {threads} host threads; no sampling or extrapolation"),
            "seconds": best, "stage12_s": min(s12), "stage3_s": min(s3),
            "labels_equal_reference": equal}


# ---------------------------------------------------------------------------------
def e2e_split(parts):
    """Mean split of the end-to-end calls: coordinate copy in (CUDA events), stage 1+2 and
    stage 3 (device stamps), and the rest of the call's wall time — the label copy out,
    the node/launch gaps and the host side."""
    out = {k: statistics.mean(getattr(p, k) or 0.0 for p in parts)
           for k in ("h2d_ms", "fused_ms", "merge_ms", "total_ms")}
    out["copy_out_and_host_ms"] = out["total_ms"] - out["h2d_ms"] - out["fused_ms"] - out["merge_ms"]
    return out


def run_b200(args):
    import torch
    import paper_1506_02226_b200 as ds
    from paper_1506_02226_b200 import _native
    from paper_1506_02226_b200 import distributed as D

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # one GPU per rank; DS_DIST_BACKEND=gloo (test hook) lets several ranks share the
    # device(s) of a smaller box to exercise this path (host-staged exchanges)
    dist_backend = os.environ.get("DS_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if dist_backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines on stderr
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(dist_backend)

    cfg = ds.CONFIGS[args.config]
    pts = cfg.points()
    params = ds.validate_params(cfg.eps, cfg.min_pts)
    formula = 1
    n, d = pts.n, pts.d
    mem_cap = 150 * 1024**3
    ctx = _native.context(local)
    dev = f"cuda:{local}"

    coords_dev = torch.from_numpy(pts.coords_aos.copy()).to(dev)
    labels_dev = torch.empty(n, dtype=torch.int64, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    backend = D.NativeShardBackend(local) if world > 1 else None

    def step():
        """One clustering of the resident points -> (tile_ms, pairs_evaluated, stage dict)."""
        if world > 1:
            labels, tm = D.run_dbscan_sharded(None, params, formula=formula, mem_cap=mem_cap,
                                              backend=backend, coords=coords_dev,
                                              return_device=True)
            labels_dev.copy_(labels)  # device to device: no host copy in the device-timed value
            return tm.tile_ms, tm.pairs_evaluated, {
                "stage12": tm.stage12_ms, "exchange1": tm.exchange1_ms,
                "stage3_local": tm.stage3_local_ms, "exchange2": tm.exchange2_ms,
                "stage3_merge": tm.stage3_merge_ms, "tile": tm.tile_ms}, 1
        t = ctx.run_dbscan_device(coords_dev.data_ptr(), n, d, params.eps_sq, params.min_pts,
                                  formula, mem_cap, labels_dev.data_ptr(), stream.cuda_stream)
        extra = {"words_emitted": t.words_emitted, "tiles_kept": t.tiles_total}
        return t.tile_ms, t.pairs_evaluated, {"fused": t.fused_ms, "merge": t.merge_ms,
                                               "tile": t.tile_ms, **extra}, t.tile_launches

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # parity of the benchmarked configuration against the committed reference labels
    parity = None
    golden = golden_labels(args.config)
    if golden is not None:
        parity = bool(np.array_equal(labels_dev.cpu().numpy(), golden))

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    times, tile_ms, last = [], [], None
    clk = ClockSampler(local).__enter__()  # spans the device-timed and the e2e legs
    if True:
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            last = step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            tile_ms.append(last[0])
    torch.cuda.synchronize()
    ms = statistics.mean(times)
    # the roofline's kernel time by CUDA events recorded around the eps-tile kernel on
    # its launching stream (a separate leg: events between kernels cost device time,
    # so the timed steps above take the stage split from the kernels' stamps)
    tile_ms_stamps = list(tile_ms)
    if world == 1:
        ctx.set_event_timing(True)
        try:
            for _ in range(args.warmup):
                step()
            tile_ms = []
            for _ in range(args.steps):
                flush.zero_()
                tile_ms.append(step()[0])
            torch.cuda.synchronize()
        finally:
            ctx.set_event_timing(False)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    pairs = last[1]

    # end-to-end through the public API with host buffers
    e2e_ms, e2e_parts = [], []
    cfg_api = ds.PipelineConfig(variant=ds.KernelVariant(ds.VariantId.FUSED_ALGEBRAIC),
                                mem_cap=mem_cap, device=local)

    def e2e_step():
        if world > 1:
            return D.run_dbscan_sharded(pts, params, formula=formula, mem_cap=mem_cap,
                                        backend=backend)[1]
        return ds.run_dbscan(pts, params, cfg_api)[1]

    for _ in range(max(1, args.warmup)):
        e2e_step()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        st = e2e_step()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_parts.append(st)
    e2e = statistics.mean(e2e_ms)
    clk.__exit__(None, None, None)
    if world > 1:
        tt = torch.tensor([e2e], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e = float(tt.item())

    # the paper's dense all-pairs schedule on the same input (stage 1+2 only): the
    # eps-tile kernel at full occupancy of work, for the FP32 roofline comparison
    dense = None
    if world == 1 and not args.no_dense:
        ctx.configure(False, False)
        dts = []
        for _ in range(3):
            _, _, _, dt = ctx.fused_build(pts.coords_aos, params.eps_sq, params.min_pts, formula,
                                          mem_cap, want_bits=False)
            dts.append(dt)
        ctx.configure(True, True)
        dense = {"tile_ms": statistics.mean(t.tile_ms for t in dts[1:]),
                 "pairs_per_launch": dts[-1].pairs_evaluated}
    # the FP32-bound case of the same kernel: BASELINE configs C4 (500k points, 16-D),
    # default culled schedule, stage 1+2 (a parity config, not a bench line)
    wide = None
    if world == 1 and not args.no_dense:
        c4 = ds.CONFIGS["C4"]
        p4 = c4.points()
        v4 = ds.validate_params(c4.eps, c4.min_pts)
        wts = []
        for _ in range(3):
            _, _, _, dt = ctx.fused_build(p4.coords_aos, v4.eps_sq, v4.min_pts, formula, mem_cap,
                                          want_bits=False)
            wts.append(dt)
        wide = {"n": p4.n, "d": p4.d, "tile_ms": statistics.mean(t.tile_ms for t in wts[1:]),
                "pairs_per_launch": wts[-1].pairs_evaluated,
                "ops_per_pair": algorithmic_ops_per_pair(p4.d, formula)}
        del p4
    peaks = load_peaks()
    clocks = clk.summary()
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    props = torch.cuda.get_device_properties(local)
    sms = props.multi_processor_count
    fp32_peak = sms * FP32_LANES_PER_SM * sm_max * 1e6 / 1e12  # T lane-ops/s
    ops = algorithmic_ops_per_pair(d, formula)
    tile_s = statistics.mean(tile_ms) / 1e3
    achieved = pairs * ops / tile_s / 1e12
    # kernels per step (1 GPU, culled schedule; the ncu launch list in profiles/): prep,
    # the spatial sort — for 1-2-D inputs up to 2^18 points the counting sort (keys +
    # histogram, scan, scatter: 3), else morton + (digit scan + radix scatter) per 8-bit
    # key digit (3 passes: 7) — permute + bounds, the culling kernel, unit list, eps-unit,
    # union diag (+ core init), union links, roots, scan + labels; a capacity re-run
    # repeats the pipeline; sharded runs add the shard-stage kernels and folds
    sort_kernels = 3 if (min(d, 4) <= 2 and n <= (1 << 18)) else 7
    launches_per_step = (9 + sort_kernels) * last[3] if world == 1 else 18

    line = {
        "metric": METRIC,
        "value": n / (ms / 1e3),
        "unit": "points/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded Gaussian blobs + uniform noise, datasets.generate_blobs)",
        "config": {"workload": f"{cfg.name}: {cfg.description}", "n": n, "d": d,
                   "eps": cfg.eps, "min_pts": cfg.min_pts, "formula": "algebraic",
                   "l2": "flushed (512 MB write) before every timed step",
                   "parallelism": (f"tile-pair items sharded over {world} ranks "
                                   f"({dist_backend}, {torch.cuda.device_count()} visible GPUs)"
                                   if world > 1 else "1 GPU")},
        "e2e": {"value": n / (e2e / 1e3), "unit": "points/s",
                "h2d_bytes_per_step": n * d * 8 * (world if world > 1 else 1),
                "d2h_bytes_per_step": n * 8, "ms_per_step": e2e,
                "parts_ms": (e2e_split(e2e_parts) if world == 1 else None)},
        "roofline": {"bound": "fp32", "kernel": "eps_unit_kernel", "achieved": achieved,
                     "peak": fp32_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp32_peak, "traffic": tile_traffic(args.config),
                     "traffic_source": "dram__bytes_read+write per launch, profiles/r02/tile_traffic.json",
                     "ncu_pipes": tile_pipes(args.config),
                     "peak_source": (f"derived: {sms} SMs x 128 FP32 lanes x {sm_max:.0f} MHz "
                                     "(no measured FP32 figure in MEASURED_PEAKS.json)"),
                     "ops_per_pair": ops, "pairs_per_launch": pairs,
                     "tile_ms": statistics.mean(tile_ms),
                     "tile_ms_stamps": statistics.mean(tile_ms_stamps),
                     "tile_timing": "CUDA events around the kernel (DS_OPT_EVENT_TIMING leg)"},
        "dense_schedule": (None if dense is None else {
            "what": "prune=False, spatial_order=False: all 512x512 upper-triangle tile pairs",
            "tile_ms": dense["tile_ms"], "pairs_per_launch": dense["pairs_per_launch"],
            "achieved": dense["pairs_per_launch"] * ops / (dense["tile_ms"] / 1e3) / 1e12,
            "frac": dense["pairs_per_launch"] * ops / (dense["tile_ms"] / 1e3) / 1e12 / fp32_peak,
            "gpair_evals_per_s": dense["pairs_per_launch"] / (dense["tile_ms"] / 1e3) / 1e9}),
        "wide_records": (None if wide is None else {
            "what": "C4 (BASELINE configs[3]): n=%d, d=%d, default culled schedule, eps kernel "
                    "only (stage-1 device stamps), mean of 2 runs after one warm-up"
                    % (wide["n"], wide["d"]),
            "tile_ms": wide["tile_ms"], "pairs_per_launch": wide["pairs_per_launch"],
            "ops_per_pair": wide["ops_per_pair"],
            "traffic": tile_traffic("C4"), "ncu_pipes": tile_pipes("C4"),
            "achieved": wide["pairs_per_launch"] * wide["ops_per_pair"] / (wide["tile_ms"] / 1e3) / 1e12,
            "frac": wide["pairs_per_launch"] * wide["ops_per_pair"] / (wide["tile_ms"] / 1e3) / 1e12
                    / fp32_peak}),
        "gpair_evals_per_s": pairs / tile_s / 1e9,
        "n2_decisions_per_s": (n * n if world == 1 else n * n / world) / tile_s / 1e9,
        "stages_ms": last[2],
        "stage3_hbm": stage3_hbm(last[2], n, peaks) if world == 1 else None,
        "gpu_launches": launches_per_step * args.steps,
        "parity_vs_reference_labels": parity,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(pts.coords_aos, params.eps_sq, params.min_pts, n,
                                            golden=golden)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_reference(args):
    """The reference arm: the reference's CPU flow (oracle port, all host threads) on the
    same workload, every warm-up and timed step a complete clustering of all N points."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_1506_02226_b200 as ds
    cfg = ds.CONFIGS[args.config]
    pts = cfg.points()
    params = ds.validate_params(cfg.eps, cfg.min_pts)
    n = pts.n
    threads = os.cpu_count() or 1
    # every step is one complete clustering (~20 s at C2 on 16 threads), so the run is
    # bounded in time instead of in steps: one warm-up run, then timed runs until the
    # requested steps or the budget (DS_REF_BUDGET_S, default 150 s) — the line reports
    # the runs actually timed ("steps") next to the request
    budget = float(os.environ.get("DS_REF_BUDGET_S", "150"))
    for _ in range(min(args.warmup, 1)):
        cpu_full_run(pts.coords_aos, params.eps_sq, params.min_pts, threads)
    runs, t_start = [], time.perf_counter()
    while len(runs) < max(1, args.steps):
        runs.append(cpu_full_run(pts.coords_aos, params.eps_sq, params.min_pts, threads))
        if time.perf_counter() - t_start > budget:
            break
    ms = statistics.mean(r[0] for r in runs) * 1e3
    value = n / (ms / 1e3)
    golden = golden_labels(args.config)
    parity = None if golden is None else bool(np.array_equal(runs[-1][3], golden))
    line = {
        "metric": METRIC,
        "impl": "reference",
        "value": value, "unit": "points/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", str(args.gpus))),
        "steps": len(runs), "warmup": min(args.warmup, 1),
        "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.description}", "n": n, "d": pts.d,
                   "eps": cfg.eps, "min_pts": cfg.min_pts, "formula": "algebraic"},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": threads, "kind": "port",
                         "sample": (f"full workload every step: {n} points clustered end to "
                                    "end (stage 1+2 and merge) by the numpy oracle port of "
                                    f"the reference's run_dbscan flow on {threads} host "
                                    "threads; no sampling or extrapolation")},
        "stages_s": {"stage12": statistics.mean(r[1] for r in runs),
                     "stage3": statistics.mean(r[2] for r in runs)},
        "parity_vs_reference_labels": parity,
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        return sock.getsockname()[1]


def _rank_entry(rank, world, port, fn, fn_args):
    os.environ.update({"RANK": str(rank), "LOCAL_RANK": str(rank), "WORLD_SIZE": str(world),
                       "LOCAL_WORLD_SIZE": str(world), "MASTER_ADDR": "127.0.0.1",
                       "MASTER_PORT": str(port)})
    fn(*fn_args)


def spawn_ranks(world: int, fn, *fn_args):
    """One process per GPU on this node (what torchrun --nproc-per-node does): each
    rank gets RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* in its environment and runs
    fn(*fn_args). Used when bench.py --gpus N > 1 is started without torchrun."""
    import torch.multiprocessing as mp
    mp.spawn(_rank_entry, args=(world, _free_port(), fn, fn_args), nprocs=world, join=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-dense", action="store_true",
                    help="skip the dense-schedule comparison leg (profiling runs)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif "WORLD_SIZE" not in os.environ and args.gpus > 1:
        spawn_ranks(args.gpus, run_b200, args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
