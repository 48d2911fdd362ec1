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


def tile_traffic(config: str):
    """DRAM bytes per launch of the eps-tile kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_tile_traffic.json")) as fh:
            t = json.load(fh)[config]
        return t["dram_read_bytes"] + t["dram_write_bytes"]
    except (OSError, KeyError, ValueError):
        return None


def algorithmic_ops_per_pair(d: int, formula: int) -> int:
    # ALGEBRAIC 2d+1, DIRECT 3d-1 separately rounded FP32 ops per pair
    return 2 * d + 1 if formula == 1 else 3 * d - 1


# ---------------------------------------------------------------------------------
def cpu_sample(points, eps_sq: float, min_pts: int, rows: int, threads: int):
    """Reference CPU path (oracle port) on `rows` rows x all N columns, threaded
    over row blocks like the reference's run_partitioned (_parallel.py:24-39)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import densescan_oracle as oracle
    p32 = oracle.narrow(points)
    norms = oracle.sq_norms(p32)
    thr = oracle.thr32(eps_sq)
    n = p32.shape[0]
    rows = min(rows, n)
    blocks = [(r0, min(r0 + 256, rows)) for r0 in range(0, rows, 256)]

    def work(b):
        r0, r1 = b
        hit = oracle.in_range_block(p32, norms, r0, r1, thr, oracle.ALGEBRAIC)
        np.packbits(hit, axis=-1)
        return int(hit.sum())

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as pool:
        list(pool.map(work, blocks))
    return time.perf_counter() - t0, rows


def cpu_baseline(points_aos, eps_sq, min_pts, n, target_s=12.0):
    threads = os.cpu_count() or 1
    # calibrate on a small slice, then size the sample for ~target_s of work
    t_small, r_small = cpu_sample(points_aos, eps_sq, min_pts, 512, threads)
    rows = int(max(512, min(n, r_small * target_s / max(t_small, 1e-6))))
    rows = (rows + 255) // 256 * 256
    secs, rows = cpu_sample(points_aos, eps_sq, min_pts, rows, threads)
    full_s = secs * n / rows  # rows are of uniform cost (every row spans all N columns)
    return {"value": n / full_s, "unit": "points/s", "cores": threads, "kind": "port",
            "sample": (f"stage-1 rows 0..{rows} of {n} x all {n} columns (algebraic, numpy "
                       f"oracle port, {threads} threads, {secs:.1f}s), extrapolated x{n / rows:.1f};"
                       " merge excluded (<3% of the reference's time, SURVEY §6)"),
            "seconds_extrapolated": full_s}


# ---------------------------------------------------------------------------------
def run_b200(args):
    import torch
    import paper_1506_02226_b200 as ds
    from paper_1506_02226_b200 import _native
    from paper_1506_02226_b200 import distributed as D

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

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
            labeling, tm = D.run_dbscan_sharded(None, params, formula=formula, mem_cap=mem_cap,
                                                backend=backend, coords=coords_dev)
            labels_dev.copy_(torch.from_numpy(labeling.labels))
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
    gpath = os.path.join(ROOT, "tests", "golden", f"{args.config.lower()}.npz")
    if os.path.exists(gpath):
        ref = np.load(gpath)
        parity = bool(np.array_equal(labels_dev.cpu().numpy(), ref["labels"]))

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
    # morton, 4 CUB radix-sort kernels, permute+bounds, 2 cull-row kernels, unit list,
    # eps-unit, union diag (+ core init), union links, roots, label scan, label = 16; a
    # word-overflow re-run repeats the pipeline; sharded runs add the forest merge and
    # a separate core init
    launches_per_step = 16 * last[3] if world == 1 else 18

    line = {
        "metric": "points clustered/sec (end-to-end DBSCAN, C2) with Gpair-evals/sec vs FP32 roofline",
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
                   "parallelism": (f"tile-pair items sharded over {world} GPUs (NCCL)"
                                   if world > 1 else "1 GPU")},
        "e2e": {"value": n / (e2e / 1e3), "unit": "points/s",
                "h2d_bytes_per_step": n * d * 8 * (world if world > 1 else 1),
                "d2h_bytes_per_step": n * 8, "ms_per_step": e2e,
                "parts_ms": ({k: statistics.mean(getattr(p, k) or 0.0 for p in e2e_parts)
                              for k in ("h2d_ms", "fused_ms", "merge_ms", "d2h_ms", "total_ms")}
                             if world == 1 else None)},
        "roofline": {"bound": "fp32", "kernel": "eps_unit_kernel", "achieved": achieved,
                     "peak": fp32_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp32_peak, "traffic": tile_traffic(args.config),
                     "traffic_source": "dram__bytes_read+write per launch, profiles/r01_tile_traffic.json",
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
        "gpair_evals_per_s": pairs / tile_s / 1e9,
        "n2_decisions_per_s": (n * n if world == 1 else n * n / world) / tile_s / 1e9,
        "stages_ms": last[2],
        "gpu_launches": launches_per_step * args.steps,
        "parity_vs_reference_labels": parity,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(pts.coords_aos, params.eps_sq, params.min_pts, n)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_1506_02226_b200 as ds
    cfg = ds.CONFIGS[args.config]
    pts = cfg.points()
    params = ds.validate_params(cfg.eps, cfg.min_pts)
    n = pts.n
    # each step: a bounded row sample of the same workload, extrapolated to N
    per_step_target = max(2.0, 60.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        cpu_baseline(pts.coords_aos, params.eps_sq, params.min_pts, n, per_step_target)
    vals = [cpu_baseline(pts.coords_aos, params.eps_sq, params.min_pts, n, per_step_target)
            for _ in range(args.steps)]
    value = statistics.mean(v["value"] for v in vals)
    last = vals[-1]
    line = {
        "metric": "points clustered/sec (end-to-end DBSCAN, C2) with Gpair-evals/sec vs FP32 roofline",
        "impl": "reference",
        "value": value, "unit": "points/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": n / value * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.description}", "n": n, "d": pts.d,
                   "eps": cfg.eps, "min_pts": cfg.min_pts, "formula": "algebraic"},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": last["cores"],
                         "kind": "port", "sample": last["sample"]},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
