#!/usr/bin/env python
"""bench.py — Soft-DTW DP cells/s (fwd+bwd) on B200, one JSON line on rank 0.

Metric (BASELINE.json): DP cells/sec (fwd+bwd, fused & unfused) at B=32 vs
L, D; peak HBM MB; 1/2/4/8 GPU.  cells/s = B*N*M / t(fwd+bwd), where one
step = loss + grad_x + grad_y of the whole batch (sdtw_with_gradients,
backward.hpp:276-304).

Default workload = the north-star config, BASELINE.json configs[2]: B=32,
N=M=4096, D=128, gamma=0.01, FUSED (the headline `value`; the largest
single-GPU config and the one `north_star`'s target is stated on), with the
UNFUSED mode of the same config measured in the same run (`unfused`).
Inputs on both arms are the reference's own bench generator (bench.hpp:61-66:
N(0,1) from mt19937_64(42), all of x then all of y), so the data-dependent
zero-tile skipping sees the same data the reference arm times.
`--config c1|c2|c4` run the other pair configs, `--config c5` the Soft-DTW
barycenter (B=1024 members, L=512, D=64): one step = objective + gradient
over all members + NCCL allreduce of grad_z across ranks + Adam update
(members sharded over ranks: strong scaling).

Arms:
  (default)         this engine (libsdtw_b200.so through the C-ABI).
  --impl reference  the reference's own CPU implementation (oracle/_ref,
                    compiled from the unmodified reference sources) with all
                    host threads, rank 0 only.

Multi-GPU: launched by torchrun, one rank per GPU; pairs are independent so
every rank runs its own B=32 batch with no collective on the data path
(weak scaling, `value`); the same run also times ONE B=32 batch split into
contiguous B/N pair shards (`strong_b32`, pairs/s); time =
max over ranks of the device-timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(B=32, L=256, D=128, gamma=1.0),
    "c2": dict(B=32, L=1024, D=128, gamma=0.1),
    "c3": dict(B=32, L=4096, D=128, gamma=0.01),
    "c4": dict(B=32, L=256, D=1024, gamma=1.0),
    "c5": dict(B=1024, L=512, D=64, gamma=1.0),
}
METRIC = "DP cells/sec (fwd+bwd, fused & unfused) at B=32 vs L,D; peak HBM MB; 1/2/4/8 GPU"
SM_COUNT = 148
MUFU_PER_CLK_SM = 16  # ex2 / lg2 / rcp lanes per clock per SM


def _mufu_rate():
    """MUFU lane-ops per clock per SM, measured on this GPU model by
    scripts/micro/mufu_rate.cu (profiles/mufu_r2.json), else the nominal 16."""
    try:
        with open(os.path.join(ROOT, "profiles", "mufu_r2.json")) as fh:
            m = json.load(fh)
        r = min(m["ex2_per_clk_sm"], m["lg2_per_clk_sm"], m["rcp_per_clk_sm"])
        return round(r), f"measured {r:.2f}/clk/SM (profiles/mufu_r2.json)"
    except Exception:
        return MUFU_PER_CLK_SM, "nominal"
# algorithmic MUFU work per DP cell
MUFU_FWD, MUFU_BWD = 3, 4


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML
    polled every 2 ms in a thread (nvidia-smi's 100 ms floor would miss a
    ~15 ms region); falls back to nvidia-smi -lms 100."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.reasons = set()
        self.stop_flag = threading.Event()
        self.thread = None
        self.smax = None
        self.proc = None
        self.lines = []

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = self.device
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                idx = int(vis.split(",")[self.device])
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self.stop_flag.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for nm, bit in self.REASONS.items():
                            if r & bit:
                                self.reasons.add(nm)
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
            return
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        self.stop_flag.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for ln in self.lines:
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    self.samples.append(float(parts[0]))
                    self.smax = max(self.smax or 0.0, float(parts[1]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[2:6]):
                    if v.lower() == "active":
                        self.reasons.add(nm)
        if self.thread:
            self.thread.join(timeout=2)
        sm = sorted(self.samples)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": self.smax,
                "samples": len(sm), "reasons": sorted(self.reasons)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_reference_rate(cfg, fused, threads, reps, warmup, max_pairs=None):
    """The reference's run_bench_row (bench.hpp:52-107), fp32, `threads`
    host threads.  Returns (cells/s, mean ms, sample description)."""
    import oracle
    ref = oracle.Reference()
    B = cfg["B"] if max_pairs is None else min(cfg["B"], max_pairs)
    rc, mean_ms, std_ms, peak, loss0 = ref.run_bench_row(B, cfg["L"], cfg["D"], cfg["gamma"],
                                                          fused=fused, repeats=reps,
                                                          warmup=warmup, threads=threads)
    if rc != 0:
        raise RuntimeError(f"reference run_bench_row failed rc={rc}")
    cells = B * cfg["L"] * cfg["L"]
    sample = (f"reference run_bench_row fp32 {'fused' if fused else 'unfused'} B={B} "
              f"L={cfg['L']} D={cfg['D']} gamma={cfg['gamma']}, {reps} timed reps after "
              f"{warmup} warm-up, threads={threads}")
    return cells / (mean_ms / 1e3), mean_ms, sample


def bench_inputs(B, L, D, seed):
    """The reference's own generator (bench.hpp:61-66) through
    oracle/_ref/libsdtw_ref.so: the engine arm's inputs equal the reference
    arm's.  Falls back to numpy N(0,1) only if that library is absent."""
    import numpy as np
    try:
        import oracle
        return oracle.Reference().bench_inputs(B, L, D, seed=seed)
    except Exception:
        rng = np.random.default_rng(seed)
        return (rng.standard_normal((B, L, D), dtype=np.float32),
                rng.standard_normal((B, L, D), dtype=np.float32))


def _ref_pairs_for(cfg):
    # bound one reference step to ~10-20 s of host work (SURVEY.md §6.3:
    # ~1.7e7 cells/s unfused, ~8e6 fused on 8 threads)
    per_pair = cfg["L"] * cfg["L"]
    return max(1, min(cfg["B"], int(8e7 // per_pair)))


def run_reference_arm(args, cfg):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    if args.config == "c5":
        return run_reference_barycenter(args, cfg, ws)
    threads = os.cpu_count() or 1
    fused = args.mode == "fused"
    pairs = _ref_pairs_for(cfg)
    times = []
    val = None
    sample = None
    for it in range(args.warmup + args.steps):
        v, ms, sample = cpu_reference_rate(cfg, fused, threads, 1, 0, max_pairs=pairs)
        if it >= args.warmup:
            times.append(ms)
    ms = sum(times) / len(times)
    cells = pairs * cfg["L"] * cfg["L"]
    val = cells / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "cells/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic N(0,1) (reference bench generator, mt19937_64 seed 42)",
        "config": _config_dict(args, cfg, ws),
        "cpu_baseline": {"value": val, "unit": "cells/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": val, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _bary_inputs(cfg, np):
    """C5 synthetic members (N(0,1), seeded) and the initial barycenter
    (member 0), identical on every rank."""
    rng = np.random.default_rng(42)
    K, L, D = cfg["B"], cfg["L"], cfg["D"]
    members = rng.standard_normal((K, L, D), dtype=np.float32)
    return members, members[0].copy()


def run_reference_barycenter(args, cfg, ws):
    """The reference's barycenter_objective (barycenter.hpp:60-86, members
    sequential, each sdtw_with_gradients on all host threads) on a bounded
    member sample; Adam on the host."""
    import numpy as np
    import oracle
    ref = oracle.Reference()
    threads = os.cpu_count() or 1
    members, z = _bary_inputs(cfg, np)
    kp = 8  # members per reference step (the sample)
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        rc, val, grad = ref.barycenter_objective(z, members[:kp], cfg["gamma"], threads=threads,
                                                 dtype=np.float32)
        times.append(time.perf_counter() - t0)
        if rc != 0:
            raise RuntimeError(f"reference barycenter_objective rc={rc}")
    ms = 1e3 * sum(times[args.warmup:]) / args.steps
    cells = kp * cfg["L"] * cfg["L"]
    val = cells / (ms / 1e3)
    sample = (f"reference barycenter_objective fp32 unfused log, {kp} of {cfg['B']} members, "
              f"L={cfg['L']} D={cfg['D']} gamma={cfg['gamma']}, threads={threads}")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "cells/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic N(0,1) members (numpy seed 42)", "config": _config_dict(args, cfg, ws),
        "cpu_baseline": {"value": val, "unit": "cells/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": val, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_barycenter_arm(args, cfg):
    """C5: Soft-DTW barycenter step on N GPUs (members sharded, strong
    scaling), grad_z summed by the engine's NCCL allreduce."""
    import numpy as np
    import torch
    from paper_2602_17206_b200 import Engine
    from paper_2602_17206_b200.build import build

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        build()
    if ws > 1:
        dist.barrier()
    eng = Engine(local)
    side = torch.cuda.Stream()
    torch.cuda.set_stream(side)
    eng.set_stream(side.cuda_stream)
    if ws > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(eng.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        eng.nccl_init(bytes(uid.cpu().numpy().tobytes()), ws, rank)
    K, L, D, gamma = cfg["B"], cfg["L"], cfg["D"], cfg["gamma"]
    members_h, z_h = _bary_inputs(cfg, np)
    from paper_2602_17206_b200.sharding import shard_range
    k0, k1 = shard_range(K, ws, rank)
    mem = torch.from_numpy(members_h[k0:k1]).cuda()
    z = torch.from_numpy(z_h).cuda()
    g = torch.empty_like(z)
    v = torch.zeros(1, dtype=torch.float64, device="cuda")
    m1 = torch.zeros(z.numel(), dtype=torch.float64, device="cuda")
    m2 = torch.zeros_like(m1)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step(t):
        eng.barycenter_objective(z, mem, gamma, grad_out=g, value_out=v)
        if ws > 1:
            eng.allreduce_grad(g, v)
        eng.adam_step(z, g, m1, m2, t)

    t = 0
    for _ in range(args.warmup):
        t += 1
        step(t)
    torch.cuda.synchronize()
    eng.reset_launches()
    eng.reset_peak()
    clocks = ClockSampler(local)
    if ws > 1:
        dist.barrier()
    clocks.start()
    stream = torch.cuda.current_stream()
    total = 0.0
    for _ in range(args.steps):
        flush.zero_()
        s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_.record(stream)
        t += 1
        step(t)
        e_.record(stream)
        e_.synchronize()
        total += s_.elapsed_time(e_)
    launches = eng.launches
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    tt = torch.tensor([total], device="cuda", dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    max_ms = float(tt.item())
    cells = K * L * L  # whole job per step
    value = cells * args.steps / (max_ms / 1e3)
    # e2e: host members and host z through the public API each step
    mh = torch.from_numpy(members_h[k0:k1]).pin_memory()
    zh = torch.from_numpy(z_h).pin_memory()
    gh = torch.empty_like(zh).pin_memory()
    e2e = 0.0
    for _ in range(args.steps):
        s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_.record(stream)
        eng.barycenter_objective(zh, mh, gamma, grad_out=gh)
        e_.record(stream)
        e_.synchronize()
        e2e += s_.elapsed_time(e_)
    te = torch.tensor([e2e], device="cuda", dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic N(0,1) members (numpy seed 42)",
            "config": _config_dict(args, cfg, ws),
            "peak_hbm_mb": eng.mem_stats()[1] / 2**20,
            "e2e": {"value": cells * args.steps / (float(te.item()) / 1e3), "unit": "cells/s",
                    "h2d_bytes_per_step": int((k1 - k0) * L * D * 4 + L * D * 4),
                    "d2h_bytes_per_step": int(L * D * 4 + 8),
                    "note": "objective+gradient only (no allreduce/Adam), host members per call"},
            "gpu_launches": launches, "roofline": None, "clocks": clk,
            "collective": "NCCL allreduce of grad_z (+ objective) per step" if ws > 1 else None,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    eng.close()


def _config_dict(args, cfg, ws):
    if args.config == "c5":
        return {"workload": f"c5: Soft-DTW barycenter, {cfg['B']} members L={cfg['L']} D={cfg['D']} "
                            f"gamma={cfg['gamma']} unfused log, objective+grad+allreduce+Adam",
                "members": cfg["B"], "global_batch": cfg["B"], "N": cfg["L"], "M": cfg["L"],
                "D": cfg["D"], "gamma": cfg["gamma"], "cost_mode": "unfused",
                "parallelism": f"dp{ws} (members sharded, NCCL allreduce of grad_z)",
                "l2": "flushed between timed steps (256 MiB write)"}
    return {"workload": f"{args.config}: B={cfg['B']} N=M={cfg['L']} D={cfg['D']} "
                        f"gamma={cfg['gamma']} {args.mode} fwd+bwd (loss, grad_x, grad_y)",
            "B_per_gpu": cfg["B"], "global_batch": cfg["B"] * ws, "N": cfg["L"], "M": cfg["L"],
            "D": cfg["D"], "gamma": cfg["gamma"], "cost_mode": args.mode,
            "backward_space": "log", "parallelism": f"dp{ws} (pairs sharded, no collective)",
            "l2": "flushed between timed steps (256 MiB write)"}


def time_engine(eng, torch, x, y, outs, fused, gamma, steps, warmup, flush):
    """Device-timed steps (CUDA events on the engine stream = torch's current
    stream).  Returns (total_ms, per-phase ms sums, launches, peak bytes)."""
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        eng.sdtw_with_gradients(x, y, gamma, fused=fused, out=outs, sync=False)
    torch.cuda.synchronize()
    eng.reset_peak()
    eng.enable_timing(True)
    phases = {}
    total = 0.0
    eng.reset_launches()
    launches = 0
    for _ in range(steps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        eng.sdtw_with_gradients(x, y, gamma, fused=fused, out=outs, sync=False)
        e.record(stream)
        e.synchronize()
        total += s.elapsed_time(e)
        for k, v in eng.phase_times().items():
            phases[k] = phases.get(k, 0.0) + v
        launches = eng.launches
    eng.enable_timing(False)
    return total, phases, launches, eng.mem_stats()[1]


def run_engine_arm(args, cfg):
    import numpy as np
    import torch
    from paper_2602_17206_b200 import Engine
    from paper_2602_17206_b200.build import build

    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    if rank == 0:
        build()
    if ws > 1:
        dist.barrier()
    eng = Engine(local)
    # a real (non-default) stream shared by torch and the engine, so the
    # CUDA events below bracket exactly the engine's work
    side = torch.cuda.Stream()
    torch.cuda.set_stream(side)
    eng.set_stream(side.cuda_stream)
    B, L, D, gamma = cfg["B"], cfg["L"], cfg["D"], cfg["gamma"]
    xh_np, yh_np = bench_inputs(B, L, D, 42 + rank)
    x = torch.from_numpy(xh_np).cuda()
    y = torch.from_numpy(yh_np).cuda()
    outs = (torch.empty(B, device="cuda"), torch.empty((B, L, D), device="cuda"),
            torch.empty((B, L, D), device="cuda"))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fused = args.mode == "fused"

    clocks = ClockSampler(local)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    total_ms, phases, launches, peak = time_engine(eng, torch, x, y, outs, fused, gamma,
                                                   args.steps, args.warmup, flush)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    cells_per_rank = B * L * L
    value = cells_per_rank * ws * args.steps / (max_ms / 1e3)

    # ---- the other cost mode of the same config (same protocol) --------
    other = None
    if not args.single_mode:
        o_ms, o_ph, _, o_peak = time_engine(eng, torch, x, y, outs, not fused, gamma,
                                            args.steps, min(args.warmup, 3), flush)
        t2 = torch.tensor([o_ms], device="cuda", dtype=torch.float64)
        if ws > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        o_max = float(t2.item())
        other = {"cost_mode": "unfused" if fused else "fused",
                 "value": cells_per_rank * ws * args.steps / (o_max / 1e3), "unit": "cells/s",
                 "ms_per_step": o_max / args.steps, "peak_hbm_mb": o_peak / 2**20,
                 "phase_ms_per_step": {k: v / args.steps for k, v in o_ph.items()}}

    # ---- strong scaling of ONE B=32 batch: contiguous
    # B/N pair shards, no collective; max-over-ranks device time ----------
    strong = None
    if ws > 1:
        from paper_2602_17206_b200.sharding import shard_range
        b0, b1 = shard_range(B, ws, rank)
        xs_, ys_ = x[b0:b1].contiguous(), y[b0:b1].contiguous()
        outs_s = (outs[0][b0:b1], outs[1][b0:b1], outs[2][b0:b1])
        dist.barrier()
        s_ms, _, _, _ = time_engine(eng, torch, xs_, ys_, outs_s, fused, gamma, args.steps,
                                    min(args.warmup, 3), flush)
        ts = torch.tensor([s_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(ts, op=dist.ReduceOp.MAX)
        s_max = float(ts.item())
        strong = {"batch": B, "pairs_per_gpu": f"{b1 - b0} (contiguous shard of one B={B} batch)",
                  "pairs_per_s": B * args.steps / (s_max / 1e3),
                  "cells_per_s": B * L * L * args.steps / (s_max / 1e3),
                  "ms_per_step": s_max / args.steps}

    # ---- e2e through the public API with pinned host buffers ----------
    xh = x.cpu().pin_memory()
    yh = y.cpu().pin_memory()
    lh = torch.empty(B).pin_memory()
    gxh = torch.empty((B, L, D)).pin_memory()
    gyh = torch.empty((B, L, D)).pin_memory()
    for _ in range(min(args.warmup, 2)):
        eng.sdtw_with_gradients(xh, yh, gamma, fused=fused, out=(lh, gxh, gyh))
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e2e_ms = 0.0
    for _ in range(args.steps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        eng.sdtw_with_gradients(xh, yh, gamma, fused=fused, out=(lh, gxh, gyh))
        e.record(stream)
        e.synchronize()
        e2e_ms += s.elapsed_time(e)
    t3 = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t3, op=dist.ReduceOp.MAX)
    e2e_max = float(t3.item())
    h2d = 2 * B * L * D * 4
    d2h = B * 4 + 2 * B * L * D * 4

    # ---- roofline of the dominant kernel --------------------------------
    peaks, src = _peaks()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    mufu_clk, mufu_src = _mufu_rate()
    mufu_peak = SM_COUNT * mufu_clk * sm_mhz * 1e6 / 1e9  # G MUFU op/s
    per_step = {k: v / args.steps for k, v in phases.items()}
    dom = max(per_step, key=per_step.get) if per_step else "backward"
    roofline = None
    if dom in ("forward", "backward"):
        mufu = MUFU_FWD if dom == "forward" else MUFU_BWD
        ach = mufu * cells_per_rank / (per_step[dom] / 1e3) / 1e9
        kname = {"forward": "sdtw_forward_tc_kernel" if fused else "sdtw_forward3_kernel",
                 "backward": "sdtw_backward4_kernel"}[dom]
        roofline = {"bound": "sfu", "kernel": kname, "achieved": ach,
                    "peak": mufu_peak, "unit": "GMUFU-op/s", "frac": ach / mufu_peak,
                    "traffic": _traffic(args, dom),
                    "algorithmic": f"{mufu} MUFU/cell x {cells_per_rank} cells per launch "
                                   "(SURVEY.md §8(d)); the backward computes only the tiles "
                                   "whose E is not exactly zero, so its dense-equivalent rate "
                                   "is reported" if dom == "backward" else
                                   f"{mufu} MUFU/cell x {cells_per_rank} cells per launch (SURVEY.md §8(d))",
                    "peak_basis": f"{SM_COUNT} SM x {mufu_clk} MUFU/clk ({mufu_src}) x {sm_mhz} MHz "
                                  f"(sm_max_mhz, {src})",
                    "share_of_step": per_step[dom] / (total_ms / args.steps)}
    elif dom == "grads":
        # the ordered contraction runs on the fp32 SIMT pipe (FFMA, fixed
        # order for determinism), so its bound is the FFMA peak, computed
        # like the MUFU one; algorithmic work counts only the stored non-zero
        # tiles' cells would be smaller, so the dense 4 D flop/cell is quoted
        flop = 2 * 2 * cells_per_rank * D
        ach = flop / (per_step[dom] / 1e3) / 1e12
        pk = SM_COUNT * 128 * 2 * sm_mhz * 1e6 / 1e12
        roofline = {"bound": "fp32-fma", "kernel": "contract_ordered_kernel", "achieved": ach,
                    "peak": pk, "unit": "TFLOP/s", "frac": ach / pk, "traffic": _traffic(args, dom),
                    "algorithmic": f"4 D flop/cell (dX and dY, 2 flop per FMA) x {cells_per_rank} cells "
                                   "(dense-equivalent: only non-zero E tiles are contracted)",
                    "peak_basis": f"{SM_COUNT} SM x 128 FFMA/clk x 2 flop x {sm_mhz} MHz (sm_max_mhz, {src})",
                    "share_of_step": per_step[dom] / (total_ms / args.steps)}
    elif dom == "costs":
        byt = 4 * cells_per_rank
        ach = byt / (per_step[dom] / 1e3) / 1e9
        pk = float(peaks.get("hbm_gbs", 6650.0))
        roofline = {"bound": "hbm", "kernel": "cost_gemm_tc_kernel", "achieved": ach, "peak": pk,
                    "unit": "GB/s", "frac": ach / pk, "traffic": _traffic(args, dom),
                    "share_of_step": per_step[dom] / (total_ms / args.steps)}

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic N(0,1) from the reference's bench generator (bench.hpp:61-66, "
                    "mt19937_64 seed 42+rank, x then y), fp32",
            "config": _config_dict(args, cfg, ws),
            "peak_hbm_mb": peak / 2**20,
            "phase_ms_per_step": per_step,
            "e2e": {"value": cells_per_rank * ws * args.steps / (e2e_max / 1e3),
                    "unit": "cells/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_max / args.steps},
            "gpu_launches": launches,
            "roofline": roofline,
            "clocks": clk,
            "pairs_per_s": B * ws * args.steps / (max_ms / 1e3),
        }
        if strong:
            line["strong_b32"] = strong
        if other:
            line["unfused" if fused else "fused"] = other
        if ws == 1 and not args.no_cpu_baseline:
            try:
                pairs = _ref_pairs_for(cfg)
                v, ms, sample = cpu_reference_rate(cfg, fused, os.cpu_count() or 1, 2, 1,
                                                   max_pairs=pairs)
                line["cpu_baseline"] = {"value": v, "unit": "cells/s",
                                        "cores": os.cpu_count() or 1, "kind": "reference",
                                        "sample": sample}
            except Exception as exc:  # the baseline is reported, not required
                line["cpu_baseline"] = {"value": None, "unit": "cells/s", "cores": 0,
                                        "kind": "reference", "sample": f"unavailable: {exc}"}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    eng.close()


def _traffic(args, dom):
    """dram bytes per launch from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh)
        return t.get(f"{args.config}_{args.mode}_{dom}")
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--mode", default="fused", choices=["fused", "unfused"])
    ap.add_argument("--single-mode", action="store_true", help="skip the other cost mode")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, cfg)
    elif args.config == "c5":
        run_barycenter_arm(args, cfg)
    else:
        run_engine_arm(args, cfg)


if __name__ == "__main__":
    main()
