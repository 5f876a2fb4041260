#!/usr/bin/env python
"""Benchmark of the PipeSP attention layer (BASELINE.json metric) -- one JSON line on rank 0.

    python bench.py [--gpus N --steps K --warmup W] [--workload hy544p129f] [--stages N_st]
    python bench.py --gpus N ...      (N > 1 without torchrun: re-launches itself through
                                       torch.distributed.run, one process per GPU, NCCL)
    torchrun --nproc-per-node N bench.py --gpus N ...
    python bench.py --impl reference ...                         (the fp64 CPU oracle arm)

A step = one SP attention layer (all SURVEY §8(a) rows: pack, per-stage input all-to-all,
tcgen05 attention, per-stage output all-to-all, Psi_g unpack) over one batch of synthetic
Q/K/V shaped like the named workload, inputs resident in HBM.  Default workload at every N:
BASELINE configs[2] (HunyuanVideo-like 1024x576x129, S = 76,032, H = 24, D = 128), the largest
configuration that fits one GPU's benchmark budget and splits over 1/2/4/8 ranks.  Strong scaling:
the global problem is fixed and split over P = N ranks.  `value` = total attention FLOPs
(4*B*S^2*H*D) / max over ranks of the per-rank MEDIAN step time, in TFLOP/s.  With N = 8 the line
adds the north-star block: configs[3] (720p x 129f, S = 118,800) over N_st in {1,2,3,4,6,8,12,24},
with exposed all-to-all and a2a GB/s per stage split.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per SP attention layer and TFLOP/s at 1/2/4/8 B200; exposed all-to-all %"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="hy544p129f")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--stages", type=int, default=0, help="N_st (0 = paper's per-head loop, h stages)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--host-groups", type=int, default=24, help="head groups of the 1-GPU host-buffer e2e call")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle sample time")
    ap.add_argument("--spawn", action="store_true", help="launch through torch.distributed.run even at N=1")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "p2p", "nccl-window"],
                    help="N>1 exchange: NCCL grouped send/recv; CUDA IPC peer memory with copy engines (f1); or the "
                         "same peer-memory exchange on an NCCL symmetric window (ncclMemAlloc + ncclCommWindowRegister)")
    ap.add_argument("--direct", action="store_true",
                    help="p2p / nccl-window transports: pack / epilogue store to peers (f1)")
    ap.add_argument("--qkv", action="store_true",
                    help="layer from hidden states: fused QKV projection (f3) + PipeSP; FLOPs include the projection")
    ap.add_argument("--north-star", type=int, default=-1,
                    help="720p N_st sweep block: 1 on, 0 off, -1 (default) on when N == 8")
    ap.add_argument("--no-one-rank", action="store_true",
                    help="N=1: skip the north-star block measured as ONE rank's share of the 8-GPU schedule")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def workload_cfg(args):
    import synthgen
    w = synthgen.WORKLOADS[args.workload]
    B = args.batch or w.B
    return w.name, B, w.S, w.H, w.D


def attn_flops(B, S, H, D):
    return 4.0 * B * S * S * H * D


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons sampled every 20 ms DURING the timed region (NVML; nvidia-smi fallback)."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu_index: int, period_s: float = 0.02):
        self.gpu, self.period = gpu_index, period_s
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self.power_w, self.power_limit_w = [], None
        self._stop = threading.Event()
        self._t = None

    def _loop(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            try:
                self.power_limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0
            except Exception:  # pragma: no cover
                pass
            while not self._stop.is_set():
                self.sm.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                try:
                    self.power_w.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
                except Exception:  # pragma: no cover
                    pass
                bits = get_reasons(h)
                for bit, name in self.REASONS.items():
                    if bits & bit:
                        self.reasons.add(name)
                self._stop.wait(self.period)
        except Exception as e:  # pragma: no cover
            self.error = str(e)[:120]

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        time.sleep(0.05)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml, 20 ms, timed region",
                "power_w": statistics.median(self.power_w) if self.power_w else None,
                "power_limit_w": self.power_limit_w}


# ------------------------------------------------------------------ CPU oracle timing
def time_oracle(S, D, rows_target_s: float, seed=0):
    """The fp64 C oracle (as it stands) on R query rows of one head with the full K/V of that head."""
    import numpy as np
    import torch

    import oracle
    import synthgen
    shape = (1, S, 1, D)
    K = synthgen.gen_head_rows(seed, synthgen.TENSOR_K, shape, 0, 0).double().numpy()
    V = synthgen.gen_head_rows(seed, synthgen.TENSOR_V, shape, 0, 0).double().numpy()
    nthreads = os.cpu_count() or 1
    # calibrate: grow the probe until it takes >= 1 s, then scale to the target duration
    R = nthreads
    while True:
        rows = torch.arange(R) % S
        Q = synthgen.gen_head_rows(seed, synthgen.TENSOR_Q, shape, 0, 0, tokens=rows).double().numpy()
        t0 = time.perf_counter()
        oracle.attention_rows(Q, K, V, nthreads)
        dt = time.perf_counter() - t0
        if dt >= 1.0 or R >= 1 << 20:
            break
        R *= 4
    if dt < rows_target_s:
        R = int(R * rows_target_s / dt) // nthreads * nthreads
        rows = torch.arange(R) % S
        Q = synthgen.gen_head_rows(seed, synthgen.TENSOR_Q, shape, 0, 0, tokens=rows).double().numpy()
        t0 = time.perf_counter()
        oracle.attention_rows(Q, K, V, nthreads)
        dt = time.perf_counter() - t0
    flops = 4.0 * S * D * R
    return {"value": flops / dt / 1e12, "unit": "TFLOP/s", "cores": nthreads, "kind": "oracle",
            "sample": f"{R} query rows of one head (each against all S={S} keys, D={D}), fp64 C oracle, "
                      f"{dt:.1f} s on {nthreads} threads; per-row work is identical, so TFLOP/s carries over "
                      f"to the full layer", "seconds": dt, "rows": R}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    name, B, S, H, D = workload_cfg(args)
    if rank != 0:
        return
    P = args.gpus
    import torch

    import oracle
    import synthgen
    # each step = the oracle on R query rows of one head against the full K/V (bounded sample of the
    # workload); R calibrated once so that warmup + steps take about 2.5 minutes
    per_step_target = max(0.5, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    cal = time_oracle(S, D, per_step_target)
    R, nthreads = cal["rows"], cal["cores"]
    shape = (1, S, 1, D)
    K = synthgen.gen_head_rows(0, synthgen.TENSOR_K, shape, 0, 0).double().numpy()
    V = synthgen.gen_head_rows(0, synthgen.TENSOR_V, shape, 0, 0).double().numpy()
    Q = synthgen.gen_head_rows(0, synthgen.TENSOR_Q, shape, 0, 0, tokens=torch.arange(R) % S).double().numpy()
    secs = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.attention_rows(Q, K, V, nthreads)
        if i >= args.warmup:
            secs.append(time.perf_counter() - t0)
    res_steps = [{"rows": R, "cores": nthreads}]
    flops = 4.0 * S * D * R * len(secs)
    secs = sum(secs)
    value = flops / secs / 1e12
    full_layer_s = attn_flops(B, S, H, D) / (value * 1e12)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": P,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": full_layer_s * 1e3 / 1,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded splitmix64 Irwin-Hall bf16 inputs)",
        "config": {"workload": name, "B": B, "S": S, "H": H, "D": D, "P": P,
                   "note": "ms_per_step extrapolated from the sampled rows to the full layer"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": res_steps[0]["cores"], "kind": "oracle",
                         "sample": f"{args.steps} steps x ~{res_steps[0]['rows']} query rows of one head, full K/V"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
NORTH_STAR_STAGES = (1, 2, 3, 4, 6, 8, 12, 24)
NVLINK_GBS = 900.0   # NVLink 5 per direction per GPU (SURVEY §8(d) overlapped roofline)


def _a2a_send_bytes(plan, rank):
    """Bytes this rank sends to OTHER ranks over all stages (input Q/K/V + output O), from the plan's messages."""
    n = 0
    G_h, C, _ = plan.stage_split
    for k in range(G_h * C):
        for d in (0, 1):
            n += sum(m.bytes for m in plan.describe_messages(k, d, rank) if not m.is_recv and m.peer != rank)
    return n


def north_star_one_rank(spa, synthgen, torch, peak, flush, P=8, stages=(1, 3, 24), reps=3):
    """One rank's share of the 8-GPU PipeSP layer at 720p (BASELINE configs[3]), measured on one GPU: per stage split,
    the layer time with no exchange, with the exchange moved by the copy kernel (NCCL-like SM transport) and with the
    direct peer stores, exposed %, and the fraction of the overlapped roofline max(FLOPs/peak, bytes sent/900 GB/s)."""
    w = synthgen.WORKLOADS["hy720p129f"]
    B, S, H, D = w.B, w.S, w.H, w.D
    S_l = S // P
    shards = [[synthgen.gen_qkv_shard(0, t, (B, S, H, D), q * S_l, (q + 1) * S_l, device="cuda") for q in range(P)]
              for t in range(3)]
    outs = [torch.empty_like(x) for x in shards[0]]
    fl_rank = attn_flops(B, S, H, D) / P
    rows = []
    for st in stages:
        plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=st)
        ws = plan.workspace()
        sent = _a2a_send_bytes(plan, 0)
        troof = max(fl_rank / (peak * 1e12), sent / (NVLINK_GBS * 1e9)) * 1e3
        spa.spa_pipesp_attention_local(plan, *shards, outs, ws)   # every buffer holds real data first
        torch.cuda.synchronize()
        res = {}
        for mode in ("skip", "kernel", "direct"):
            plan.set_option(spa.SPA_OPT_RANK_ONLY, 1)
            plan.set_option(spa.SPA_OPT_DIRECT, int(mode == "direct"))
            plan.set_option(spa.SPA_OPT_SKIP_COMM, int(mode == "skip"))
            for _ in range(2):
                spa.spa_pipesp_attention_local(plan, *shards, outs, ws)
            torch.cuda.synchronize()
            ts = []
            for _ in range(reps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                spa.spa_pipesp_attention_local(plan, *shards, outs, ws)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            res[mode] = statistics.median(ts)
        for mode in ("kernel", "direct"):
            rows.append({"stages": st, "stage_split": list(plan.stage_split), "transport": mode,
                         "ms_per_layer": res[mode], "ms_no_exchange": res["skip"],
                         "exposed_a2a_pct": max(0.0, 100.0 * (res[mode] - res["skip"]) / res[mode]),
                         "tflops_per_gpu": fl_rank / (res[mode] * 1e-3) / 1e12,
                         "frac_overlapped_roofline": troof / res[mode], "t_roofline_ms": troof,
                         "bytes_sent_per_rank": sent})
        plan.close()
        del ws
    del shards, outs
    best = max(rows, key=lambda r: r["frac_overlapped_roofline"])
    return {"workload": "hy720p129f", "P": P, "rank": 0, "best": best, "rows": rows,
            "what": "one rank's share of the 8-GPU layer measured on ONE GPU (loopback plan, SPA_OPT_RANK_ONLY): "
                    "its attention stages, pack/unpack and the bytes it sends / receives as local copies or direct "
                    "stores; NVLink time of those bytes at 900 GB/s enters the roofline",
            "target": ">= 0.60 of the overlapped roofline, <= 10 % exposed all-to-all (BASELINE.json)"}


def aco_one_rank(spa, synthgen, torch, flush, P=8, n_src=6, reps=3):
    """BASELINE configs[4] (Aco: 720p attention over 6 denoising + 2 decoding GPUs) measured as single
    ranks' shares on one GPU: a source rank and a co-processor rank of the 6 + 2 plan against one rank of PipeSP on the
    6 denoising GPUs alone; speed-up vs Eq. 3's ideal N / N_d = 8 / 6 for t_L = 0.  Staged
    exchange by the copy kernel, one stage."""
    w = synthgen.WORKLOADS["hy720p129f"]
    B, S, H, D = w.B, w.S, w.H, w.D
    S_l = S // n_src
    shards = [[synthgen.gen_qkv_shard(0, t, (B, S, H, D), q * S_l, (q + 1) * S_l, device="cuda") for q in range(n_src)]
              for t in range(3)]
    outs = [torch.empty_like(x) for x in shards[0]]

    def one(plan, call, rank):
        ws = plan.workspace()
        call(plan, *shards, outs, ws)   # every buffer holds real data first
        torch.cuda.synchronize()
        plan.set_option(spa.SPA_OPT_RANK_ONLY, rank + 1)
        for _ in range(2):
            call(plan, *shards, outs, ws)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            call(plan, *shards, outs, ws)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        plan.set_option(spa.SPA_OPT_RANK_ONLY, 0)
        del ws
        return statistics.median(ts)

    aco = spa.Plan(spa.Comm.loopback(P), B, S, H, D, n_src=n_src)
    t_src = one(aco, spa.spa_aco_attention_local, 0)
    t_cop = one(aco, spa.spa_aco_attention_local, P - 1)
    aco.close()
    pip = spa.Plan(spa.Comm.loopback(n_src), B, S, H, D)
    t_pip = one(pip, spa.spa_pipesp_attention_local, 0)
    pip.close()
    del shards, outs
    return {"workload": "hy720p129f", "P": P, "n_src": n_src, "ms_source_rank": t_src, "ms_coprocessor_rank": t_cop,
            "ms_pipesp_on_n_src_gpus": t_pip, "speedup": t_pip / max(t_src, t_cop), "eq3_ideal": P / n_src,
            "what": "single ranks' shares measured on ONE GPU (loopback plans, SPA_OPT_RANK_ONLY), copy-kernel exchange"}


def single_gpu_config(spa, synthgen, torch, peak, flush, workload="osp480p93f", reps=5):
    """Another BASELINE configuration's whole layer on this one GPU (the attention kernel over all heads), CUDA events,
    L2 flushed before each of `reps` launches: ms, TF/s and the fraction of the measured peak."""
    w = synthgen.WORKLOADS[workload]
    q, k, v = (synthgen.gen_qkv_shard(0, t, (w.B, w.S, w.H, w.D), 0, w.S, device="cuda") for t in range(3))
    o = torch.empty_like(q)
    for _ in range(3):
        spa.attention(q, k, v, o)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        spa.attention(q, k, v, o)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    tf = attn_flops(w.B, w.S, w.H, w.D) / (ms * 1e-3) / 1e12
    return {"workload": workload, "B": w.B, "S": w.S, "H": w.H, "D": w.D, "ms_per_layer": ms, "tflops": tf,
            "frac_of_peak": tf / peak}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import synthgen
    from paper_2511_12056_b200 import spa

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # SPA_BENCH_SHARED_GPU=1: every rank on cuda:0 with a gloo process group -- exercises the N-rank p2p plumbing
    # (spawn, CUDA IPC set-up, cross-process flags) on a one-GPU box; its timings mean nothing
    shared = os.environ.get("SPA_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
        if world > 1 and args.transport != "p2p":
            raise SystemExit("SPA_BENCH_SHARED_GPU needs --transport p2p (NCCL refuses two ranks on one GPU)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    name, B, S, H, D = workload_cfg(args)
    P = world
    if S % P or H % P:
        raise SystemExit(f"workload {name} does not split over {P} ranks")
    stages = args.stages or (H // P if P > 1 else 1)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > L2 (126 MB)

    if P == 1:
        comm = spa.Comm.loopback(1, local)
    elif args.transport == "p2p":
        comm = spa.Comm.p2p(P, rank, local)
    else:
        obj = [spa.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = spa.Comm.nccl(obj[0], P, rank, local)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        t = torch.tensor([float(x)], device="cpu" if shared else dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def make(workload, n_st, qkv_mode=False):
        w = synthgen.WORKLOADS[workload]
        Bw = args.batch or w.B
        S_l = w.S // P
        plan = spa.Plan(comm, Bw, w.S, w.H, w.D, stages=n_st)
        if qkv_mode:   # hidden states X [B, S_l, C = H*D], the fused weight packed once for the plan
            C = w.H * w.D
            x = synthgen.gen_hidden_shard(0, (Bw, w.S, C), rank * S_l, (rank + 1) * S_l, device=dev)
            wp = plan.pack_qkv_weight(synthgen.gen_qkv_weight(0, C, w.H, w.D, device=dev),
                                      synthgen.gen_qkv_bias(0, w.H, w.D, device=dev))
            out = torch.empty((Bw, S_l, w.H, w.D), dtype=torch.bfloat16, device=dev)
            return plan, ("qkv", C, x, wp), out, p2p_setup(plan, plan.qkv_workspace(dev))
        qkv = [synthgen.gen_qkv_shard(0, t, (Bw, w.S, w.H, w.D), rank * S_l, (rank + 1) * S_l, device=dev)
               for t in range(3)]
        return plan, qkv, torch.empty_like(qkv[0]), p2p_setup(plan, plan.workspace(dev))

    def split_of(pl):
        return pl.stage_split[0]

    def p2p_setup(plan, ws):
        if P > 1 and args.transport == "p2p":   # map every rank's workspace (CUDA IPC handles over torch.distributed)
            plan.ipc_setup(ws)
            if args.direct:
                plan.set_option(spa.SPA_OPT_DIRECT, 1)
        elif P > 1 and args.transport == "nccl-window":   # a window of ws's size from NCCL's allocator replaces ws
            ws = plan.window_setup(ws.numel())
            if args.direct:
                plan.set_option(spa.SPA_OPT_DIRECT, 1)
        return ws

    def call(plan, qkv, out, ws):
        if qkv[0] == "qkv":
            _, C, x, wp = qkv
            if P == 1:
                spa.spa_pipesp_qkv_attention_local(plan, C, [x], wp, [out], ws, stream)
            else:
                spa.spa_pipesp_qkv_attention(plan, C, x, wp, out, ws, stream)
        elif P == 1:
            spa.spa_pipesp_attention_local(plan, [qkv[0]], [qkv[1]], [qkv[2]], [out], ws, stream)
        else:
            spa.spa_pipesp_attention(plan, *qkv, out, ws, stream)

    def timed(plan, qkv, out, ws, n, warm, profile):
        """Per-step CUDA-event times (ms) on the calling stream, L2 flushed (untimed) before every step."""
        for _ in range(warm):
            call(plan, qkv, out, ws)
            if P > 1:   # a stuck exchange aborts the communicator and fails the run instead of hanging it
                comm.wait(stream, timeout_ms=300_000)
        barrier()
        plan.set_option(spa.SPA_OPT_PROFILE, int(profile))
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        profs = []
        for i in range(n):
            flush.zero_()
            ev[i][0].record(stream)
            call(plan, qkv, out, ws)
            ev[i][1].record(stream)
            if profile:
                torch.cuda.synchronize()
                profs.append(plan.last_profile())
        barrier()
        plan.set_option(spa.SPA_OPT_PROFILE, 0)
        return [a.elapsed_time(b) for a, b in ev], profs

    def exposed_pct(plan, qkv, out, ws, t_layer, n):
        """(t_layer - t_skipcomm) / t_layer: the same plan and schedule with the all-to-alls not issued."""
        plan.set_option(spa.SPA_OPT_SKIP_COMM, 1)
        ms, _ = timed(plan, qkv, out, ws, n, 2, False)
        plan.set_option(spa.SPA_OPT_SKIP_COMM, 0)
        t_nc = max_over_ranks(statistics.median(ms))
        return max(0.0, (t_layer - t_nc) / t_layer * 100.0), t_nc

    peaks, peak_src = load_peaks()
    peak = peaks["bf16_tflops"]

    # ---------------------------------------------------------------- headline
    plan, qkv, out, ws = make(name, stages, args.qkv)
    with ClockSampler(local) as clk:
        step_ms, profs = timed(plan, qkv, out, ws, args.steps, args.warmup, True)
    t_max = max_over_ranks(statistics.median(step_ms))
    proj_flops = 2.0 * B * S * (H * D) * 3 * H * D if args.qkv else 0.0
    flops = attn_flops(B, S, H, D) + proj_flops
    value = flops / (t_max * 1e-3) / 1e12
    attn_ms = [sum(p.attn_ms[k] for k in range(p.n_stages)) for p in profs]
    a2a_in = [sum(p.a2a_in_ms[k] for k in range(p.n_stages)) for p in profs]
    a2a_out = [sum(p.a2a_out_ms[k] for k in range(p.n_stages)) for p in profs]
    launches = sum(p.attn_launches + p.copy_launches + p.gemm_launches for p in profs)
    qkv_info = None
    if args.qkv:
        proj_ms = statistics.median([p.pack_ms for p in profs])
        qkv_info = {"projection_ms": proj_ms, "projection_flops_per_rank": proj_flops / P,
                    "projection_tflops": proj_flops / P / (proj_ms * 1e-3) / 1e12,
                    "projection_frac_of_peak": proj_flops / P / (proj_ms * 1e-3) / 1e12 / peak,
                    "kernel": "qkv_gemm_kernel (tcgen05, fused pack)", "C": H * D}
    exposed, t_nocomm = (None, None)
    a2a = None
    if P > 1:
        exposed, t_nocomm = exposed_pct(plan, qkv, out, ws, t_max, args.steps)
        sent = _a2a_send_bytes(plan, rank)
        a2a_ms = statistics.median([a + b for a, b in zip(a2a_in, a2a_out)])
        a2a = {"in_ms": statistics.median(a2a_in), "out_ms": statistics.median(a2a_out),
               "sent_bytes_per_rank": sent, "gbs_per_rank": sent / (a2a_ms * 1e-3) / 1e9 if a2a_ms > 0 else None,
               "vs_nvlink_900": (sent / (a2a_ms * 1e-3) / 1e9) / NVLINK_GBS if a2a_ms > 0 else None}
    roof_t = max(flops / P / (peak * 1e12), (_a2a_send_bytes(plan, rank) if P > 1 else 0) / (NVLINK_GBS * 1e9))
    overlapped = {"t_roofline_ms": roof_t * 1e3, "frac": roof_t * 1e3 / t_max,
                  "formula": "max(4BS^2HD/(P*peak_bf16), a2a bytes sent per rank / 900 GB/s)"}

    # end-to-end through the public API with host buffers: H2D inputs, the call, D2H output.  One GPU: the
    # library's host-buffer call (spa_attention_host), which overlaps head group i's attention with group i+1's
    # H2D and group i-1's D2H; N GPUs: H2D, the SP call, D2H in sequence.
    e2e = None
    if args.qkv:
        pass   # e2e of the hidden-state layer: not separately measured (the attention-only line carries e2e)
    elif not args.no_e2e and P == 1:
        hq = [x.cpu().pin_memory() for x in qkv]
        hout = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
        hplan = spa.Plan(comm, B, S, H, D, stages=args.host_groups)
        hws = torch.empty(hplan.host_workspace_bytes, dtype=torch.uint8, device=dev)
        for _ in range(2):
            spa.spa_attention_host(hplan, *hq, hout, hws, stream)
        barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for i in range(args.steps):
            ev[i][0].record(stream)
            spa.spa_attention_host(hplan, *hq, hout, hws, stream)
            ev[i][1].record(stream)
        barrier()
        te = statistics.median([a.elapsed_time(b) for a, b in ev])
        e2e = {"value": flops / (te * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": te,
               "h2d_bytes_per_step": sum(x.numel() * x.element_size() for x in hq),
               "d2h_bytes_per_step": hout.numel() * hout.element_size(),
               "path": f"spa_attention_host, {hplan.stage_split[0]} head groups pipelined H2D / attention / D2H"}
        hplan.close()
        del hws
    elif not args.no_e2e:
        # N ranks: the library's host-buffer SP call (spa_pipesp_attention_hostbuf): per head group, the H2D of its
        # columns and the D2H of its output overlap the other groups' exchange and attention
        hq = [x.cpu().pin_memory() for x in qkv]
        hout = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
        hplan = spa.Plan(comm, B, S, H, D, stages=stages)
        hws = p2p_setup(hplan, torch.empty(hplan.host_sp_workspace_bytes, dtype=torch.uint8, device=dev))
        for _ in range(2):
            spa.spa_pipesp_attention_hostbuf(hplan, *hq, hout, hws, stream)
        barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for i in range(args.steps):
            ev[i][0].record(stream)
            spa.spa_pipesp_attention_hostbuf(hplan, *hq, hout, hws, stream)
            ev[i][1].record(stream)
        barrier()
        te = max_over_ranks(statistics.median([a.elapsed_time(b) for a, b in ev]))
        e2e = {"value": flops / (te * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": te,
               "h2d_bytes_per_step": sum(x.numel() * x.element_size() for x in hq),
               "d2h_bytes_per_step": hout.numel() * hout.element_size(),
               "path": f"per rank: spa_pipesp_attention_hostbuf, {split_of(hplan)} head groups pipelined "
                       f"H2D / exchange / attention / D2H (max over ranks)"}
        hplan.close()
        del hws

    # roofline of the dominant kernel (attention): algorithmic FLOPs per launch / measured duration
    rank_attn_flops = attn_flops(B, S, H, D) / P
    attn_ms_med = statistics.median(attn_ms)
    achieved = rank_attn_flops / (attn_ms_med * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(f"{name}/P{P}/D{D}")
    except Exception:
        pass
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": f"{peak_src} bf16_tflops (burst cuBLAS 8192^3)",
                "frac_of_sustained": achieved / peaks.get("bf16_tflops_sustained", peak),
                "frac_of_datasheet_2250": achieved / 2250.0, "kernel": "attn_fwd_kernel (tcgen05)",
                "attn_ms_per_step": attn_ms_med,
                "algorithmic": f"4*B*S^2*H*D/P = {rank_attn_flops:.4g} FLOP per rank per step"}
    split = list(plan.stage_split)
    plan.close()
    del ws, qkv, out

    # ---------------------------------------------------------------- north-star block (720p, N_st sweep)
    north = None
    if args.north_star == 1 or (args.north_star == -1 and P == 8):
        wn = synthgen.WORKLOADS["hy720p129f"]
        fl = attn_flops(wn.B, wn.S, wn.H, wn.D)
        n = max(3, min(args.steps, 10))
        sweep = []
        for st in NORTH_STAR_STAGES:
            pl, x, o, w_ = make("hy720p129f", st)
            ms, pr = timed(pl, x, o, w_, n, 3, True)
            t = max_over_ranks(statistics.median(ms))
            ex, tnc = exposed_pct(pl, x, o, w_, t, n) if P > 1 else (0.0, t)
            sent = _a2a_send_bytes(pl, rank) if P > 1 else 0
            a2a_ms = statistics.median([sum(p.a2a_in_ms[k] + p.a2a_out_ms[k] for k in range(p.n_stages)) for p in pr])
            troof = max(fl / P / (peak * 1e12), sent / (NVLINK_GBS * 1e9)) * 1e3
            sweep.append({"stages": st, "stage_split": list(pl.stage_split), "ms_per_layer": t,
                          "tflops": fl / (t * 1e-3) / 1e12, "exposed_a2a_pct": ex, "ms_skip_comm": tnc,
                          "a2a_gbs_per_rank": max_over_ranks(sent / (a2a_ms * 1e-3) / 1e9) if a2a_ms > 0 else None,
                          "frac_overlapped_roofline": troof / t, "t_roofline_ms": troof})
            pl.close()
            del x, o, w_
        best = min(sweep, key=lambda r: r["ms_per_layer"])
        north = {"workload": "hy720p129f", "P": P, "best": best, "sweep": sweep,
                 "target": ">= 0.60 of the overlapped roofline, <= 10 % exposed all-to-all (BASELINE.json)"}

    # ---------------------------------------------------------------- north star, one rank's share (N = 1)
    # BASELINE configs[3] (720p, P = 8) cannot run on one GPU; its per-rank schedule can: a loopback plan over 8 virtual
    # ranks with SPA_OPT_RANK_ONLY runs only rank 0's launches and the messages rank 0 sends or receives through the
    # real scheduler (tools/rank_schedule.py).  Labelled as such; not the bench value.
    def extra(fn, *a):   # informational blocks: a failure there is reported in the line, never fatal to the bench
        try:
            return fn(*a)
        except Exception as e:  # pragma: no cover
            torch.cuda.synchronize()
            return {"error": f"{type(e).__name__}: {str(e)[:200]}"}

    one_rank = aco = other = None
    if P == 1 and not args.no_one_rank and not args.qkv:
        one_rank = extra(north_star_one_rank, spa, synthgen, torch, peak, flush)
        aco = extra(aco_one_rank, spa, synthgen, torch, flush)
    if P == 1 and not args.qkv and name != "osp480p93f":   # configs[1] on this GPU, next to the headline
        other = extra(single_gpu_config, spa, synthgen, torch, peak, flush)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = time_oracle(S, D, args.cpu_seconds)
        cpu.pop("seconds", None)
        cpu.pop("rows", None)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded splitmix64 Irwin-Hall, D0, seed 0)",
            "config": {"workload": name + ("+qkv" if args.qkv else ""), "B": B, "S": S, "H": H, "D": D, "P": P,
                       "stages": stages,
                       "stage_split": split,
                       "parallelism": f"ulysses-sp{P} (PipeSP)" if P > 1 else "single",
                       "transport": (args.transport + ("-direct" if args.direct else "")) if P > 1 else None,
                       "timing": "median of per-step CUDA events, max over ranks",
                       "l2": "flushed between timed steps (256 MiB memset, untimed); inputs > L2"},
            "exposed_a2a_pct": exposed, "ms_skip_comm": t_nocomm, "a2a": a2a, "overlapped_roofline": overlapped,
            "clocks": clk.summary(), "e2e": e2e, "gpu_launches": launches,
            "roofline": roofline, "cpu_baseline": cpu, "north_star": north, "qkv_projection": qkv_info,
            "north_star_one_rank": one_rank, "aco_one_rank": aco, "osp_single_gpu": other,
        }
        print(json.dumps(line), flush=True)
    comm.close()
    if world > 1:
        dist.destroy_process_group()


def spawn(args) -> int:
    """N > 1 without a launcher: re-run this script under torch.distributed.run, one rank per GPU."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    argv = [a for a in sys.argv[1:] if a != "--spawn"]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif "WORLD_SIZE" not in os.environ and (args.gpus > 1 or args.spawn):
        sys.exit(spawn(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
