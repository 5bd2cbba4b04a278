#!/usr/bin/env python3
"""Benchmark: seconds per 256^3-particle periodic FMM velocity + stretching evaluation.

BASELINE.json metric "s per 256^3-particle FMM velocity+stretching eval; P2P interactions/s,
%FP32 peak" on configuration c4 (256^3 isotropic Re_lambda = 50 field, overlap 1, p = 10,
depth 6, 27^3 periodic images).  A step is one whole evaluate() (Morton keys, radix sort,
gather, P2M, M2M, M2L, periodic images, L2L, P2P, L2P + un-permute) on inputs resident in
HBM (403 MB of inputs, larger than the 126 MB L2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4]

--impl reference times the CPU oracle (oracle/, float64 direct periodic sum) on a bounded
sample of the same workload (the tier's reference arm; extrapolated to a full evaluation).
Under torchrun (N > 1) the ONE 256^3 problem is split across the ranks by Morton range
(vfmm_partition) and evaluated with the halo-particle + LET exchange over NCCL
(DESIGN.md "Multi-GPU"): strong scaling, value = seconds per whole evaluation (max over ranks).
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

METRIC = "s per 256³-particle FMM velocity+stretching eval; P2P interactions/s, %FP32 peak"
PAPER_CONTEXT = ("paper: ~20 s/time step at p=10 (~10 s at p=6) on one Tesla C2070, FP32, "
                 "N=256^3, 27^3 images (PAPER.md:174-176); hit3d ~1 s/step on 6 Xeon E5650 cores")
P2P_FLOP_PER_PAIR = 69  # 3 FADD + 16 FMUL + 25 FFMA per pair (FFMA = 2), independent of the kernel variant


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 4 + k and "Active" in r[4 + k] and "Not" not in r[4 + k]:
                    reasons.add(nm)
        pw = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(pw) if pw else None}


def host_cpu():
    """lscpu model / sockets / cores of this host (recorded with the CPU baseline)."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            k = k.strip()
            if k in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                info[k] = v.strip()
    except Exception:
        pass
    return info


def cpu_baseline(field, p_unused, budget_s=15.0, threads=None):
    """Oracle O1 (float64 direct periodic sum, oracle/) on a bounded sample: T targets x a
    strided subset of sources x all 27^3 images; extrapolated to the full evaluation."""
    import numpy as np

    import oracle

    n = field.pos.shape[1]
    threads = threads or os.cpu_count() or 1
    stride = 512
    src = np.arange(0, n, stride)
    tg = np.arange(7, n, n // 4)[:4]
    pos_s = field.pos[:, src]
    gam_s = field.gamma[:, src]
    # calibrate on one target, then size the sample to ~budget_s
    t0 = time.perf_counter()
    oracle.direct(pos_s, gam_s, field.sigma, field.box_lo, field.box_len, 3, 0,
                  probe_pos=field.pos[:, tg[:1]].astype(np.float64),
                  probe_gamma=field.gamma[:, tg[:1]].astype(np.float64), nthreads=1)
    t1 = time.perf_counter() - t0
    # at least one target per thread, so every core works
    ntg = max(threads, min(256, int(budget_s / max(t1, 1e-6) * threads * 0.8)))
    tg = np.linspace(7, n - 1, ntg).astype(np.int64)
    t0 = time.perf_counter()
    oracle.direct(pos_s, gam_s, field.sigma, field.box_lo, field.box_len, 3, 0,
                  probe_pos=field.pos[:, tg].astype(np.float64),
                  probe_gamma=field.gamma[:, tg].astype(np.float64), nthreads=threads)
    dt = time.perf_counter() - t0
    pairs_sample = len(tg) * len(src) * 27 ** 3
    pairs_full = n * n * 27 ** 3
    return {"value": dt * pairs_full / pairs_sample, "unit": "s/eval (extrapolated)",
            "cores": threads, "kind": "oracle", "host_cpu": host_cpu(),
            "sample": (f"{len(tg)} targets x {len(src)} sources (every {stride}th) x 27^3 "
                       f"images = {pairs_sample:.3e} pair evals in {dt:.2f} s; scaled by "
                       f"{pairs_full / pairs_sample:.3e} to N^2 27^3")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import synthgen

    f = synthgen.make(args.config)
    vals = []
    cb = None
    for _ in range(args.warmup + args.steps):
        cb = cpu_baseline(f, None, budget_s=args.ref_budget)
        vals.append(cb["value"])
    v = statistics.median(vals[args.warmup:]) if args.steps else vals[-1]
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, f), "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, f):
    import synthgen

    c = synthgen.CONFIGS[args.config]
    return {"workload": f"{args.config}: {f.n}^3 lattice particles, {f.name}, overlap h/sigma=1, "
                        f"p={args.p or c['p']}, depth {args.depth or c['depth']}, 27^3 periodic images",
            "n": int(f.pos.shape[1]), "p": args.p or c["p"], "depth": args.depth or c["depth"],
            "image_levels": 3, "scheme": "classical",
            "l2": "inputs (403 MB at 256^3) and working set larger than the 126 MB L2",
            "parallelism": f"morton-partition+LET x{args.gpus}" if args.gpus > 1 else "single"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--p", type=int, default=0)
    ap.add_argument("--depth", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-accurate", action="store_true",
                    help="skip the p = 13 (north_star accuracy) timing that follows the main line")
    ap.add_argument("--ref-budget", type=float, default=8.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import synthgen
    import paper_1110_2921_b200 as vf

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = synthgen.CONFIGS[args.config]
    p = args.p or cfg["p"]
    depth = args.depth or cfg["depth"]
    f = synthgen.make(args.config)
    n_total = f.pos.shape[1]
    kw = dict(p=p, depth=depth, image_levels=3, sigma=f.sigma, box_lo=f.box_lo,
              box_len=f.box_len)
    if world > 1:
        # this rank's share of the one problem: a contiguous chunk of the input order (particles
        # anywhere in the box); the library redistributes them to their Morton owners and
        # returns the results
        lo = n_total * rank // world
        hi = n_total * (rank + 1) // world
        f.pos = np.ascontiguousarray(f.pos[:, lo:hi])
        f.gamma = np.ascontiguousarray(f.gamma[:, lo:hi])
        ev = vf.init_distributed(**kw)
    else:
        ev = vf.Evaluator(device=local, **kw)
    n = f.pos.shape[1]
    dev = torch.device("cuda", local)
    pos = torch.from_numpy(f.pos).to(dev)
    gam = torch.from_numpy(f.gamma).to(dev)
    vel = torch.empty_like(pos)
    dg = torch.empty_like(pos)
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(args.warmup, 0)):
        ev.evaluate_into(pos, gam, vel, dg, stream)
    ev.sync_status()
    torch.cuda.synchronize()

    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        ev.evaluate_into(pos, gam, vel, dg, stream)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / max(args.steps, 1)
    ev.sync_status()
    # per-phase CUDA-event times (library events on this stream) of the last timed step
    phases = [ev.stats()]

    # ---- e2e: host (pinned) in, host out, through the public C API ----
    e2e = None
    if not args.no_e2e:
        hp = torch.from_numpy(f.pos).pin_memory()
        hg = torch.from_numpy(f.gamma).pin_memory()
        hv = torch.empty_like(hp).pin_memory()
        hs = torch.empty_like(hp).pin_memory()
        ev.evaluate_host_ptr(n, hp.data_ptr(), hg.data_ptr(), hv.data_ptr(), hs.data_ptr())
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ev.evaluate_host_ptr(n, hp.data_ptr(), hg.data_ptr(), hv.data_ptr(), hs.data_ptr())
        te = torch.tensor([(time.perf_counter() - t0) / max(args.steps, 1)], device=dev,
                          dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": float(te.item()), "unit": "s",
               "h2d_bytes_per_step": int(hp.numel() * 4 + hg.numel() * 4),
               "d2h_bytes_per_step": int(hv.numel() * 4 + hs.numel() * 4)}

    # the configuration that meets north_star's accuracy target (u <= 1e-5, sdot <= 3e-5 vs
    # the direct sum at 27^3 images takes p = 13 with ws = 1), timed the
    # same way on the same inputs after the main measurement
    accurate = None
    if world == 1 and not args.no_accurate and args.config in ("c4", "c5") and p == 10:
        ev13 = vf.Evaluator(device=local, **dict(kw, p=13))
        for _ in range(2):
            ev13.evaluate_into(pos, gam, vel, dg, stream)
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        ka = max(2, min(args.steps, 5))
        a0.record(stream)
        for _ in range(ka):
            ev13.evaluate_into(pos, gam, vel, dg, stream)
        a1.record(stream)
        torch.cuda.synchronize()
        ev13.sync_status()
        st13 = ev13.stats()
        accurate = {"p": 13, "ms_per_step": a0.elapsed_time(a1) / ka, "steps": ka,
                    "phase_ms": {k[3:]: round(v, 4) for k, v in st13.items()
                                 if k.startswith("ms_") and v},
                    "accuracy": "u <= 1e-5, dgamma/dt <= 3e-5 relative L2 vs the direct sum at "
                                "27^3 images (tests/test_gpu_parity.py::"
                                "test_north_star_accuracy_p13_27cubed_vs_direct)"}
        ev13.close()

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel ----
    peaks = load_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12  # TFLOP/s
    nc = (p + 1) ** 2
    avg = {k: statistics.mean(ph[k] for ph in phases) for k in phases[0]}
    t_p2p = max(avg["ms_p2p"], 1e-9) * 1e-3  # per-kernel events exist on single-rank contexts
    t_m2l = max(avg["ms_m2l"], 1e-9) * 1e-3
    pairs = phases[0]["n_p2p_pairs"] or 27 * 64 * n_total
    p2p_tf = pairs * P2P_FLOP_PER_PAIR / t_p2p / 1e12
    m2l_tf = phases[0]["n_m2l"] * 6 * nc * nc / t_m2l / 1e12
    engine = os.environ.get("VFMM_M2L", "f16")  # same selection as the library (capi.cu)
    tc_m2l = p <= 10 and depth >= 2 and engine != "simt"  # levels >= 2 run M2L on tcgen05
    bf16 = float(peaks.get("bf16_tflops", 1630.5))
    if engine == "tf32":
        tc_peak, tc_note, tc_split = bf16 * (1.1 / 2.25), \
            "measured bf16 burst x nominal tf32/bf16 (1.1/2.25 PF)", "3xTF32"
    else:  # kind::f16 runs at the dense fp16/bf16 rate
        tc_peak, tc_note, tc_split = bf16, "measured bf16 burst (fp16 dense = bf16 dense rate)", \
            "scaled 3xFP16"
    if t_m2l >= t_p2p:
        if tc_m2l:
            roof = {"kernel": f"m2l (m2l_tc_kernel tcgen05 {tc_split} at levels >= 2, SIMT level 1)",
                    "bound": "tensor", "achieved": m2l_tf, "peak": tc_peak, "unit": "TFLOP/s",
                    "frac": m2l_tf / tc_peak, "traffic": None,
                    "per_unit": f"6(p+1)^4 = {6 * nc * nc} useful flop per M2L translation; "
                                f"{tc_split} issues 3 tensor products per useful product",
                    "peak_note": tc_note}
        else:
            roof = {"kernel": "m2l (translate_kernel<M2L>, all levels)", "bound": "alu",
                    "achieved": m2l_tf, "peak": fp32_peak, "unit": "TFLOP/s",
                    "frac": m2l_tf / fp32_peak, "traffic": None,
                    "per_unit": f"6(p+1)^4 = {6 * nc * nc} flop per M2L translation"}
    else:
        roof = {"kernel": "p2p_kernel", "bound": "alu", "achieved": p2p_tf, "peak": fp32_peak,
                "unit": "TFLOP/s", "frac": p2p_tf / fp32_peak, "traffic": None,
                "per_unit": f"{P2P_FLOP_PER_PAIR} FP32 flop per ordered pair"}
    if world > 1:  # distributed contexts time whole phases only: roofline comes from N = 1
        roof.update(achieved=None, frac=None, note="per-kernel events measured at n_gpus=1")
    roof.setdefault("peak_source", f"FP32 SIMT: 148 SMs x 128 lanes x 2 x {sm_max:.0f} MHz "
                                   "(sm_max_mhz of MEASURED_PEAKS.json)")
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        try:
            tr = json.load(open(tr_path))
            key = "m2l" if roof["kernel"].startswith("m2l") else "p2p"
            roof["traffic"] = tr.get(key)
        except Exception:
            pass

    cb = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cb = cpu_baseline(f, p)
        except Exception as e:  # oracle not built: say so
            cb = {"value": None, "unit": "s/eval", "cores": os.cpu_count(), "kind": "oracle",
                  "sample": f"unavailable: {e}"}

    s_per_eval = ms_step * 1e-3  # one whole 256^3 evaluation per step (max over ranks)
    line = {
        "metric": METRIC, "value": s_per_eval, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": False, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f32", "data": "synthetic", "config": workload_config(args, f),
        "p2p_interactions_per_s": pairs / t_p2p,
        "p2p_pairs_per_eval": pairs,
        "fp32_frac_p2p": p2p_tf / fp32_peak, "m2l_useful_tflops": m2l_tf,
        "m2l_engine": engine if tc_m2l else "simt",
        "p2p_variant": "cross" if os.environ.get("VFMM_P2P") == "cross" else "sj",
        "phase_ms": {k[3:]: round(v, 4) for k, v in avg.items() if k.startswith("ms_")},
        "roofline": roof, "cpu_baseline": cb, "e2e": e2e,
        "gpu_launches": int(phases[0]["n_kernel_launches"]) * args.steps,
        "accurate_config": accurate,
        "clocks": clocks, "paper_context": PAPER_CONTEXT,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
