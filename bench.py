#!/usr/bin/env python
"""Benchmark of the B200 Fast Guided Filter (BASELINE.json metric: output Mpixel/s at s=4
and achieved HBM GB/s vs peak).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fgf|reference]
                    [--config 4] [--s 4]

A step is one pass of the whole hot path (Alg. 2, all five stages) over one batch of the
workload: by default BASELINE.json config 4 (256 x 4096^2 gray, r=32, eps=0.01, s=4,
nearest), one C-ABI call (fgf_filter_ws) per step.  N > 1 runs one process per GPU under
torchrun; each rank filters its own 256 images (weak scaling, no collective on the data
path); the time is the max over ranks.  Rank 0 prints one JSON line.

--impl reference times the fp64 CPU oracle (oracle/) on the host cores on a bounded sample
of the same workload (one image per step) and prints the same line with "impl": "reference".
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "output Mpixel/s (FGF s=4)"
UNIT = "Mpixel/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["fgf", "reference"], default="fgf")
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--s", type=int, default=None)
    ap.add_argument("--batch", type=int, default=None, help="override the config batch per GPU")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="replay each step from a CUDA graph (small single-image configs: no "
                         "per-launch host overhead)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dtype", choices=["f32", "f16", "bf16", "u8"], default="f32",
                    help="element type of I, p, q (f16 / bf16: the reduced-precision I/O variant)")
    ap.add_argument("--band-mode", choices=["single", "two-step"], default="single",
                    help="config 5: one 2r'+1-row exchange of I', p', or r' rows then r'+1 rows of a, b")
    ap.add_argument("--band-impl", choices=["c", "torch"], default="c",
                    help="config 5 (4b): C-ABI band call with NCCL inside, or the Python stages")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id):
        self.rows = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", gpu_id, f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = [r for (t, r) in self.rows if t0 <= t <= t1] or [r for (_, r) in self.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower() == "active"})
        pw = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w_max": max(pw) if pw else None, "samples": len(rows)}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_oracle_images(cfg, prm, count, first=0):
    """fp64 oracle (test infrastructure) on `count` images of config cfg; returns (seconds, px)."""
    import oracle
    import synth
    secs, px = 0.0, 0
    for i in range(count):
        I, p = synth.make_image(cfg, first + i, "cpu")
        In, pn = I.numpy()[None], p.numpy()[None]
        t0 = time.perf_counter()
        oracle.fast_guided_filter(In, pn, prm["r"], prm["eps"], prm["s"], prm["sub_mode"])
        secs += time.perf_counter() - t0
        px += In.shape[-1] * In.shape[-2]
    return secs, px


def cpu_baseline(cfg, prm, budget_s=12.0):
    """Oracle as it stands on the host cores: images of the workload until ~budget_s."""
    import oracle
    oracle.build()
    secs, px, n = 0.0, 0, 0
    while secs < budget_s and n < 64:
        s1, p1 = run_oracle_images(cfg, prm, 1, first=n)
        secs += s1
        px += p1
        n += 1
    return {"value": px / secs / 1e6, "unit": UNIT, "cores": host_cores(), "kind": "oracle",
            "cpu": cpu_model(),
            "sample": f"{n} image(s) of the workload (full 5-stage FGF per image, fp64), "
                      f"{secs:.1f} s of CPU work, OpenMP over all host cores"}


def workload(cfg, s_over, batch_over):
    import synth
    c = dict(synth.CONFIGS[cfg])
    prm = synth.params(cfg, **({"s": s_over} if s_over else {}))
    B = batch_over or c["batch"]
    return c, prm, B


def config_json(c, prm, B, ngpu):
    return {"workload": c["name"], "batch_per_gpu": B, "global_batch": B * ngpu, "H": c["H"],
            "W": c["W"], "C_I": c["C_I"], "C_p": c["C_p"], "r": prm["r"], "eps": prm["eps"],
            "s": prm["s"], "sub_mode": "nearest" if prm["sub_mode"] == 0 else "bilinear(block mean)",
            "parallelism": f"batch shard x{ngpu}, no collective",
            "l2": "inputs larger than L2 (no flush needed)"}


def reference_main(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # the oracle arm runs on rank 0 only
    c, prm, B = workload(args.config, args.s, args.batch)
    import oracle
    oracle.build()
    for i in range(args.warmup):
        run_oracle_images(args.config, prm, 1, first=i)
    secs, px = 0.0, 0
    for i in range(args.steps):
        s1, p1 = run_oracle_images(args.config, prm, 1, first=args.warmup + i)
        secs += s1
        px += p1
    value = px / secs / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_json(c, prm, B, args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": host_cores(), "kind": "oracle",
                             "cpu": cpu_model(),
                             "sample": "one image of the workload per step (bounded sample)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return reference_main(args)

    import torch
    import torch.distributed as dist

    import paper_1505_00996_b200 as fgf
    import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    if args.config == 5:
        return band_main(args, fgf, torch, dist, world, rank, local, dev, barrier)

    c, prm, B = workload(args.config, args.s, args.batch)
    H, W, CI, CP = c["H"], c["W"], c["C_I"], c["C_p"]
    r, eps, s, sub = prm["r"], prm["eps"], prm["s"], prm["sub_mode"]
    N = H * W
    h, w = -(-H // s), -(-W // s)
    n = h * w
    NC = (CI + 1) * CP

    # Inputs resident in HBM before timing; rank k owns global images [k*B, (k+1)*B).
    I, p = synth.make_batch(args.config, dev, batch=B, first=rank * B)
    # --dtype f16 / bf16 / u8: the reduced-precision I/O variant (fgf_filter_ex_ws; not the
    # BASELINE.json configuration, which is fp32)
    tdt = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16,
           "u8": torch.uint8}[args.dtype]
    code = {"f32": fgf.FGF_F32, "f16": fgf.FGF_F16, "bf16": fgf.FGF_BF16, "u8": fgf.FGF_U8}[args.dtype]
    esize = {"f32": 4, "f16": 2, "bf16": 2, "u8": 1}[args.dtype]
    if args.dtype != "f32":
        same = p is I
        if args.dtype == "u8":   # 8-bit codes k / 255 (R19)
            conv = lambda t: torch.round(t.clamp(0, 1) * 255.0).to(torch.uint8).contiguous()
        else:
            conv = lambda t: t.to(tdt).contiguous()
        I = conv(I)
        p = I if same else conv(p)
    q = torch.empty((B, CP, H, W), dtype=tdt, device=dev)
    ws_bytes = fgf.fgf_workspace_bytes_ex(B, H, W, CI, CP, r, s, code)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    # the library's own stream discipline: every call on one non-default stream (small calls
    # are then replayed from the library's CUDA-graph cache; the legacy default stream is not
    # capturable)
    torch.cuda.synchronize()
    stream = torch.cuda.Stream(dev)

    def step(st=stream):
        if args.dtype == "f32":
            fgf.fgf_filter_ws(I, p, q, B, H, W, CI, CP, r, eps, s, sub, ws, ws_bytes, st)
        else:
            fgf.fgf_filter_ex_ws(I, p, q, B, H, W, CI, CP, r, eps, s, sub, code, ws, ws_bytes,
                                 st)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    launches_per_step = fgf.fgf_last_launch_count()
    eager_step = step
    if args.graph:
        # the same call captured once; each timed step replays it on `stream`
        gstream = torch.cuda.Stream(dev)
        gstream.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gstream):
            step(gstream)
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        def step(st=stream):
            # replay on the timed stream (CUDAGraph.replay launches on the current stream)
            with torch.cuda.stream(st):
                graph.replay()

    props = torch.cuda.get_device_properties(dev)
    gpu_id = "GPU-" + str(props.uuid) if getattr(props, "uuid", None) else str(local)
    sampler = ClockSampler(gpu_id)
    time.sleep(0.3)

    # ---------------- timed region: K steps, barrier + sync on both sides, max over ranks.
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    t_host0 = time.time()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    t_host1 = time.time()
    t_ms = e0.elapsed_time(e1)
    time.sleep(0.15)
    sampler.stop()
    clocks = sampler.summary(t_host0, t_host1)
    tmax = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    t_ms = float(tmax.item())
    ms_per_step = t_ms / args.steps
    value = world * B * N / (t_ms / 1e3 / args.steps) / 1e6

    # ---------------- per-kernel CUDA events over the same K steps (diagnostic pass).
    fgf.fgf_profile_enable(True)
    for _ in range(args.steps):
        eager_step()        # the library records its events at enqueue time (not in a graph)
    torch.cuda.synchronize()
    prof = fgf.fgf_profile_read()
    fgf.fgf_profile_enable(False)
    kern = {k: {"ms_per_launch": (v[0] / v[1]) if v[1] else 0.0,
                "launches_per_step": v[1] / args.steps,
                "share_of_kernel_time": 0.0} for k, v in prof.items()}
    tot = sum(v[0] for v in prof.values()) or 1.0
    for k, v in prof.items():
        kern[k]["share_of_kernel_time"] = v[0] / tot
    # K13 (fused low-res chain): algorithmic DRAM bytes per step = the nearest sample rows of I
    # and p (every s-th row, all of its sectors for s <= 8) + the mean maps written; it is
    # issue/latency-bound, not HBM-bound, so this is context, not a roofline.
    if "lowres_fused" in kern and prof["lowres_fused"][1]:
        planes_in = CI + (0 if args.config == 0 else CP)
        if sub == 0:      # samples read in place from the full-resolution rows
            k13_bytes = B * (esize * N * planes_in / s + 4 * NC * n)
        else:             # K0's compact fp32 planes
            k13_bytes = B * (4 * n * planes_in + 4 * NC * n)
        k13_ms = prof["lowres_fused"][0] / args.steps
        kern["lowres_fused"]["alg_bytes_per_step"] = k13_bytes
        kern["lowres_fused"]["alg_GBs"] = k13_bytes / (k13_ms / 1e3) / 1e9
        # its real bound: instruction issue (warp-instructions per image from the committed
        # ncu capture) against 148 SMs x 4 schedulers x the SM clock seen during the run
        try:
            ij = json.load(open(os.path.join(ROOT, "profiles", "k13_instructions.json")))
            key = f"{c['name']}_s{s}"
            if key in ij and args.dtype == "f32":
                mhz = (clocks or {}).get("sm_mhz") or 1965.0
                rate = ij[key]["warp_instructions_per_image"] * B / (k13_ms / 1e3)
                peak_issue = 148 * 4 * mhz * 1e6
                kern["lowres_fused"]["issue"] = {
                    "bound": "issue", "achieved": rate, "peak": peak_issue,
                    "unit": "warp-instr/s", "frac": rate / peak_issue,
                    "source": "profiles/k13_instructions.json"}
        except Exception:
            pass

    peak, peak_src = peaks()
    # Roofline of the dominant kernel (largest share of the step's kernel time): algorithmic
    # bytes per launch / its CUDA-event time per launch.
    #   K4 upsample + output: read I (esize C_I N) + write q (esize C_p N) + read maps (4 NC n)
    #   K5 at s = 1 (Alg. 1 fused): read I and p, write q (esize N (C_I + C_p + C_p); p = I
    #     read once when self-guided)
    #   K13 / K5 low-res chain: sample rows of I, p (1/s of the rows, or K0's compact planes)
    #     + the mean maps written (4 NC n)
    planes_in = CI + (0 if args.config == 0 else CP)
    lowres_bytes = B * ((esize * N * planes_in / s) if sub == 0 else (4 * n * planes_in)) \
        + B * 4 * NC * n
    alg = {"upsample_output": B * (esize * CI * N + esize * CP * N + 4 * NC * n),
           "lowres_fused": lowres_bytes,
           "wide_fused": (B * esize * N * (planes_in + CP)) if s == 1 else lowres_bytes,
           # K6 (whole filter of a small image in one kernel): read I once (its sample rows
           # are part of it), the sample rows of p (all of p for block means), write q
           "tiny_fused": B * esize * N * (CI + CP + (0 if args.config == 0 else
                                                     (CP / s if sub == 0 else CP)))}
    names = {"upsample_output": "output_kernel (K4: bilinear upsample + q = A.I + B)",
             "lowres_fused": "lowres_gray_kernel (K13: fused low-res chain)",
             "wide_fused": ("wide_gray_kernel (K5: exact guided filter, Alg. 1, one kernel)"
                            if s == 1 else "wide_gray_kernel (K5: wide-window low-res chain)"),
             "tiny_fused": "tiny_gray_kernel (K6: whole filter of a small image, one kernel)"}
    dom = max((k for k in prof if prof[k][1] and k in alg), key=lambda k: prof[k][0], default=None)
    roofline = None
    if dom is not None:
        d_ms, d_n = prof[dom]
        d_bytes = alg[dom] / (d_n / args.steps)          # per launch
        d_gbs = d_bytes / (d_ms / d_n / 1e3) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "k4_traffic.json" if dom == "upsample_output"
                             else f"{dom}_traffic.json")
        if os.path.exists(tpath):
            try:
                tj = json.load(open(tpath))
                key = f"{c['name']}_s{s}"
                if key in tj and args.dtype == "f32":
                    traffic = tj[key]["dram_bytes_per_image"] * B / (d_n / args.steps)
            except Exception:
                traffic = None
        roofline = {"bound": "hbm", "kernel": names[dom], "achieved": d_gbs, "peak": peak,
                    "peak_source": peak_src, "unit": "GB/s", "frac": d_gbs / peak,
                    "traffic": traffic, "alg_bytes_per_launch": d_bytes,
                    "share_of_step": d_ms / tot}
    # Whole filter against BASELINE's byte model (read I and p, write q, + low-res traffic).
    B_model = B * (esize * N * (CI + 2 * CP) + 8 * n * NC)
    rho = 1.0 if (s == 1 or sub == 1) else 1.0 / min(s, 8)
    B_alg = B * esize * N * (CI + rho * CP + CP)
    whole = {"B_model_per_step": B_model, "B_alg_per_step": B_alg,
             "model_GBs": B_model / (ms_per_step / 1e3) / 1e9,
             "alg_GBs": B_alg / (ms_per_step / 1e3) / 1e9}
    whole["frac_model_of_8000"] = whole["model_GBs"] / 8000.0
    whole["frac_model_of_measured"] = whole["model_GBs"] / peak
    whole["frac_alg_of_measured"] = whole["alg_GBs"] / peak

    # ---------------- e2e: host buffers through fgf_filter_host (H2D + filter + D2H inside).
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(fgf, torch, dist, world, rank, local, args, c, prm, B, tdt, code, esize)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, prm)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": args.dtype, "data": "synthetic",
                "config": dict(config_json(c, prm, B, world), io_dtype=args.dtype,
                               cuda_graph=bool(args.graph)),
                "gpu_launches": launches_per_step * args.steps,
                "roofline": roofline, "hbm_whole_filter": whole, "kernels": kern,
                "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu,
                "device": props.name}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def band_main(args, fgf, torch, dist, world, rank, local, dev, barrier):
    """BASELINE.json config 4b: ONE 16384^2 image split into row bands across the ranks, with
    the 2r'+1-row low-res halo exchanged over torch.distributed P2P (NCCL over NVLink).  Strong
    scaling (the image is fixed); value = the image's pixels / max-over-ranks step time."""
    import synth
    from paper_1505_00996_b200 import bands
    c, prm, _ = workload(5, args.s, None)
    H, W = c["H"], c["W"]
    r, eps, s, sub = prm["r"], prm["eps"], prm["s"], prm["sub_mode"]
    pl = bands.plan_band(H, W, r, s, world, rank)
    I, p = synth.make_batch(5, dev)
    I_own = I[:, :, pl.Y0:pl.Y1].contiguous()
    p_own = p[:, :, pl.Y0:pl.Y1].contiguous()
    del I, p
    stream = torch.cuda.current_stream(dev)
    comm = None
    if args.band_impl == "c":
        # fgf_filter_band: subsample, NCCL halo exchange and the rest inside libfgf.so; the
        # NCCL unique id travels over the torch.distributed process group
        if world > 1:
            uid = [fgf.fgf_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            comm = fgf.fgf_nccl_comm_init(uid[0], rank, world)
        rows = pl.Y1 - pl.Y0
        q_own = torch.empty_like(p_own)
        nb = fgf.fgf_band_workspace_bytes(H, W, pl.Y0, rows, 1, 1, r, s, world)
        ws = torch.empty(nb, dtype=torch.uint8, device=dev)

        mode = fgf.FGF_BAND_TWO_STEP if args.band_mode == "two-step" else fgf.FGF_BAND_SINGLE

        def step():
            fgf.fgf_filter_band_ex(I_own, p_own, q_own, H, W, pl.Y0, rows, 1, 1, r, eps, s, sub,
                                   mode, comm, rank, world, ws, nb, stream)
            return q_own
    else:
        ex = bands.DistExchange(rank, world)
        backend = bands.GpuBackend()

        def step():
            return bands.filter_band(I_own, p_own, r, eps, s, sub, H, rank, world, ex, backend)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps
    if rank == 0:
        line = {"metric": METRIC, "value": H * W / (ms / 1e3) / 1e6, "unit": UNIT,
                "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
                "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": c["name"], "H": H, "W": W, "r": r, "eps": eps, "s": s,
                           "parallelism": f"row bands x{world}, halo {pl.halo} low-res rows "
                                          + (f"fgf_filter_band_ex {args.band_mode} (NCCL P2P inside libfgf.so)"
                                             if args.band_impl == "c" else
                                             "over torch.distributed P2P"),
                           "l2": "inputs larger than L2 (no flush needed)"}}
        print(json.dumps(line), flush=True)
    if comm is not None:
        fgf.fgf_nccl_comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(fgf, torch, dist, world, rank, local, args, c, prm, B, tdt, code, esize):
    """Same metric through fgf_filter_host: each step copies the step's inputs from pinned
    host memory to the device and q back.  The host batch is bounded by host RAM."""
    import synth
    H, W, CI, CP = c["H"], c["W"], c["C_I"], c["C_p"]
    N = H * W
    per_img = esize * N * (CI + (0 if args.config == 0 else CP) + CP)
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except Exception:
        avail = 64 << 30
    # the whole batch when host RAM allows (pinned I, p and q take per_img per image; keep
    # half of the available memory free), else the largest batch that fits
    Be = int(max(1, min(B, (avail // max(1, world)) // 2 // per_img)))
    dev = torch.device("cuda", local)

    def agree(x, op):   # one value for every rank (the host batch must match across ranks)
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=op)
        return int(t.item())

    Be = agree(Be, dist.ReduceOp.MIN if world > 1 else None)

    def pinned(t):   # one pinned host copy (no pageable intermediate)
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h
    while True:   # pinning can fail below the free-memory estimate: halve the batch and retry
        ok = 1
        try:
            Id, pd = synth.make_batch(args.config, dev, batch=Be, first=rank * B)
            if args.dtype == "u8":     # 8-bit codes k / 255 (R19)
                Id = torch.round(Id.clamp(0, 1) * 255.0).to(torch.uint8)
                pd = torch.round(pd.clamp(0, 1) * 255.0).to(torch.uint8)
            elif args.dtype != "f32":
                Id, pd = Id.to(tdt), pd.to(tdt)
            Ih = pinned(Id)
            ph = Ih if args.config == 0 else pinned(pd)
            del Id, pd
            qh = torch.empty((Be, CP, H, W), dtype=tdt, pin_memory=True)
        except (RuntimeError, MemoryError):
            ok = 0
            Ih = ph = qh = Id = pd = None
            torch.cuda.empty_cache()
        if agree(ok, dist.ReduceOp.MIN if world > 1 else None) == 1:
            break
        if Be == 1:
            raise RuntimeError("e2e: no pinned host batch could be allocated")
        Be = max(1, Be // 2)

    def step():
        fgf.fgf_filter_host_ex(Ih, ph, qh, Be, H, W, CI, CP, prm["r"], prm["eps"], prm["s"],
                               prm["sub_mode"], code, local)

    step()
    steps = args.e2e_steps or max(2, min(args.steps, 5))
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64,
                      device=torch.device("cuda", local))
    if world > 1:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    dt = float(dt.item())
    # bytes the call copies (the library's own rule: with nearest samples only the sample rows
    # of p are read from the host buffer, include/fgf.h)
    h2d = fgf.fgf_filter_host_input_bytes(Be, H, W, CI, CP, prm["r"], prm["s"], prm["sub_mode"],
                                          code, args.config == 0)
    h2d_dense = Be * esize * N * (CI + (0 if args.config == 0 else CP))
    d2h = Be * esize * N * CP
    return {"value": world * Be * N * steps / dt / 1e6, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "h2d_bytes_dense_inputs": h2d_dense,
            "batch_per_gpu": Be, "steps": steps,
            "api": "fgf_filter_host_ex (C ABI; fgf_filter_host is its fp32 form; pinned host buffers, H2D/compute/D2H overlapped; "
                   "nearest samples: I whole + the sample rows of p cross the link, the rows "
                   "Alg. 2 reads)"}


if __name__ == "__main__":
    main()
