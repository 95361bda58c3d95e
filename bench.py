#!/usr/bin/env python
"""Benchmark of the forward splatting rasterizer (BASELINE.json metric: rendered
FPS & Mpixel/s at 300k primitives 1245x825; % of binding roofline).

One step = the whole hot path for one view per GPU: snp_project (K1) ->
snp_bin_sort (K2 count/scan/duplicate, K3 onesweep sort, K4 ranges) ->
snp_render (K5 + K6), replayed as one captured CUDA graph, with the scene
resident in HBM.  Workload at N=1: config C3 (300k neural primitives, one
1245x825 view).  For N>1 every rank renders its own C4 orbit view each step
(weak scaling, one view per GPU per step, no data-path collective; the scene
is broadcast once from rank 0 with NCCL).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl snp|reference]

--impl reference times the CPU oracle (the only reference this paper-only task
has) on a bounded pixel sample of the same workload on the host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rendered FPS & Mpixel/s at 300k primitives 1245×825; % of binding roofline"
# SURVEY.md 8(d) algorithmic work of K5: 15 FP32 per tested (pixel, listed primitive)
# pair; 102 FP32 + 28 XU (MUFU) per exact hit.  An XU op occupies 8 FP32 issue
# slots (16 vs 128 lanes/SM/clk), so work is counted in FP32-lane equivalents.
FP32_PER_PAIR = 15
FP32_PER_HIT = 102
XU_PER_HIT = 28
XU_WEIGHT = 8
SMS, FP32_LANES = 148, 128


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p.get("sm_max_mhz", 1965.0)), float(p.get("hbm_gbs", 6536.0)), "measured"
    except Exception:
        return 1965.0, 6650.0, "fallback"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: an NVML thread
    every 5 ms (nvidia-smi -lms 100 as the fallback when NVML is unavailable)."""

    REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.thread = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_gpu{index}.csv")

    def start(self):
        try:
            import threading
            import pynvml as nv
            nv.nvmlInit()
            h = None
            try:   # the CUDA ordinal's NVML handle through its PCI address (CUDA_VISIBLE_DEVICES)
                import torch
                pr = torch.cuda.get_device_properties(self.index)
                h = nv.nvmlDeviceGetHandleByPciBusId(
                    f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0")
            except Exception:
                h = None
            if h is None:
                h = nv.nvmlDeviceGetHandleByIndex(self.index)
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            self.samples, self.reasons = [], set()
            self.smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.stop_flag = threading.Event()

            def run():
                while not self.stop_flag.is_set():
                    try:
                        self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.reasons.update(k for k, v in bits.items() if r & v)
                    except Exception:
                        pass
                    self.stop_flag.wait(0.005)

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self.stop_flag.set()
            self.thread.join()
            sm = self.samples
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax,
                    "samples": len(sm), "source": "nvml, 5 ms", "reasons": sorted(self.reasons)}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, smax, reasons = [], [], set()
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(self.REASONS, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "source": "nvidia-smi, 100 ms", "reasons": sorted(reasons)}


def run_snp(args):
    import torch
    import torch.distributed as dist

    import synth
    from paper_2510_08491_b200 import multigpu as mg
    from paper_2510_08491_b200 import snp

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)

    # ---- workload: C3 scene; rank 0's view is the C3 camera, others take C4 orbit views
    scene, cams3, bg = synth.make_config("C3")
    cam = cams3[0]
    if ws > 1 and rank > 0:
        c4 = synth.orbit_cameras(64, 4.0, cam.width, cam.height, cam.fx, elev_deg=(15.0, 30.0), az0_deg=30.0)
        cam = c4[(rank * 64 // ws) % 64]
    W, H = cam.width, cam.height
    st = torch.cuda.Stream(device=dev)

    # X1: parameters broadcast once from rank 0 (flat [n, 99] fp32); every rank builds its
    # scene from the broadcast copy
    flat = mg.pack_params(scene, dev) if rank == 0 else torch.empty(0, device=dev)
    flat = mg.broadcast_params(flat, scene.n, src=0)
    dscene = mg.unpack_params(flat)
    dscene.omega, dscene.sh_degree = scene.omega, scene.sh_degree

    h = snp.create_scene(dscene, local, st)
    out = torch.empty((1, H, W, 4), device=dev)
    cams_c = snp.make_cameras([cam])
    opts_sync = snp.make_opts(bg, 1e-4, sync_check=1)
    opts = snp.make_opts(bg, 1e-4, sync_check=0)
    with torch.cuda.stream(st):
        snp.render_views(h, cams_c, opts_sync, out, st)      # sizes every buffer
        st.synchronize()
        # capture the whole step (K1..K6) as one CUDA graph
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            snp.render_views(h, cams_c, opts, out, st)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2

    def step():
        g.replay()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stats = snp.get_stats(h, st)
    passes = (19 + int(np.ceil(np.log2(((W + 15) // 16) * ((H + 15) // 16)))) + 7) // 8
    # K1a, K1b, K2 (single-pass dup), K3 x passes, K4, tile order, K5, K6
    launches_per_step = 7 + passes

    clk = ClockSampler(local)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.start()
    times = []
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with torch.cuda.stream(st):
        for i in range(args.steps):
            flush.zero_()                      # evict L2 between timed steps (untimed)
            ev[i][0].record(st)
            step()
            ev[i][1].record(st)
    st.synchronize()
    torch.cuda.synchronize()
    clocks = clk.stop()
    if ws > 1:
        dist.barrier()
    times = [a.elapsed_time(b) for a, b in ev]
    total_ms = mg.max_over_ranks(float(sum(times)), dev)
    ms_per_step = total_ms / args.steps
    fps = ws * args.steps / (total_ms / 1e3)     # views (frames) per second, all GPUs

    # ---- per-stage timing (same stream, CUDA events, non-graph) for the roofline
    stage = {"project": [], "bin_sort": [], "render": []}
    with torch.cuda.stream(st):
        for _ in range(max(3, min(args.steps, 20))):
            flush.zero_()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record(st)
            snp.project(h, cams_c, st)
            e[1].record(st)
            snp.bin_sort(h, opts, st)
            e[2].record(st)
            snp.render(h, opts, out, st)
            e[3].record(st)
            st.synchronize()
            stage["project"].append(e[0].elapsed_time(e[1]))
            stage["bin_sort"].append(e[1].elapsed_time(e[2]))
            stage["render"].append(e[2].elapsed_time(e[3]))
    stats = snp.get_stats(h, st)
    stage_ms = {k: statistics.median(v) for k, v in stage.items()}
    sm_mhz_max, _, peak_kind = _peaks()
    peak = SMS * FP32_LANES * sm_mhz_max * 1e6 / 1e12          # T FP32-lane-op/s
    work = (FP32_PER_PAIR * stats["tested_pairs"] + (FP32_PER_HIT + XU_WEIGHT * XU_PER_HIT) * stats["hit_pairs"])
    achieved = work / (stage_ms["render"] / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "render_traffic_bytes.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("bytes_per_launch")
        except Exception:
            traffic = None

    # ---- e2e through the C ABI with HOST buffers: every step uploads the scene from pinned
    # host memory (snp_update_scene: H2D + device validation) and reads its frame back into
    # pinned host memory (SNP_MEM_HOST_ASYNC); copies inside the timed region.  Two scene
    # handles alternate so that step i+1's upload overlaps step i's render and read-back
    # (PCIe is full duplex), as a serving loop would run it.
    host = {}
    for f in ("centers", "rotations", "scales", "w1", "b1", "w2", "b2", "sh"):
        host[f] = torch.from_numpy(np.ascontiguousarray(getattr(scene, f))).pin_memory()
    import types
    hscene = types.SimpleNamespace(omega=scene.omega, sh_degree=scene.sh_degree, **host)
    hout = [torch.empty((1, H, W, 4)).pin_memory() for _ in range(2)]
    opts_first = snp.make_opts(bg, 1e-4, out_memory=snp.SNP_MEM_HOST, sync_check=1)
    opts_async = snp.make_opts(bg, 1e-4, out_memory=snp.SNP_MEM_HOST_ASYNC, sync_check=0)
    h2d = sum(int(v.numel()) * 4 for v in host.values()) + 88
    d2h = int(hout[0].numel()) * 4
    e2e_steps = max(6, min(args.steps, 50))
    s_up, s_rn = torch.cuda.Stream(), torch.cuda.Stream()
    he = [snp.create_scene(hscene, local, s_up) for _ in range(2)]
    for k in range(2):
        snp.render_views(he[k], cams_c, opts_first, hout[k], s_rn)   # sizing call (outside timing)
    ev_up = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    for k in range(2):
        ev_done[k].record(s_rn)

    def e2e_step(i):
        k = i & 1
        s_up.wait_event(ev_done[k])            # handle k's previous render and read-back are done
        snp.update_scene(he[k], hscene, s_up)  # H2D + validation (returns once validated)
        ev_up[k].record(s_up)
        s_rn.wait_event(ev_up[k])
        snp.render_views(he[k], cams_c, opts_async, hout[k], s_rn)
        ev_done[k].record(s_rn)

    e2e_step(0)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        e2e_step(i)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    for k in range(2):
        snp.destroy(he[k])
    e2e_fps = ws * e2e_steps / mg.max_over_ranks(e2e_s, dev)

    # X2: gather the last frames to rank 0 once (outside the timed region)
    mg.gather_frames(out, dst=0)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(scene, cam, bg, budget_s=args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(fps, 3), "unit": "frames/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "C3: 300k neural primitives (N=8, omega=30, SH deg 3), 1245x825, "
                                   "1 view per GPU per step (C4 orbit views on ranks > 0)",
                       "primitives": scene.n, "width": W, "height": H, "views_per_gpu_per_step": 1,
                       "parallelism": f"views x{ws}" if ws > 1 else "single GPU",
                       "l2": "flushed between timed steps (256 MiB write, untimed)",
                       "graph": "project+bin_sort+render captured as one CUDA graph"},
            "mpix_per_s": round(fps * W * H / 1e6, 2),
            "stages_ms": {k: round(v, 5) for k, v in stage_ms.items()},
            "workload_stats": stats,
            "roofline": {"bound": "alu", "kernel": "k_render (K5)", "achieved": round(achieved, 4),
                         "peak": round(peak, 3), "unit": "T FP32-lane-op/s (XU op = 8 lanes)",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "peak_source": f"148 SMs x 128 FP32 lanes x {sm_mhz_max:.0f} MHz ({peak_kind} sm_max_mhz)",
                         "work": f"{FP32_PER_PAIR}*tested_pairs + ({FP32_PER_HIT}+{XU_WEIGHT}*{XU_PER_HIT})*hit_pairs"},
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_fps, 3), "unit": "frames/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "what": "per step: snp_update_scene from pinned host arrays (H2D + device validation) + "
                            "snp_render_views into a pinned host frame (SNP_MEM_HOST_ASYNC D2H); two scene "
                            "handles alternate so that one step's upload overlaps the previous step's render "
                            "and read-back; wall clock"},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line))
    snp.destroy(h)
    if ws > 1:
        dist.destroy_process_group()


def cpu_baseline(scene, cam, bg, budget_s=15.0):
    """The oracle as it stands on the host cores, on seeded pixel samples of the
    same view until ~budget_s of CPU time; frames/s = sampled pixels/s / (W*H)."""
    import oracle
    oracle.build()
    rng = np.random.default_rng(123)
    W, H = cam.width, cam.height
    cores = os.cpu_count() or 1
    chunk = max(64, 16 * cores)
    n, dt = 0, 0.0
    while dt < budget_s:
        px, py = rng.integers(0, W, chunk), rng.integers(0, H, chunk)
        t0 = time.perf_counter()
        oracle.render_pixels(scene, cam, px, py, bg, nthreads=0)
        dt += time.perf_counter() - t0
        n += chunk
        chunk = min(chunk * 2, 1 << 16)
    pps = n / dt
    return {"value": pps / (W * H), "unit": "frames/s", "cores": cores, "kind": "oracle",
            "sample": f"{n} seeded random pixels of the C3 view ({dt:.1f} s, OpenMP over pixels)",
            "pixels_per_s": round(pps, 1)}


def run_reference(args):
    """--impl reference: the CPU oracle, as it stands, on the host cores."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    import synth
    scene, cams3, bg = synth.make_config("C3")
    cam = cams3[0]
    budget = max(1.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    import oracle
    oracle.build()
    rng = np.random.default_rng(321)
    W, H = cam.width, cam.height
    cores = os.cpu_count() or 1
    n0 = max(64, 16 * cores)
    t0 = time.perf_counter()
    oracle.render_pixels(scene, cam, rng.integers(0, W, n0), rng.integers(0, H, n0), bg, nthreads=0)
    per_px = (time.perf_counter() - t0) / n0
    n = int(max(n0, budget / max(per_px, 1e-9)))
    for _ in range(args.warmup):
        oracle.render_pixels(scene, cam, rng.integers(0, W, 64), rng.integers(0, H, 64), bg, nthreads=0)
    tot_px, tot_s = 0, 0.0
    for _ in range(args.steps):
        px, py = rng.integers(0, W, n), rng.integers(0, H, n)
        t0 = time.perf_counter()
        oracle.render_pixels(scene, cam, px, py, bg, nthreads=0)
        tot_s += time.perf_counter() - t0
        tot_px += n
    fps = tot_px / tot_s / (W * H)
    line = {"impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_s / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "C3: 300k neural primitives, 1245x825, 1 view; each step = a seeded "
                                   f"sample of {n} pixels of that view (CPU oracle)"},
            "cpu_baseline": {"kind": "oracle", "cores": cores, "value": fps, "unit": "frames/s",
                             "sample": f"{n} random pixels per step x {args.steps} steps"},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="snp", choices=["snp", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_snp(args)


if __name__ == "__main__":
    main()
