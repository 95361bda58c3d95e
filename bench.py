#!/usr/bin/env python
"""Benchmark of the forward splatting rasterizer (BASELINE.json metric: rendered
FPS & Mpixel/s at 300k primitives 1245x825; % of binding roofline).

One step = the whole hot path for one view per GPU: snp_project (K1) ->
snp_bin_sort (K2 count/scan/duplicate, K3 onesweep sort, K4 ranges) ->
snp_render (K5 + K6), replayed as one captured CUDA graph, with the scene
resident in HBM.  Workload at N=1: config C3 (300k neural primitives, one
1245x825 view).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl snp|reference]
                  [--workload c3|c4]

N > 1 (or --workload c4): config C4 -- the 64-view orbit batch of the C3 scene,
sharded in contiguous blocks of 64/N views per GPU, one snp_render_views per rank
per step (strong scaling of the fixed batch); X2 gathers every rank's frames to
rank 0 on a second stream, overlapped with the next step's render.  --gpus N
without WORLD_SIZE in the environment re-launches itself under torch.distributed.run
with N ranks (one GPU each, NCCL).

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
# pair; 102 FP32 + 28 XU (MUFU) per exact hit.  The pipes issue concurrently, so the
# model's lower bound of the render time is the largest of (8(d)(ii)):
#   FP32  sum FP32 ops / (SMs x 128 lanes x f)
#   XU    sum XU ops   / (SMs x 16 lanes x f)
#   issue sum ops / 32 (warp instructions) / (SMs x 4 schedulers x f)
# and the roofline fraction is that bound over the measured time (the binding pipe's).
FP32_PER_PAIR = 15
FP32_PER_HIT = 102
XU_PER_HIT = 28
SMS, FP32_LANES, XU_LANES, ISSUE_PER_SM = 148, 128, 16, 4
C4_VIEWS = 64


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



def roofline_k5(stats, render_ms, sm_mhz):
    """the K5 model's per-pipe lower bounds against the measured render."""
    P, Hh = float(stats["tested_pairs"]), float(stats["hit_pairs"])
    f = sm_mhz * 1e6
    fp32 = FP32_PER_PAIR * P + FP32_PER_HIT * Hh
    xu = XU_PER_HIT * Hh
    inst = (fp32 + xu) / 32.0
    t = render_ms / 1e3
    pipes = {
        "fp32": {"work": fp32, "peak_per_s": SMS * FP32_LANES * f, "unit": "FP32 lane-ops"},
        "xu": {"work": xu, "peak_per_s": SMS * XU_LANES * f, "unit": "XU lane-ops"},
        "issue": {"work": inst, "peak_per_s": SMS * ISSUE_PER_SM * f, "unit": "warp-instructions"},
    }
    for v in pipes.values():
        v["model_us"] = v["work"] / v["peak_per_s"] * 1e6
        v["frac"] = v["model_us"] / (render_ms * 1e3)
    bind = max(pipes, key=lambda k: pipes[k]["frac"])
    b = pipes[bind]
    return {"bound": "alu", "kernel": "k_render + k_fallback (K5 + K6: snp_render)", "pipe": bind,
            "achieved": round(b["work"] / t / 1e12, 5), "peak": round(b["peak_per_s"] / 1e12, 5),
            "unit": f"T {b['unit']}/s", "frac": round(b["frac"], 4),
            "pipes": {k: {"frac": round(v["frac"], 4), "model_us": round(v["model_us"], 2)} for k, v in pipes.items()},
            "peak_source": f"{SMS} SMs x (128 FP32 | 16 XU lanes | 4 issue) x {sm_mhz:.0f} MHz (sm_max_mhz)",
            "work": f"FP32 {FP32_PER_PAIR}*tested + {FP32_PER_HIT}*hits; XU {XU_PER_HIT}*hits; "
                    "warp-instr = (FP32 + XU)/32 (SURVEY 8(d))",
            "render_us": round(render_ms * 1e3, 2)}


def _device_scene(scene, dev, rank, ws):
    """X1: the parameters broadcast once from rank 0 (one flat [n, 99] fp32 tensor)."""
    from paper_2510_08491_b200 import multigpu as mg
    flat = mg.pack_params(scene, dev) if rank == 0 else torch_empty(dev)
    flat = mg.broadcast_params(flat, scene.n, src=0, n_hidden=scene.n_hidden)
    dscene = mg.unpack_params(flat)
    dscene.omega, dscene.sh_degree = scene.omega, scene.sh_degree
    return dscene


def torch_empty(dev):
    import torch
    return torch.empty(0, device=dev)


def _timed(args, fn, st, ws, dev, flush=None):
    """K timed steps of fn() bracketed by a barrier + synchronize, CUDA events on st;
    returns (total ms max over ranks, clocks)."""
    import torch
    import torch.distributed as dist
    from paper_2510_08491_b200 import multigpu as mg
    clk = ClockSampler(torch.cuda.current_device())
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with torch.cuda.stream(st):
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()                  # evict L2 between timed steps (untimed)
            ev[i][0].record(st)
            fn(i)
            ev[i][1].record(st)
    st.synchronize()
    torch.cuda.synchronize()
    clocks = clk.stop()
    if ws > 1:
        dist.barrier()
    total = sum(a.elapsed_time(b) for a, b in ev)
    return mg.max_over_ranks(float(total), dev), clocks


def run_c3(args):
    """N = 1 headline: config C3, one view per step (the whole hot path as one graph)."""
    import torch

    import synth
    from paper_2510_08491_b200 import snp

    local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    scene, cams3, bg = synth.make_config("C3")
    cam = cams3[0]
    W, H = cam.width, cam.height
    st = torch.cuda.Stream(device=dev)
    dscene = _device_scene(scene, dev, 0, 1)
    h = snp.create_scene(dscene, local, st)
    out = torch.empty((1, H, W, 4), device=dev)
    cams_c = snp.make_cameras([cam])
    opts_sync = snp.make_opts(bg, 1e-4, sync_check=1)
    opts = snp.make_opts(bg, 1e-4, sync_check=0)
    with torch.cuda.stream(st):
        snp.render_views(h, cams_c, opts_sync, out, st)      # sizes every buffer
        st.synchronize()
        g = torch.cuda.CUDAGraph()                          # the whole step (K1..K6) as one graph
        with torch.cuda.graph(g, stream=st):
            snp.render_views(h, cams_c, opts, out, st)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    for _ in range(args.warmup):
        g.replay()
    torch.cuda.synchronize()
    passes = (19 + int(np.ceil(np.log2(((W + 15) // 16) * ((H + 15) // 16)))) + 7) // 8
    launches_per_step = 8 + passes   # K1a, K1b, K2, K3 x passes, K4, tile order, K5, K6w, K6
    total_ms, clocks = _timed(args, lambda i: g.replay(), st, 1, dev, flush)
    ms_per_step = total_ms / args.steps
    fps = args.steps / (total_ms / 1e3)

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
    roof = roofline_k5(stats, stage_ms["render"], sm_mhz_max)
    roof["peak_kind"] = peak_kind
    tpath = os.path.join(ROOT, "profiles", "render_traffic_bytes.json")
    roof["traffic"] = None
    if os.path.exists(tpath):
        try:
            roof["traffic"] = json.load(open(tpath)).get("bytes_per_launch")
        except Exception:
            pass
    frame = out[0].cpu().numpy()

    e2e = e2e_c3(args, scene, cams_c, bg, W, H, local)
    e2e_resident = e2e_resident_c3(args, scene, cams_c, bg, W, H, local)

    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(scene, cam, bg, budget_s=args.cpu_seconds, gpu_frame=frame)

    line = {
        "metric": METRIC, "value": round(fps, 3), "unit": "frames/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "C3: 300k neural primitives (N=8, omega=30, SH deg 3), one 1245x825 view per step",
                   "primitives": scene.n, "width": W, "height": H, "views_per_step": 1,
                   "parallelism": "single GPU",
                   "l2": "flushed between timed steps (256 MiB write, untimed)",
                   "graph": "project+bin_sort+render captured as one CUDA graph"},
        "mpix_per_s": round(fps * W * H / 1e6, 2),
        "stages_ms": {k: round(v, 5) for k, v in stage_ms.items()},
        "workload_stats": stats,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_scene_resident": e2e_resident,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
        "paper_context": "115 FPS, Mip-NeRF360 9-scene average (~2.4e5 trained primitives), RTX 4090 "
                         "(PAPER.md:607 Table 2; resolution not stated): another GPU and workload",
    }
    print(json.dumps(line))
    snp.destroy(h)


def e2e_c3(args, scene, cams_c, bg, W, H, local):
    """The same metric through the C ABI with HOST buffers: every step uploads the scene from
    pinned host memory (snp_update_scene: H2D + device validation) and reads its frame back
    into pinned host memory (SNP_MEM_HOST_ASYNC); copies inside the timed region.  Two scene
    handles alternate so that step i+1's upload overlaps step i's render and read-back (PCIe
    is full duplex), as a serving loop would run it."""
    import types

    import torch

    from paper_2510_08491_b200 import snp
    host = {}
    for f in ("centers", "rotations", "scales", "w1", "b1", "w2", "b2", "sh"):
        host[f] = torch.from_numpy(np.ascontiguousarray(getattr(scene, f))).pin_memory()
    hscene = types.SimpleNamespace(omega=scene.omega, sh_degree=scene.sh_degree, **host)
    nv = len(cams_c)
    hout = [torch.empty((nv, H, W, 4)).pin_memory() for _ in range(2)]
    opts_first = snp.make_opts(bg, 1e-4, out_memory=snp.SNP_MEM_HOST, sync_check=1)
    opts_async = snp.make_opts(bg, 1e-4, out_memory=snp.SNP_MEM_HOST_ASYNC, sync_check=0)
    h2d = sum(int(v.numel()) * 4 for v in host.values()) + 88
    d2h = int(hout[0].numel()) * 4
    steps = max(6, min(args.steps, 50))
    s_up, s_rn = torch.cuda.Stream(), torch.cuda.Stream()
    he = [snp.create_scene(hscene, local, s_up) for _ in range(2)]
    for k in range(2):
        snp.render_views(he[k], cams_c, opts_first, hout[k], s_rn)   # sizing call (outside timing)
    ev_up = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    for k in range(2):
        ev_done[k].record(s_rn)

    def step(i):
        k = i & 1
        s_up.wait_event(ev_done[k])            # handle k's previous render and read-back are done
        snp.update_scene(he[k], hscene, s_up)  # H2D + validation (returns once validated)
        ev_up[k].record(s_up)
        s_rn.wait_event(ev_up[k])
        snp.render_views(he[k], cams_c, opts_async, hout[k], s_rn)
        ev_done[k].record(s_rn)

    step(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(steps):
        step(i)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    for k in range(2):
        snp.destroy(he[k])
    return {"value": round(nv * steps / dt, 3), "unit": "frames/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps,
            "what": "per step: snp_update_scene from pinned host arrays (H2D + device validation) + "
                    "snp_render_views into a pinned host frame (SNP_MEM_HOST_ASYNC D2H); two scene handles "
                    "alternate so that one step's upload overlaps the previous step's render and read-back; "
                    "wall clock"}


def e2e_resident_c3(args, scene, cams_c, bg, W, H, local):
    """A second end-to-end figure for the serving case: the scene is uploaded once
    (outside the timed region) and every step renders the view from a host camera into a
    pinned host frame (SNP_MEM_HOST_ASYNC D2H inside the timed region).  Two handles on
    two streams alternate so that one frame's read-back overlaps the next render."""
    import types

    import torch

    from paper_2510_08491_b200 import snp
    host = {f: torch.from_numpy(np.ascontiguousarray(getattr(scene, f))).pin_memory()
            for f in ("centers", "rotations", "scales", "w1", "b1", "w2", "b2", "sh")}
    hscene = types.SimpleNamespace(omega=scene.omega, sh_degree=scene.sh_degree, **host)
    nv = len(cams_c)
    hout = [torch.empty((nv, H, W, 4)).pin_memory() for _ in range(2)]
    opts_first = snp.make_opts(bg, 1e-4, out_memory=snp.SNP_MEM_HOST, sync_check=1)
    opts_async = snp.make_opts(bg, 1e-4, out_memory=snp.SNP_MEM_HOST_ASYNC, sync_check=0)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    he = [snp.create_scene(hscene, local, streams[k]) for k in range(2)]
    for k in range(2):
        snp.render_views(he[k], cams_c, opts_first, hout[k], streams[k])   # sizing call (outside timing)
    torch.cuda.synchronize()
    steps = max(6, min(args.steps, 100))
    t0 = time.perf_counter()
    for i in range(steps):
        k = i & 1
        snp.render_views(he[k], cams_c, opts_async, hout[k], streams[k])
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    for k in range(2):
        snp.destroy(he[k])
    return {"value": round(nv * steps / dt, 3), "unit": "frames/s", "h2d_bytes_per_step": 88 * nv,
            "d2h_bytes_per_step": int(hout[0].numel()) * 4, "steps": steps,
            "what": "scene resident (uploaded once, untimed); per step a host camera in, the frame into "
                    "pinned host memory out (SNP_MEM_HOST_ASYNC); two handles on two streams, so two frames "
                    "are in flight and no L2 flush separates them (unlike `value`'s serialised steps); "
                    "wall clock"}


def c4_launches_per_step(nv, W, H):
    """Kernels one snp_render_views of nv views launches: per camera batch (<= 32 views)
    K1a, K1b, the tile order, K5, K6w, K6; once K2 and K4; K3 once per 8-bit digit of
    the (view | tile | depth) key."""
    batches = (nv + 31) // 32
    bits = lambda v: int(np.ceil(np.log2(v))) if v > 1 else 0   # (bits_for in api.cu)
    passes = (19 + bits(((W + 15) // 16) * ((H + 15) // 16)) + bits(nv) + 7) // 8
    return 6 * batches + 2 + passes


def run_c4(args):
    """Config C4 on N ranks: 64 orbit views of the C3 scene, contiguous blocks of 64/N views
    per GPU, one snp_render_views per rank per step; X2 gathers the frames to rank 0 on a
    second stream, overlapped with the next step's render (multigpu.ShardedFrames)."""
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
    scene, cams64, bg = synth.make_config("C4")
    W, H = cams64[0].width, cams64[0].height
    st = torch.cuda.Stream(device=dev)
    comm = torch.cuda.Stream(device=dev)
    dscene = _device_scene(scene, dev, rank, ws)
    h = snp.create_scene(dscene, local, st)
    views = mg.views_for_rank(rank, ws, C4_VIEWS)
    cams_c = snp.make_cameras([cams64[v] for v in views])
    opts_sync = snp.make_opts(bg, 1e-4, sync_check=1)
    opts = snp.make_opts(bg, 1e-4, sync_check=0)
    graphs = {}

    def render_fn(buf):
        graphs[buf.data_ptr()].replay()

    with torch.cuda.stream(st):
        sf = mg.ShardedFrames(render_fn, C4_VIEWS, (H, W), dev, comm)
        for k in range(2):
            b = sf.bufs[k][:len(views)]
            snp.render_views(h, cams_c, opts_sync, b, st)     # sizes every buffer
            st.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                snp.render_views(h, cams_c, opts, b, st)
            graphs[b.data_ptr()] = g
        for i in range(args.warmup):
            sf.step(i)
    torch.cuda.synchronize()
    # K5 roofline of this rank's shard: the snp_render stage (K5 + fallbacks) timed alone
    # (CUDA events on the render stream, after a project + bin_sort of the same views)
    rt = []
    with torch.cuda.stream(st):
        for _ in range(5):
            snp.project(h, cams_c, st)
            snp.bin_sort(h, opts, st)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            snp.render(h, opts, sf.bufs[0][:len(views)], st)
            e1.record(st)
            st.synchronize()
            rt.append(e0.elapsed_time(e1))
    stats = snp.get_stats(h, st)
    sm_mhz_max, _, peak_kind = _peaks()
    roof = roofline_k5(stats, statistics.median(rt), sm_mhz_max)
    roof["peak_kind"] = peak_kind
    roof["scope"] = f"rank 0's {len(views)} views in one snp_render"
    # render only
    render_ms, clocks = _timed(args, lambda i: sf.render(i), st, ws, dev)
    # render + gather (the gather of step i overlaps the render of step i + 1); the timed
    # region ends when the last gather has completed on the communication stream
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for i in range(args.steps):
            sf.step(i)
        st.wait_stream(comm)
        e1.record(st)
    torch.cuda.synchronize()
    rg_ms = mg.max_over_ranks(e0.elapsed_time(e1), dev)
    # correctness: the gathered frames are bit-identical to one GPU's render
    last = (args.steps - 1)
    bit_identical = None
    if rank == 0:
        ref_h = snp.create_scene(dscene, local, st)
        ref = torch.empty((C4_VIEWS, H, W, 4), device=dev)
        with torch.cuda.stream(st):
            snp.render_views(ref_h, snp.make_cameras(cams64), opts_sync, ref, st)
        torch.cuda.synchronize()
        bit_identical = bool(torch.equal(sf.frames(last), ref))
        snp.destroy(ref_h)
    e2e = None
    if rank == 0 or ws > 1:
        e2e_local = e2e_c3(args, scene, cams_c, bg, W, H, local)
        e2e_val = mg.max_over_ranks(len(views) / e2e_local["value"], dev)   # s per step, slowest rank
        e2e = dict(e2e_local, value=round(C4_VIEWS / e2e_val, 3), unit="views/s",
                   what="per rank and step: snp_update_scene from pinned host arrays + snp_render_views of the "
                        "rank's 64/N views into pinned host frames; value = 64 views / slowest rank's time")
    views_s = C4_VIEWS * args.steps / (render_ms / 1e3)
    rg_views_s = C4_VIEWS * args.steps / (rg_ms / 1e3)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(views_s, 3), "unit": "views/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(render_ms / args.steps, 5),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"C4: 300k neural primitives, 64 orbit views of 1245x825 per step, "
                                   f"{len(views)} views per GPU (contiguous blocks)", "views_per_step": C4_VIEWS,
                       "primitives": scene.n, "width": W, "height": H,
                       "parallelism": f"views x{ws}" if ws > 1 else "single GPU",
                       "l2": "inputs larger than L2 (64 views of records: 64 x 48.8 MB)",
                       "graph": "each rank's snp_render_views (K1..K6 over its views) as one CUDA graph"},
            "mpix_per_s": round(views_s * W * H / 1e6, 2),
            "render_gather": {"value": round(rg_views_s, 3), "unit": "views/s",
                              "ms_per_step": round(rg_ms / args.steps, 5),
                              "what": "render + X2 gather of every rank's frames to rank 0 (NCCL, second "
                                      "stream, overlapped with the next step's render); max over ranks"},
            "bit_identical_to_single_gpu": bit_identical,
            "workload_stats_rank0": stats,
            "roofline": roof,
            "e2e": e2e,
            "gpu_launches": c4_launches_per_step(len(views), W, H) * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line))
    snp.destroy(h)
    if ws > 1:
        dist.destroy_process_group()


def run_selftest_cpu(args):
    """--selftest-cpu: the N-rank launcher and the X2 protocol of run_c4 on CPU (gloo), with
    a deterministic stand-in for the GPU render (no CUDA); used by the tests."""
    import torch
    import torch.distributed as dist

    from paper_2510_08491_b200 import multigpu as mg
    ws, rank, _ = _dist()
    if ws > 1:
        dist.init_process_group("gloo")
    H, W = 6, 5

    def fake_render(views, step):
        v = torch.tensor(views, dtype=torch.float32).view(-1, 1, 1, 1)
        return v * 1000.0 + step + torch.arange(H * W * 4, dtype=torch.float32).view(1, H, W, 4) * 1e-3

    state = {"i": 0}

    def render_fn(buf):
        buf.copy_(fake_render(mg.views_for_rank(rank, ws, C4_VIEWS), state["i"]))

    sf = mg.ShardedFrames(render_fn, C4_VIEWS, (H, W), "cpu")
    for i in range(args.steps):
        state["i"] = i
        sf.step(i)
    if rank == 0:
        got = sf.frames(args.steps - 1)
        ok = bool(torch.equal(got, fake_render(list(range(C4_VIEWS)), args.steps - 1)))
        print(json.dumps({"metric": METRIC, "n_gpus": ws, "selftest": "cpu", "views": C4_VIEWS,
                          "bit_identical_to_single_gpu": ok}))
    if ws > 1:
        dist.destroy_process_group()


def relaunch(args):
    """--gpus N without a torch.distributed environment: N ranks under torch.distributed.run."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def cpu_baseline(scene, cam, bg, budget_s=15.0, gpu_frame=None):
    """The oracle as it stands on the host cores, on seeded pixel samples of the
    same view until ~budget_s of CPU time; frames/s = sampled pixels/s / (W*H).
    Every sampled pixel is also compared with the GPU frame of the timed region
    (gpu_frame [H, W, 4]): parity = max |gpu - oracle| over unflagged pixels (R23)."""
    import oracle
    oracle.build()
    rng = np.random.default_rng(123)
    W, H = cam.width, cam.height
    cores = os.cpu_count() or 1
    chunk = max(64, 16 * cores)
    n, dt = 0, 0.0
    worst, n_flag, n_bad, worst_all = 0.0, 0, 0, 0.0
    while dt < budget_s:
        px, py = rng.integers(0, W, chunk), rng.integers(0, H, chunk)
        t0 = time.perf_counter()
        ref, flags, _ = oracle.render_pixels(scene, cam, px, py, bg, nthreads=0)
        dt += time.perf_counter() - t0
        n += chunk
        if gpu_frame is not None:
            err = np.abs(gpu_frame[py, px].astype(np.float64) - ref).max(axis=1)
            ok = flags == 0
            worst = max(worst, float(err[ok].max()) if ok.any() else 0.0)
            worst_all = max(worst_all, float(err.max()))
            n_flag += int((~ok).sum())
            n_bad += int((err[ok] > 1e-4).sum())
        chunk = min(chunk * 2, 1 << 16)
    pps = n / dt
    # the same oracle on one core (both timings), a smaller seeded sample
    m1, t1 = max(256, int(pps * 3.0 / max(cores, 1))), 0.0
    px1, py1 = rng.integers(0, W, m1), rng.integers(0, H, m1)
    t0 = time.perf_counter()
    oracle.render_pixels(scene, cam, px1, py1, bg, nthreads=1)
    t1 = time.perf_counter() - t0
    res = {"value": pps / (W * H), "unit": "frames/s", "cores": cores, "kind": "oracle",
           "sample": f"{n} seeded random pixels of the C3 view ({dt:.1f} s, OpenMP over pixels)",
           "pixels_per_s": round(pps, 1),
           "single_thread": {"pixels_per_s": round(m1 / t1, 1), "frames_per_s": m1 / t1 / (W * H),
                             "sample": f"{m1} seeded random pixels ({t1:.1f} s, 1 thread; includes the "
                                       "oracle's per-call scene setup)"}}
    if gpu_frame is not None:
        res["parity"] = {"max_unflagged": worst, "max_all": worst_all, "n_flagged": n_flag, "n": n,
                         "n_over_tol": n_bad, "tol": 1e-4,
                         "what": "the sampled pixels of the last timed GPU frame against the oracle"}
    return res


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
    # size the per-step sample from two calls, so that the oracle's per-call scene setup
    # (a fixed cost) is separated from its per-pixel cost and amortised over the sample
    n0, n1 = max(64, 16 * cores), max(1024, 256 * cores)
    t0 = time.perf_counter()
    oracle.render_pixels(scene, cam, rng.integers(0, W, n0), rng.integers(0, H, n0), bg, nthreads=0)
    ta = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.render_pixels(scene, cam, rng.integers(0, W, n1), rng.integers(0, H, n1), bg, nthreads=0)
    tb = time.perf_counter() - t0
    per_px = max((tb - ta) / (n1 - n0), tb / n1 * 0.05, 1e-9)
    n = int(max(n1, budget / per_px))
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
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
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
    ap.add_argument("--workload", default=None, choices=["c3", "c4"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--selftest-cpu", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    ws = _dist()[0]
    if args.selftest_cpu:
        run_selftest_cpu(args)
    elif args.impl == "reference":
        run_reference(args)
    elif (args.workload or ("c4" if ws > 1 else "c3")) == "c4":
        run_c4(args)
    else:
        run_c3(args)


if __name__ == "__main__":
    main()
