"""Training-step throughput: forward + L1 + K7 backward + one
gradient all-reduce + Adam over a multi-view batch, views sharded over the ranks
(torchrun for N > 1, NCCL).  Times K steps with CUDA events (max over ranks).

usage: python tools/train_bench.py [--config C4] [--views 64] [--steps 5]
       torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/train_bench.py ...
"""
import argparse, json, os, sys, types
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2510_08491_b200 import snp, train, multigpu as mg

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--views", type=int, default=64)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=2)
args = ap.parse_args()
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
if world > 1:
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("nccl")
scene, cams, bg = synth.make_config(args.config, views=args.views)
mine = [cams[v] for v in mg.views_for_rank(rank, world, len(cams))]
ns = types.SimpleNamespace(omega=scene.omega, sh_degree=scene.sh_degree)
for f in snp.FIELDS:
    setattr(ns, f, torch.from_numpy(np.ascontiguousarray(getattr(scene, f))).cuda())
h = snp.create_scene(ns, torch.cuda.current_device())
H, W = mine[0].height, mine[0].width
g = torch.Generator(device="cuda").manual_seed(rank)
target = torch.rand((len(mine), H, W, 3), device="cuda", generator=g)
tr = train.Trainer(h, scene, len(mine), H, W, "cuda", opts=snp.make_opts(bg))
for _ in range(args.warmup):
    tr.step(mine, target)
torch.cuda.synchronize()
if world > 1:
    dist.barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.steps):
    loss = tr.step(mine, target)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / args.steps
ms = mg.max_over_ranks(ms, "cuda") if world > 1 else ms
if rank == 0:
    print(json.dumps({"metric": "training steps/s (forward + 3DGS loss (L1 + D-SSIM, lambda 0.2) + backward + all-reduce + Adam)",
                      "value": round(1000.0 / ms, 3), "unit": "steps/s", "ms_per_step": round(ms, 2),
                      "views_per_s": round(1000.0 * len(cams) / ms, 1), "n_gpus": world,
                      "config": {"workload": args.config, "views_per_step": len(cams), "primitives": scene.n,
                                 "width": W, "height": H}, "loss": round(loss.item(), 5),
                      "skipped_pixels": int(snp.get_stats(h)["backward_skipped"])}))
snp.destroy(h)
if world > 1:
    dist.destroy_process_group()
