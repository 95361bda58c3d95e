"""Multi-GPU plumbing for the forward rasterizer.

The forward path has no cross-GPU reduction: views (and tile stripes) are
independent work units.  One process per GPU (torchrun), torch.distributed over
NCCL for exactly two collectives:

  X1  broadcast of the primitive parameters from rank 0, once per scene;
  X2  gather of rendered frames to rank 0.

Everything here is host-side plumbing over torch.distributed; rendering itself
always runs in libsnp.so on the rank's own GPU.  The functions are backend
agnostic so the same code is exercised with gloo on CPU by the tests.
"""
from __future__ import annotations

from typing import List, Sequence

import torch
import torch.distributed as dist

PARAM_FIELDS = ("centers", "rotations", "scales", "w1", "b1", "w2", "b2", "sh")
PARAM_WIDTHS = (3, 4, 3, 24, 8, 8, 1, 48)          # 99 fp32 per primitive


def views_for_rank(rank: int, world: int, n_views: int) -> List[int]:
    """Contiguous block partition of n_views over world ranks (blocks differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_views, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


def stripe_for_rank(rank: int, world: int):
    """Interleaved tile-row stripe (tile_row_begin, tile_row_stride) for single-view sharding."""
    return rank, world


def pack_params(scene, device) -> torch.Tensor:
    """[n, 99] fp32 tensor of the scene's parameters (field order of PARAM_FIELDS)."""
    n = int(getattr(scene, "centers").shape[0])
    cols = []
    for f, w in zip(PARAM_FIELDS, PARAM_WIDTHS):
        a = getattr(scene, f)
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(a)
        cols.append(t.reshape(n, w).to(device=device, dtype=torch.float32))
    return torch.cat(cols, dim=1).contiguous()


def unpack_params(flat: torch.Tensor):
    """Inverse of pack_params: a namespace of contiguous per-field tensors (views of one copy)."""
    import types
    n = flat.shape[0]
    out = types.SimpleNamespace()
    o = 0
    shapes = {"centers": (n, 3), "rotations": (n, 4), "scales": (n, 3), "w1": (n, 8, 3), "b1": (n, 8),
              "w2": (n, 8), "b2": (n,), "sh": (n, 16, 3)}
    for f, w in zip(PARAM_FIELDS, PARAM_WIDTHS):
        setattr(out, f, flat[:, o:o + w].contiguous().reshape(shapes[f]))
        o += w
    return out


def broadcast_params(flat: torch.Tensor, n: int, src: int = 0) -> torch.Tensor:
    """X1: every rank ends with rank src's [n, 99] parameters (allocated here on non-src ranks)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return flat
    if dist.get_rank() != src:
        flat = torch.empty((n, sum(PARAM_WIDTHS)), dtype=torch.float32, device=flat.device)
    dist.broadcast(flat, src=src)
    return flat


def gather_frames(frames: torch.Tensor, dst: int = 0):
    """X2: rank dst receives every rank's frame tensor (same shape on every rank)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [frames]
    ws = dist.get_world_size()
    out = [torch.empty_like(frames) for _ in range(ws)] if dist.get_rank() == dst else None
    dist.gather(frames, out, dst=dst)
    return out


def max_over_ranks(value: float, device) -> float:
    """Max of a per-rank scalar (multi-GPU timings are the slowest rank's)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def merge_stripes(frames: Sequence[torch.Tensor], height: int, tile: int = 16) -> torch.Tensor:
    """Rebuild one frame from per-rank stripe renders (rank r owns tile rows r, r+W, ...)."""
    world = len(frames)
    out = frames[0].clone()
    for y in range(height):
        r = (y // tile) % world
        out[..., y, :, :] = frames[r][..., y, :, :]
    return out
