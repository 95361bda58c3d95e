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


def param_widths(n_hidden: int = 8):
    """fp32 per primitive of each field: 99 in all at the paper's N_sigma = 8."""
    return (3, 4, 3, 3 * n_hidden, n_hidden, n_hidden, 1, 48)


PARAM_WIDTHS = param_widths(8)


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


def _n_hidden(scene) -> int:
    return int(getattr(scene, "w1").shape[1])


def pack_params(scene, device) -> torch.Tensor:
    """[n, 5 + 5 N + 54] fp32 tensor of the scene's parameters (field order of
    PARAM_FIELDS; 99 columns at N_sigma = 8)."""
    n = int(getattr(scene, "centers").shape[0])
    cols = []
    for f, w in zip(PARAM_FIELDS, param_widths(_n_hidden(scene))):
        a = getattr(scene, f)
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(a)
        cols.append(t.reshape(n, w).to(device=device, dtype=torch.float32))
    return torch.cat(cols, dim=1).contiguous()


def unpack_params(flat: torch.Tensor):
    """Inverse of pack_params (N_sigma from the column count): a namespace of contiguous
    per-field tensors."""
    import types
    n = flat.shape[0]
    nh = (flat.shape[1] - 59) // 5
    if flat.shape[1] != sum(param_widths(nh)):
        raise ValueError(f"{flat.shape[1]} columns is no parameter layout")
    out = types.SimpleNamespace()
    o = 0
    shapes = {"centers": (n, 3), "rotations": (n, 4), "scales": (n, 3), "w1": (n, nh, 3), "b1": (n, nh),
              "w2": (n, nh), "b2": (n,), "sh": (n, 16, 3)}
    for f, w in zip(PARAM_FIELDS, param_widths(nh)):
        setattr(out, f, flat[:, o:o + w].contiguous().reshape(shapes[f]))
        o += w
    return out


def broadcast_params(flat: torch.Tensor, n: int, src: int = 0, n_hidden: int = 8) -> torch.Tensor:
    """X1: every rank ends with rank src's [n, 5 + 5 N + 54] parameters (allocated here on
    non-src ranks; N = n_hidden must agree on every rank)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return flat
    if dist.get_rank() != src:
        flat = torch.empty((n, sum(param_widths(n_hidden))), dtype=torch.float32, device=flat.device)
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


class ShardedFrames:
    """The N-GPU view batch: rank r renders its contiguous block of the
    batch's views (views_for_rank) each step with one render call, and X2 gathers every
    rank's frames to rank 0.  Frames are double buffered: step i renders into buffer
    i % 2 while the gather of step i - 1 (buffer (i - 1) % 2) runs on a separate stream,
    so collection overlaps rendering; step i + 1 waits only for the gather of step i - 1
    before overwriting that buffer.

    render_fn(buf) enqueues one step's render of this rank's views into buf [k, H, W, 4]
    (on the current stream).  Shards are padded to the largest block so the gather has
    equal sizes.  Backend agnostic (NCCL on GPUs, gloo on CPU in the tests)."""

    def __init__(self, render_fn, n_views: int, frame_hw, device, comm_stream=None):
        self.render_fn = render_fn
        self.n_views = n_views
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.views = views_for_rank(self.rank, self.world, n_views)
        self.shard = max(len(views_for_rank(r, self.world, n_views)) for r in range(self.world))
        H, W = frame_hw
        self.device = torch.device(device)
        self.cuda = self.device.type == "cuda"
        self.bufs = [torch.zeros((self.shard, H, W, 4), dtype=torch.float32, device=self.device) for _ in range(2)]
        self.recv = None
        if self.rank == 0:
            self.recv = [[torch.empty_like(self.bufs[0]) for _ in range(self.world)] for _ in range(2)]
        self.comm = comm_stream
        self.ev_rendered = [torch.cuda.Event() for _ in range(2)] if self.cuda else None
        self.ev_gathered = [None, None]
        self.works = [None, None]

    def render(self, i: int):
        """Render step i into buffer i % 2 (no gather)."""
        k = i & 1
        if self.cuda and self.ev_gathered[k] is not None:
            torch.cuda.current_stream(self.device).wait_event(self.ev_gathered[k])
        self.render_fn(self.bufs[k][:len(self.views)])
        if self.cuda:
            self.ev_rendered[k].record()

    def gather(self, i: int):
        """X2 of step i's buffer to rank 0, on the communication stream (async on CUDA)."""
        k = i & 1
        if self.world == 1:
            return
        if self.cuda:
            with torch.cuda.stream(self.comm):
                self.comm.wait_event(self.ev_rendered[k])
                dist.gather(self.bufs[k], self.recv[k] if self.rank == 0 else None, dst=0)
                ev = torch.cuda.Event()
                ev.record(self.comm)
                self.ev_gathered[k] = ev
        else:
            dist.gather(self.bufs[k], self.recv[k] if self.rank == 0 else None, dst=0)

    def step(self, i: int):
        self.render(i)
        self.gather(i)

    def frames(self, i: int):
        """Rank 0: step i's gathered frames in view order [n_views, H, W, 4] (after sync)."""
        if self.rank != 0:
            return None
        k = i & 1
        if self.world == 1:
            return self.bufs[k][:self.n_views]
        parts = [self.recv[k][r][:len(views_for_rank(r, self.world, self.n_views))] for r in range(self.world)]
        return torch.cat(parts, dim=0)
