"""Data-parallel training step over camera views: every rank
renders its own views, takes the L1 loss (+ optional std(s) regulariser) and K7's
gradients, ONE all-reduce averages the flat gradient buffer over the ranks (NCCL over
NVLink on a multi-GPU node; gloo in the CPU tests), and every rank applies the same Adam
step to its replica of the parameters.  All arithmetic runs in libsnp's kernels; this
module only owns buffers and the collective."""
from __future__ import annotations

import numpy as np

from . import snp

CAMERA_BATCH = 32   # kCamsPerLaunch: the views one render / backward launch covers


def flat_grads(scene, device):
    """One contiguous float32 buffer with a view per parameter array (FIELDS order), so
    that the gradient exchange is a single all-reduce."""
    import torch
    shapes = [tuple(np.asarray(getattr(scene, f)).shape) for f in snp.FIELDS]
    sizes = [int(np.prod(s)) for s in shapes]
    flat = torch.zeros(sum(sizes), dtype=torch.float32, device=device)
    views, o = {}, 0
    for f, s, n in zip(snp.FIELDS, shapes, sizes):
        views[f] = flat[o:o + n].view(s)
        o += n
    return flat, views


def allreduce_mean(flat, group=None):
    """Sums the flat gradient buffer over the ranks and divides by the world size."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return flat
    dist.all_reduce(flat, group=group)
    flat.div_(dist.get_world_size(group))
    return flat


class Trainer:
    """Owns the per-rank buffers of one scene handle: image, dL/d(image), flat gradients,
    the loss scalar and the Adam step counter."""

    def __init__(self, h, scene, n_views, height, width, device, lr=None, reg_weight=0.0, opts=None,
                 check_every=50, dssim_lambda=0.2):
        import torch
        self.h, self.lr, self.reg = h, lr, float(reg_weight)
        # the paper's loss is 3DGS's: (1 - lambda) L1 + lambda D-SSIM, lambda = 0.2;
        # dssim_lambda = 0 takes the plain L1 kernel
        self.dssim_lambda = float(dssim_lambda)
        self.check_every = int(check_every)   # steps between checks of K7's skipped-pixel count
        self.opts = opts if opts is not None else snp.make_opts()
        self.out = torch.zeros((n_views, height, width, 4), device=device)
        self.gout = torch.zeros_like(self.out)
        self.flat, self.grads = flat_grads(scene, device)
        self.loss = torch.zeros(1, device=device)
        self.step_count = 0
        # the forward records its composited hits, so that the backward needs no second
        # traversal (snp_set_record); a step runs one camera batch (<= 32 views) at a time
        snp.set_record(h, True)

    def step(self, cams, target_rgb, group=None):
        """One training step on this rank's views (target_rgb [n_views, H, W, 3]); returns
        this rank's loss (a device scalar, read by the caller when it wants it)."""
        self.flat.zero_()
        self.loss.zero_()
        V = len(cams)
        for v0 in range(0, V, CAMERA_BATCH):   # render + loss + backward per camera batch
            v1 = min(V, v0 + CAMERA_BATCH)
            out, gout = self.out[v0:v1], self.gout[v0:v1]
            snp.render_views(self.h, cams[v0:v1], self.opts, out)
            if self.dssim_lambda > 0.0 or V > CAMERA_BATCH:   # (the means are the whole step's)
                snp.loss_3dgs(self.h, out, target_rgb[v0:v1], gout, self.loss, self.dssim_lambda, step_views=V)
            else:
                snp.loss_l1(out, target_rgb, gout, self.loss)
            snp.render_backward(self.h, self.opts, gout, self.grads, fwd_rgba=out)
            if self.check_every and self.step_count % self.check_every == 0:
                skipped = snp.get_stats(self.h)["backward_skipped"]   # (synchronises; per backward call)
                if skipped:
                    raise RuntimeError(f"snp_render_backward skipped {skipped} pixels with more than 16384 hits")
        if self.reg > 0.0:
            snp.scale_regularizer(self.h, self.reg, self.grads["scales"], self.loss)
        allreduce_mean(self.flat, group)
        self.step_count += 1
        snp.adam_step(self.h, self.grads, self.step_count, self.lr)
        return self.loss
