"""The N>1 path's host logic (view partition, X1 broadcast, X2 gather, max over
ranks) on world_size 2 with the gloo backend on CPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_08491_b200 import multigpu as mg


def test_views_partition():
    for n in (1, 7, 64):
        for w in (1, 2, 3, 8):
            got = [mg.views_for_rank(r, w, n) for r in range(w)]
            flat = [v for g in got for v in g]
            assert flat == list(range(n))
            assert max(map(len, got)) - min(map(len, got)) <= 1


def test_pack_unpack_roundtrip():
    import synth
    sc = synth.make_scene(0, 17)
    flat = mg.pack_params(sc, "cpu")
    assert flat.shape == (17, 99)
    back = mg.unpack_params(flat)
    for f in mg.PARAM_FIELDS:
        assert np.array_equal(getattr(back, f).numpy(), getattr(sc, f))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        n = 33
        flat = mg.pack_params(synth.make_scene(5, n), "cpu") if rank == 0 else torch.zeros(0)
        flat = mg.broadcast_params(flat, n, src=0)
        frames = torch.full((1, 4, 5, 4), float(rank + 1))
        got = mg.gather_frames(frames, dst=0)
        mx = mg.max_over_ranks(10.0 * (rank + 1), "cpu")
        q.put((rank, flat.sum().item(), None if got is None else [g[0, 0, 0, 0].item() for g in got], mx,
               mg.views_for_rank(rank, world, 64)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_collectives():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import synth
    want = mg.pack_params(synth.make_scene(5, 33), "cpu").sum().item()
    assert res[0][1] == pytest.approx(want) and res[1][1] == pytest.approx(want)   # X1
    assert res[0][2] == [1.0, 2.0] and res[1][2] is None                          # X2 at rank 0
    assert res[0][3] == 20.0 and res[1][3] == 20.0                                 # max over ranks
    assert res[0][4] == list(range(32)) and res[1][4] == list(range(32, 64))


def test_merge_stripes():
    H = 40
    fr = [torch.full((1, H, 3, 4), float(r)) for r in range(3)]
    m = mg.merge_stripes(fr, H)
    for y in range(H):
        assert m[0, y, 0, 0].item() == (y // 16) % 3


def _train_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2510_08491_b200 import train
        flat, views = train.flat_grads(synth.make_scene(5, 9), "cpu")
        for k, f in enumerate(views):            # rank-dependent per-field gradients
            views[f].fill_(float((rank + 1) * (k + 1)))
        train.allreduce_mean(flat)
        q.put((rank, {f: views[f].flatten()[0].item() for f in views}, flat.numel()))
    finally:
        dist.destroy_process_group()


def test_two_rank_gradient_allreduce():
    """the training step's single gradient exchange -- one flat
    buffer (views per parameter array) averaged over the ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_train_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 9
    assert res[0][2] == n * (3 + 4 + 3 + 24 + 8 + 8 + 1 + 48)
    for rank in (0, 1):
        for k, (f, v) in enumerate(res[rank][1].items()):
            assert v == pytest.approx(1.5 * (k + 1)), (rank, f, v)   # mean of 1x and 2x


def test_bench_launcher_two_ranks_gloo():
    """bench.py --gpus 2 re-launches itself under torch.distributed.run (2 ranks); the C4
    view-sharding and X2 protocol (multigpu.ShardedFrames, double-buffered gather to rank 0)
    runs over gloo with a deterministic stand-in for the GPU render, and rank 0 finds the
    gathered 64-view batch equal to the single-process one."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--selftest-cpu",
                        "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    assert lines[0]["n_gpus"] == 2 and lines[0]["bit_identical_to_single_gpu"] is True
