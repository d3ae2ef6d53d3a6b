"""Multi-process (world_size 2, gloo, CPU) coverage of the frame-sharded path.

The per-rank compute is the FP64 oracle here (these are CPU tests): what is under test is
the host-side logic — frame partition, reference handling in both modes (recompute /
NCCL-style broadcast), max-over-ranks timing — and that sharded results equal the
single-process stack bit for bit."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1910_11872_b200 import sharding, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_rank_frame_indices_partition():
    T = 5
    world = 3
    seen = []
    for r in range(world):
        idx = sharding.rank_frame_indices(r, world, T)
        assert idx[0] == 0 and len(idx) == T
        seen += idx[1:]
    assert sorted(seen) == list(range(1, world * (T - 1) + 1))
    assert sharding.distinct_output_frames(world, T) == world * (T - 1) + 1
    with pytest.raises(ValueError):
        sharding.rank_frame_indices(0, 1, 1)


def _oracle_demod(M):
    from oracle import rootmusic as R

    def demod_raw(frame):
        a, _ = R.demod_frame(frame.numpy(), M, threads=2)
        return torch.from_numpy(a.astype(np.float32))

    def demod(frames, ref):
        outs = []
        for t in range(frames.shape[0]):
            a, _ = R.demod_frame(frames[t].numpy(), M, threads=2)
            outs.append(R.wrap(a - ref.numpy().astype(np.float64)))
        return torch.from_numpy(np.stack(outs).astype(np.float32))

    return demod, demod_raw


def _worker(rank, world, port, mode, T, H, W, M, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = synth.workload("C3", H=H, W=W)
        idx = sharding.rank_frame_indices(rank, world, T)
        frames = synth.make_stack(w, frames=idx)
        demod, demod_raw = _oracle_demod(M)
        ref_buf = torch.empty(H, W, dtype=torch.float32)
        out, ref = sharding.sharded_stack_step(frames, demod, demod_raw, mode, ref_buf)
        t = sharding.max_over_ranks(float(rank + 1))
        g = sharding.gather_results(out)
        q.put((rank, idx, out.numpy(), ref.numpy(), t, None if g is None else g.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["recompute", "broadcast"])
def test_two_rank_sharded_stack_matches_single_process(mode):
    T, H, W, M = 3, 24, 20, 5
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, T, H, W, M, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    # single process over the global stack
    w = synth.workload("C3", H=H, W=W)
    demod, demod_raw = _oracle_demod(M)
    g = synth.make_stack(w, frames=range(world * (T - 1) + 1))
    ref = demod_raw(g[0])
    full = demod(g, ref).numpy()
    for rank, idx, out, rref, tmax, gathered in res:
        assert tmax == float(world)                       # MAX over ranks
        assert np.array_equal(rref, ref.numpy())          # identical reference on every rank
        assert np.array_equal(out, full[idx])             # bitwise equal to the 1-process stack
        if rank == 0:                                     # optional result gather (§8(e))
            assert np.array_equal(gathered, full)
        else:
            assert gathered is None


def test_bench_reference_arm_two_ranks_gloo():
    """`bench.py --impl reference` under torchrun (2 ranks, gloo on CPU): rank 0 prints one
    JSON line with impl=reference, the other rank exits 0 without work."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--size", "64",
           "--cpu-sample-px", "2048", "--cpu-sample-frames", "1"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
