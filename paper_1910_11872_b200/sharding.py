"""Frame sharding across ranks (one process per GPU; torch.distributed for the plumbing).

Every frame and pixel is independent; the only cross-frame dependency of a
time-lapse stack is the reference phase φ_ref.  Each rank holds a stack of
T frames: local frame 0 is the global reference frame, local frames 1..T−1 are the global
flow frames r·(T−1)+1 … (r+1)·(T−1).  Two reference modes:

* "recompute" (default): every rank demodulates the reference frame itself.  The kernel is
  deterministic, so φ_ref is bitwise identical on all ranks, and it costs exactly what
  waiting for rank 0's result would — no collective on the data path.
* "broadcast": rank 0 demodulates the reference and NCCL-broadcasts φ_ref (4·H·W bytes)
  over NVLink; the others wait for it.  For streams whose reference frame lives on one
  rank only.

``gather_results`` is the optional result gather of SURVEY §8(e): the ranks' flow-frame phase
maps assembled on one rank in global frame order (not part of the timed step).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def rank_frame_indices(rank: int, world: int, T: int) -> list[int]:
    """Global frame indices of rank's local stack: [0] + its T−1 flow frames."""
    if T < 2:
        raise ValueError("a time-lapse stack needs a reference and at least one flow frame")
    del world
    return [0] + list(range(rank * (T - 1) + 1, (rank + 1) * (T - 1) + 1))


def fixed_stack_indices(rank: int, world: int, T: int) -> list[int]:
    """Strong scaling of ONE fixed T-frame stack (C5): rank r owns the global
    frames [⌊rT/G⌋, ⌊(r+1)T/G⌋); its local stack is the reference (global frame 0) followed by
    its own frames other than 0 (rank 0's range starts with the reference itself, whose output
    is φ_ref − φ_ref = 0 and is written by the raw reference demod's difference anyway)."""
    if T < 2 or not 0 <= rank < world:
        raise ValueError("need T >= 2 and 0 <= rank < world")
    lo, hi = rank * T // world, (rank + 1) * T // world
    return [0] + [t for t in range(lo, hi) if t != 0]


def distinct_output_frames(world: int, T: int) -> int:
    """Distinct output frames of the whole job: the reference plus every rank's flow frames."""
    return world * (T - 1) + 1


def is_dist() -> bool:
    return dist.is_available() and dist.is_initialized()


def max_over_ranks(x: float, device=None) -> float:
    if not is_dist() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sharded_stack_step(local_frames: torch.Tensor, demod, demod_raw, ref_mode: str = "recompute",
                       ref_buf: torch.Tensor | None = None):
    """One step on this rank's local stack (local frame 0 = global reference).

    demod(frames, ref) -> phases;  demod_raw(frame) -> raw α of one frame.
    Returns (phases [T,H,W], φ_ref [H,W])."""
    rank = dist.get_rank() if is_dist() else 0
    if ref_mode == "recompute" or not is_dist():
        ref = demod_raw(local_frames[0])
    elif ref_mode == "broadcast":
        if rank == 0:
            ref = demod_raw(local_frames[0])
            if ref_buf is not None:
                ref_buf.copy_(ref)
                ref = ref_buf
        else:
            ref = ref_buf if ref_buf is not None else torch.empty(
                local_frames.shape[-2:], dtype=torch.float32, device=local_frames.device)
        dist.broadcast(ref, src=0)
    else:
        raise ValueError(ref_mode)
    return demod(local_frames, ref), ref


def gather_results(local_out: torch.Tensor, dst: int = 0):
    """Assemble the job's output stack on rank ``dst``: [world·(T−1)+1, H, W] in global frame
    order (frame 0 = the reference's own output, identical on every rank), None elsewhere.
    local_out: this rank's [T, H, W] output (local frame 0 = the reference).  One collective
    (all_gather of the flow frames: NCCL supports it on every build; gather is not universal)."""
    if not is_dist() or dist.get_world_size() == 1:
        return local_out
    world, rank = dist.get_world_size(), dist.get_rank()
    flows = local_out[1:].contiguous()
    parts = [torch.empty_like(flows) for _ in range(world)]
    dist.all_gather(parts, flows)
    if rank != dst:
        return None
    return torch.cat([local_out[:1]] + parts, dim=0)

