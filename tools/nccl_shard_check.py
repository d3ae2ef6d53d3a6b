"""Multi-GPU check of the frame-sharded CUDA path (run under torchrun, one rank per GPU, NCCL).

Every rank demodulates its local stack with libbosrm.so (sharding.sharded_stack_step, the
reference either recomputed on every rank or demodulated on rank 0 and NCCL-broadcast), then
rank 0 gathers the flow-frame maps (sharding.gather_results) and compares them bit for bit
with a single-GPU demodulation of the whole global stack.  Prints one JSON line on rank 0.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/nccl_shard_check.py --mode broadcast
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1910_11872_b200 import bosrm, sharding, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="recompute", choices=["recompute", "broadcast"])
    ap.add_argument("--frames", type=int, default=4, help="frames per rank incl. the reference")
    ap.add_argument("--size", type=int, default=256)
    ap.add_argument("--window-len", type=int, default=8)
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    M, T, H = a.window_len, a.frames, a.size
    w = synth.workload("C3", H=H, W=H, window_len=M)
    idx = sharding.rank_frame_indices(rank, world, T)
    frames = synth.make_stack(w, frames=idx, device=dev)
    ref_buf = torch.empty(H, H, dtype=torch.float32, device=dev)

    def demod_raw(fr):
        bosrm.bos_rootmusic_demod(fr.unsqueeze(0), M, out_phase=ref_buf.view(1, H, H))
        return ref_buf

    def demod(fr, ref):
        return bosrm.bos_rootmusic_demod(fr, M, ref_phase=ref)[0]

    out, ref = sharding.sharded_stack_step(frames, demod, demod_raw, a.mode, ref_buf)
    torch.cuda.synchronize()
    gathered = sharding.gather_results(out)
    ok = None
    if rank == 0:
        full = synth.make_stack(w, frames=range(sharding.distinct_output_frames(world, T)), device=dev)
        single, _, ref1 = bosrm.bos_rootmusic_demod_stack(full, M, ref_index=0)
        ok = bool(torch.equal(gathered.to(dev), single)) and bool(torch.equal(ref, ref1))
        print(json.dumps({"world": world, "mode": a.mode, "bitwise_equal": ok,
                          "frames": int(single.shape[0]), "H": H, "window_len": M}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
