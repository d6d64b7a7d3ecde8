"""NCCL grouped send/recv vs raw peer copy bandwidth (torchrun, 2+ ranks)."""
import os
import time

import torch
import torch.distributed as dist


def main():
    rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    total = 32 << 20  # bytes per peer
    for pieces in (1, 8, 32):
        n = total // 2 // pieces
        sb = [torch.ones(n, dtype=torch.bfloat16, device=dev) for _ in range(pieces * world)]
        rb = [torch.empty(n, dtype=torch.bfloat16, device=dev) for _ in range(pieces * world)]
        def run():
            ops = []
            for p in range(world):
                if p == rank:
                    continue
                for i in range(pieces):
                    ops.append(dist.P2POp(dist.isend, sb[p * pieces + i], p))
                    ops.append(dist.P2POp(dist.irecv, rb[p * pieces + i], p))
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        for _ in range(3):
            run()
        torch.cuda.synchronize(); dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            run()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        gbs = total * (world - 1) / ms / 1e6
        if rank == 0:
            print(f"nccl send/recv pieces={pieces:3d}: {ms*1e3:8.1f} us  {gbs:7.1f} GB/s per rank egress "
                  f"(MIN_P2P_NCHANNELS={os.environ.get('NCCL_MIN_P2P_NCHANNELS','-')})", flush=True)
    dist.barrier()
    # all-to-all single call
    x = torch.ones(total // 2 * world, dtype=torch.bfloat16, device=dev)
    y = torch.empty_like(x)
    for _ in range(3):
        dist.all_to_all_single(y, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        dist.all_to_all_single(y, x)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    if rank == 0:
        print(f"nccl all_to_all_single: {ms*1e3:8.1f} us  {total*(world-1)/ms/1e6:7.1f} GB/s per rank egress", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
