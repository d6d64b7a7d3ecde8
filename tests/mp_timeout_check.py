"""A peer that never arrives must yield a status, not a hang (one process per GPU).

Rank 1 creates its layer (windows mapped) and then stays away from moe_forward; rank 0's
forward enqueues the fused dispatch and the window barrier, whose bounded spin gives up
after peer_timeout_ms and records the failure in the communicator's host-mapped error
word. Rank 0's next call returns MOE_ERR_TIMEOUT, the one after MOE_ERR_STATE (poisoned).

    torchrun --nproc-per-node 2 tests/mp_timeout_check.py
"""
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2305_13525_b200 import MoEConfig, MoEError, MoELayer  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo")
    cfg = MoEConfig(1024, 256, 512, 8, 1.0, 1, world, True, 1, peer_timeout_ms=2000)
    layer = MoELayer(cfg, world, rank, dev)
    x = torch.randn(1024, 256, device=dev).to(torch.bfloat16)
    wg = torch.randn(256, 8, device=dev) / 16
    w1 = (torch.randn(8 // world, 512, 256, device=dev) / 16).to(torch.bfloat16)
    w2 = (torch.randn(8 // world, 256, 512, device=dev) / 22).to(torch.bfloat16)
    ok = True
    if rank == 0:
        names = []
        t0 = time.time()
        for _ in range(3):
            try:
                layer.moe_forward(x, wg, w1, w2)
                torch.cuda.synchronize()
                names.append("MOE_OK")
            except MoEError as e:
                names.append(e.name)
        dt = time.time() - t0
        # the first forward is enqueued fine; its barrier times out on the device
        ok = names == ["MOE_OK", "MOE_ERR_TIMEOUT", "MOE_ERR_STATE"] and dt < 30
        print(f"[rank 0] {names} in {dt:.1f}s", "ok" if ok else "FAIL", flush=True)
    dist.barrier()  # rank 1 keeps its windows mapped until rank 0 is done
    layer.close()
    flag = torch.tensor([0 if ok else 1])
    dist.all_reduce(flag)
    dist.destroy_process_group()
    sys.exit(int(flag.item()))


if __name__ == "__main__":
    main()
