"""N > 1 host logic on CPU: world-size-2 and -4 gloo process groups (no GPU).

Each rank plans its layout and collective schedule through the C ABI and the
ranks cross-check over gloo: the rank grid is a bijection onto (d, ep, t),
expert / F shards tile the weights exactly once per G_data replica, every
member of a TP or EP group issues the same collective sequence with the same
sizes (NCCL matching), and the NCCL unique id broadcast used by MoELayer
works over a CPU process group.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_13525_b200 import MoEConfig, binding, moe_plan_collectives, moe_plan_layout

CASES = [(2, 2, 1), (2, 1, 2), (4, 2, 2), (4, 1, 4), (4, 4, 1), (4, 1, 2)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, gt, gep, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cfg = MoEConfig(4096, 512, 2048, 16, 1.0, gt, gep, True)
        lay = moe_plan_layout(cfg, world, rank)
        sched = moe_plan_collectives(cfg, world, rank)
        out = [None] * world
        dist.all_gather_object(out, (lay, sched))
        # unique-id broadcast as MoELayer does it
        obj = [binding.moe_get_unique_id() if rank == 0 else None]
        uid_ok = True
        try:
            dist.broadcast_object_list(obj, src=0)
            uid_ok = isinstance(obj[0], bytes) and len(obj[0]) == 128
        except binding.MoEError:
            uid_ok = None
        if rank == 0:
            q.put((out, uid_ok))
        dist.destroy_process_group()
    except Exception as e:  # surface to the parent
        q.put(("error", repr(e)))


@pytest.mark.parametrize("world,gt,gep", CASES)
def test_rank_grid_and_schedules_over_gloo(world, gt, gep):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, gt, gep, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert res[0] != "error", res
    out, uid_ok = res
    assert uid_ok in (True, None)
    lays = [o[0] for o in out]
    scheds = [o[1] for o in out]
    gd = world // (gt * gep)
    coords = {(L["d"], L["ep"], L["t"]) for L in lays}
    assert len(coords) == world and coords == {(d, e, t) for d in range(gd) for e in range(gep) for t in range(gt)}
    El, Fl = lays[0]["experts_local"], lays[0]["ffn_local"]
    for d in range(gd):
        owned = {}
        for L in lays:
            if L["d"] != d:
                continue
            for e in range(L["ep"] * El, (L["ep"] + 1) * El):
                owned.setdefault(e, []).append((L["t"] * Fl, (L["t"] + 1) * Fl))
        assert sorted(owned) == list(range(16))
        for e, spans in owned.items():
            assert sorted(spans) == [(t * Fl, (t + 1) * Fl) for t in range(gt)]
    # NCCL matching: same sequence and sizes within TP groups and within EP groups
    key = lambda s: [(c["kind"], c["pass"], c["group_size"], c["buffer_bytes"]) for c in s]  # noqa: E731
    for r, L in enumerate(lays):
        for r2, L2 in enumerate(lays):
            same_tp = (L["d"], L["ep"]) == (L2["d"], L2["ep"])
            same_ep = (L["d"], L["t"]) == (L2["d"], L2["t"])
            if same_tp or same_ep:
                assert key(scheds[r]) == key(scheds[r2])
    # DTD cuts a2a bytes by G_tensor
    if gep > 1 and gt > 1:
        van = moe_plan_collectives(MoEConfig(4096, 512, 2048, 16, 1.0, gt, gep, False), world, 0)
        a2a = lambda s: sum(c["wire_bytes"] for c in s if c["kind"] == "a2a")  # noqa: E731
        assert a2a(scheds[0]) * gt == a2a(van)
