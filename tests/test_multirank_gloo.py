"""N > 1 host logic on CPU: two gloo ranks each own the blocks k % 2 == rank
(R17), run their shard of the working-set step (oracle shards stand in for the
per-GPU path here: no GPU on this box) and do the two collectives of the
multi-GPU path -- C1 active-set all-gather and C2 count all-reduce -- with the
same paper_2605_20150_b200.shard functions the bench uses over NCCL."""
import json
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, iters):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import oracle as O
    from helpers import tiny
    from paper_2605_20150_b200 import shard

    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, sc, tr = tiny()
    cap = shard.shard_capacity(cfg.capacity, world)
    o = O.Oracle(O.make_config(sc.N, sc.B, cap, world_size=world, rank=rank), sc.bounds(),
                 fill=None, track_all=False)
    full = O.Oracle(O.make_config(sc.N, sc.B, cfg.capacity), sc.bounds(), fill=None,
                    track_all=False) if rank == 0 else None
    log = []
    for t in range(iters):
        planes = tr.batch_planes(t, cfg.J)
        assert o.activate(planes) == O.OK
        A = o.list("A")
        K = o.list("K")
        gathered, union = shard.exchange_active(torch.from_numpy(A.astype(np.int64)), cap)
        every = [None] * world
        dist.all_gather_object(every, {"A": A.tolist(), "K": K.tolist()})
        st = o.stats()
        counts = torch.tensor([len(K), o.list("R").size, o.list("S+").size, o.list("S-").size,
                               len(A)], dtype=torch.int64)
        shard.reduce_counts(counts)
        rec = {"union": union.tolist(), "every": every, "counts": counts.tolist(),
               "mine": [len(K), int(o.list("R").size), int(o.list("S+").size),
                        int(o.list("S-").size), len(A)],
               "owned_ok": bool(all(int(k) % world == rank for k in np.concatenate([A, K]))),
               "h2d": st["h2d_bytes"]}
        if full is not None:
            full.activate(planes)
            rec["K_single"] = full.list("K").tolist()
        log.append(rec)
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(log, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_gloo_ranks_exchange_and_reduce(tmp_path):
    import torch.multiprocessing as mp
    world, iters = 2, 10
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), iters), nprocs=world, join=True)
    logs = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    for t in range(iters):
        r0, r1 = logs[0][t], logs[1][t]
        assert r0["owned_ok"] and r1["owned_ok"]
        A_all = sorted(r0["every"][0]["A"] + r0["every"][1]["A"])
        # C1: every rank holds the same global active set = union of the shards'
        assert r0["union"] == r1["union"] == A_all
        # C2: summed counts on both ranks
        summed = [a + b for a, b in zip(r0["mine"], r1["mine"])]
        assert r0["counts"] == r1["counts"] == summed
        # Level-1 culling is per block, so the shards' K partition the single-GPU K
        K_union = sorted(r0["every"][0]["K"] + r0["every"][1]["K"])
        assert K_union == r0["K_single"]


def test_shard_arithmetic():
    from paper_2605_20150_b200 import shard
    K = 64
    for G in (1, 2, 3, 8):
        assert sum(shard.shard_blocks(K, G, r) for r in range(G)) == K
        for k in range(K):
            r = shard.owner(k, G)
            assert shard.global_from_local([shard.local_id(k, G)], G, r)[0] == k
    assert shard.shard_capacity(6309, 8) == 789
