"""The sharded path with the library's own collectives: two
processes, each a rank of libtidegs (world size 2, rank r, capacity C_g) on the
same GPU, gloo as the transport of tgs_set_comm (NCCL refuses two ranks on one
device).  Every batch, every rank's lists, slots and counters are compared with
the oracle's shard r; the C1 result (tgs_activation.d_global_active) must hold
every rank's oracle A list, and after every step the C2 result
(tgs_get_global_stats) must equal the sum of the oracle shards' counters."""
import json
import os
import socket
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, iters, moments, xfer):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle as O
    from gpu_harness import Pair
    from helpers import tiny
    from paper_2605_20150_b200 import shard
    from paper_2605_20150_b200 import tidegs as T

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfg, sc, tr = tiny()
    cap = shard.shard_capacity(cfg.capacity, world)
    pr = Pair(sc, capacity=cap, world_size=world, rank=rank, moments=moments, xfer=xfer)
    pr.gpu.set_comm(T.torch_comm())
    log = {"batches": 0, "c1_rows": [], "errors": []}
    try:
        for t in range(iters):
            act = pr.activate(tr.batch_planes(t, cfg.J))
            pr.t = t
            pr.compare_plan(cfg.J)
            pr.compare_evicted_dirty()
            A = pr.orc.list("A")
            every = [None] * world
            dist.all_gather_object(every, A.tolist())
            got = pr.gpu.global_active(act)
            for r in range(world):
                row = got[r]
                ids = row[row != 0xFFFFFFFF].tolist()
                assert ids == every[r], (t, r, ids, every[r])
                assert (row[len(ids):] == 0xFFFFFFFF).all()
            assert pr.step(act, t) == O.OK
            ostats = [None] * world
            dist.all_gather_object(ostats, pr.orc.stats())
            want = {k: sum(s[k] for s in ostats) for k in ostats[0]}
            g = pr.gpu.global_stats()
            for k in ("flush_bytes", "n_flush_blocks"):
                want[k] = g[k] = 0
            assert g == want, {k: (g[k], want[k]) for k in g if g[k] != want[k]}
            pr.compare_stats()
            log["batches"] += 1
            log["c1_rows"].append([len(e) for e in every])
        assert pr.compare_blocks([k for k in range(sc.K) if k % world == rank]) == 0
    except Exception as e:  # reported by the parent
        log["errors"].append(repr(e))
    finally:
        pr.close()
        with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
            json.dump(log, f)
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.parametrize("moments,xfer", [(0, 0), (1, 0), (0, 1)])
def test_two_ranks_of_libtidegs_with_c1_c2(tmp_path, moments, xfer):
    """xfer: 0 = TMA transfer kernels, 1 = copy-engine runs (the bench default)"""
    import torch.multiprocessing as mp
    world, iters = 2, 16
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), iters, moments, xfer),
             nprocs=world, join=True)
    for r in range(world):
        log = json.load(open(tmp_path / f"rank{r}.json"))
        assert not log["errors"], log["errors"]
        assert log["batches"] == iters
        assert any(sum(x) > 0 for x in log["c1_rows"])
