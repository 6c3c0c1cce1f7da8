"""The N>1 bench path on CPU: 2 ranks over gloo (127.0.0.1).  Each rank must
draw its own disjoint block of the global cfg3 system stream (weak scaling,
no data-path collective) and the timing reduction must be the max over
ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import bench
    from paper_2412_08076_b200 import configs
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = configs.cfg3(first=rank * 2, count=2, n=32)          # small grid: host recipe only
    t = bench.max_over_ranks(float(rank + 1), world)           # rank-dependent "time"
    bench.barrier(world)
    out[rank] = {"eps": [p.epsilon for p in wl["problems"]], "f0": wl["F"][:, :4].copy(),
                 "tmax": t}
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_sharding_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    from paper_2412_08076_b200 import configs
    full = configs.cfg3(first=0, count=4, n=32)
    eps_all = [p.epsilon for p in full["problems"]]
    assert res[0]["eps"] + res[1]["eps"] == eps_all           # disjoint, in stream order
    assert np.array_equal(np.concatenate([res[0]["f0"], res[1]["f0"]]), full["F"][:, :4])
    assert res[0]["tmax"] == res[1]["tmax"] == 2.0            # max over ranks
