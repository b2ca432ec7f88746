"""Multi-process host logic of the prompt-sharded path on CPU (gloo, world 2):
shard bounds cover every prompt exactly once, counter vectors and metric
counters sum like SimReport.merge (engine.py:94-110), per-prompt counters
gather, and the combined report equals a single-process reference report."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.timeout(240)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2508_17137_b200 as m
    from paper_2508_17137_b200 import distributed as D
    shape = m.ModelShape(3, 8, 2)
    L = shape.num_layers
    lens = np.array([5, 1, 9, 2, 7, 3, 3, 8, 4])
    off = np.concatenate([[0], np.cumsum(lens * L)]).astype(np.int64)
    packed = m.PackedTraces(shape, torch.zeros((int(off[-1]), 1), dtype=torch.int64),
                            torch.from_numpy(off), off, np.arange(100, 109))
    local = packed.shard(rank, world)
    # synthetic per-prompt counters: derived from prompt id so the total is known
    pp = np.stack([np.array([pid, pid % 7, pid % 3, 0]) for pid in local.prompt_ids])
    vec = np.zeros(4 + 3 * L, dtype=np.int64)
    vec[:4] = pp.sum(0)
    vec[4:4 + L] = len(local.prompt_ids)
    rep = D.combine_reports(shape, torch.from_numpy(vec), pp, local.prompt_ids)
    met = D.combine_metrics(torch.arange(3 * 8 + 3, dtype=torch.int64) * (rank + 1), 8)
    out_q.put((rank, local.prompt_ids.tolist(), rep.measured_accesses, rep.cache_hits,
               sorted(rep.per_prompt), rep.layer_accesses.tolist(), met.tp.tolist(),
               met.positions))
    dist.destroy_process_group()


def test_gloo_world2_combine():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=200) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids = res[0][1] + res[1][1]
    assert ids == list(range(100, 109))  # every prompt exactly once, in order
    pids = np.arange(100, 109)
    for r in res:
        assert r[2] == pids.sum()                  # summed measured accesses
        assert r[3] == (pids % 7).sum()            # summed cache hits
        assert r[4] == list(range(100, 109))       # gathered per-prompt
        assert r[5] == [9, 9, 9]                   # per-layer sums
        assert r[6] == [3 * i for i in range(8)]   # metric counters summed (1x + 2x)
        assert r[7] == 3 * 24
