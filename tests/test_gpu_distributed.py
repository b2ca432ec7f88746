"""The drop-in replay_traces / sweep with a torch.distributed group of two
ranks (gloo, both ranks on cuda:0 as bench.py's MOEB_BENCH_ONE_DEVICE path
does on a one-GPU box): each rank passes the same traces, replays its
row-balanced prompt shard on the GPU, and every rank returns a SimReport
bit-identical to the one-process replay, per-prompt counters included -- the
analogue of the reference's jobs-invariance test (test_engine.py:104-119);
the sharded metric counters (distributed.metrics_sharded) equal the
one-process prediction_metrics.
jobs > 1 in one process with one visible GPU is the one-device replay."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]

FRACS = [0.05, 0.1, 0.25]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _setup(m):
    shape = m.ModelShape(26, 64, 6)
    packed = m.generate_packed(m.GeneratorConfig(37, 40, shape, 8, 0.9, 7), "cuda:0")
    w = np.random.default_rng(0).normal(0.0, 0.01, (64, 91))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    cfg = m.ReplayConfig(shape, m.CacheConfig(capacity_fraction=0.1, prefetch_budget=6),
                         warmup_tokens=8)
    return shape, packed, model, cfg


def _summary(rep):
    return (rep.measured_accesses, rep.cache_hits, rep.prediction_hits, rep.uncovered_queries,
            rep.layer_accesses.tolist(), rep.layer_cache_hits.tolist(),
            rep.layer_prediction_hits.tolist(),
            sorted((pid, c.measured_accesses, c.cache_hits, c.prediction_hits)
                   for pid, c in rep.per_prompt.items()))


def _metrics(mc):
    return (mc.tp.tolist(), mc.fp.tolist(), mc.fn.tolist(), mc.positions, mc.exact,
            mc.label_correct)


def _results(m):
    shape, packed, model, cfg = _setup(m)
    out = {}
    lin = m.make_predictor("learned_linear", shape, model=model)
    if dist.is_initialized():  # the sharded metric counters (one all-reduce)
        from paper_2508_17137_b200.distributed import metrics_sharded
        out["metrics"] = _metrics(metrics_sharded(packed, lin, cfg))
    else:
        out["metrics"] = _metrics(m.prediction_metrics(packed, lin, cfg))
    for kind in ("learned_linear", "lru_only"):
        pred = (m.make_predictor(kind, shape, model=model) if kind == "learned_linear"
                else m.make_predictor(kind, shape))
        out[kind] = _summary(m.replay_traces(packed, pred, cfg))
        pts = m.sweep(packed, (lambda: m.make_predictor(kind, shape, model=model))
                      if kind == "learned_linear" else (lambda: m.make_predictor(kind, shape)),
                      kind, FRACS, shape, 6, 8)
        out[kind + "_sweep"] = [_summary(p.report) for p in pts]
    return out


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2508_17137_b200 as m
    m.load_library()
    q.put((rank, _results(m)))
    dist.destroy_process_group()


def test_replay_traces_world2_equals_one_process():
    import paper_2508_17137_b200 as m
    m.load_library()
    want = _results(m)
    shape, packed, model, cfg = _setup(m)
    jobs = m.replay_traces(packed, m.make_predictor("learned_linear", shape, model=model), cfg,
                           jobs=4)
    assert _summary(jobs) == want["learned_linear"]
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted((q.get(timeout=240) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, res in got:
        assert res == want, rank
