"""Benchmark: trace tokens/sec of predict + cache-sim (+ F1/accuracy counters)
on DeepSeek-V2-Lite-shaped synthetic traces (BASELINE.json configs[1], C2:
6,994 prompts x 363 decode tokens x 26 MoE layers x 64 experts, top-6,
~66 M trace rows per GPU), learned_linear predictor with random-init weights,
expert cache at 10 % capacity (166 entries), prefetch budget 6, warm-up 8.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0 (contract in the task statement). Multi-GPU: one
process per GPU under torchrun; every rank replays its own C2-sized prompt
range (weak scaling, prompts are independent) and the int64 counters are
summed with one NCCL all-reduce per step.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

C2 = dict(prompts=6994, tokens=363, layers=26, experts=64, top_k=6, hot=8, skew=0.9, seed=7)
CAP_FRACTION = 0.1
BUDGET = 6
WARMUP_TOKENS = 8


def _config(P, rows, cap, world):
    """The workload description both arms report (BASELINE configs[1], C2)."""
    return {"workload": f"C2: {P} prompts x {C2['tokens']} tokens per GPU, "
                        "DeepSeek-V2-Lite 26 MoE layers x 64 experts top-6",
            "rows_per_gpu": rows, "predictor": "learned_linear (random init, seed 0)",
            "capacity_entries": cap, "prefetch_budget": BUDGET,
            "warmup_tokens": WARMUP_TOKENS, "parallelism": f"prompt-sharded x{world}",
            "l2": "inputs (528 MB/GPU) larger than L2"}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), float(
            p.get("bf16_tflops_sustained", p["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None
        self.out = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        if os.environ.get("MOEB_BENCH_NO_CLOCKS") == "1":  # diagnosis only
            return self
        try:
            self.out = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.out, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.proc = None
        if self.out is not None:
            self.out.close()
            self.out = None

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 8:
                    continue
                try:
                    sm.append(float(f[1]))
                    smax = float(f[2])
                except ValueError:
                    continue
                for n, v in zip(names, f[-4:]):
                    if v.lower() == "active":
                        reasons.add(n)
        except Exception:
            pass
        finally:
            if self.path and os.path.exists(self.path):
                os.remove(self.path)
        busy = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# Reference CPU arm: the unmodified reference package (baseline/_ref).
# ---------------------------------------------------------------------------

def _import_reference():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "moesim")) and ref not in sys.path:
        sys.path.insert(0, ref)
    import moesim  # noqa: F401
    return moesim


def reference_sample(n_prompts: int, tokens: int = C2["tokens"], first: int = 0):
    moesim = _import_reference()
    from moesim.learner import LearnerConfig, LinearModel
    shape = moesim.ModelShape(C2["layers"], C2["experts"], C2["top_k"])
    traces = moesim.generate_synthetic(moesim.GeneratorConfig(
        n_prompts, tokens, shape, C2["hot"], C2["skew"], C2["seed"], first_prompt_id=first))
    w = __import__("numpy").random.default_rng(0).normal(0.0, 0.01, (C2["experts"],
                                                                   C2["layers"] + C2["experts"] + 1))
    model = LinearModel(shape, LearnerConfig(epochs=0), w, trained=True)
    pred = moesim.make_predictor("learned_linear", shape, model=model)
    cfg = moesim.ReplayConfig(shape, moesim.CacheConfig(capacity_fraction=CAP_FRACTION,
                                                        prefetch_budget=BUDGET),
                              warmup_tokens=WARMUP_TOKENS)
    return moesim, traces, pred, cfg


def time_reference(n_prompts: int, jobs: int, repeats: int = 1, sample=None):
    """Reference predict + cache-sim (replay_traces, its own ProcessPool with
    `jobs` workers) over a bounded sample; returns (tok/s, seconds, report)."""
    moesim, traces, pred, cfg = sample if sample is not None else reference_sample(n_prompts)
    best = None
    rep = None
    for _ in range(repeats):
        t0 = time.perf_counter()
        rep = moesim.replay_traces(traces, pred, cfg, jobs=jobs)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    toks = n_prompts * C2["tokens"]
    return toks / best, best, rep


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor()


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    n_sample = max(16 * cores, 256)  # ~10 s of the reference's predict + replay per step
    try:
        _import_reference()
    except Exception as exc:  # pragma: no cover
        print(json.dumps({"impl": "reference", "unavailable": f"reference import failed: {exc}"}))
        return 0
    sample = reference_sample(n_sample)  # generation is not timed
    for _ in range(min(args.warmup, 1)):
        time_reference(n_sample, cores, sample=sample)
    vals = []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        v, dt, rep = time_reference(n_sample, cores, sample=sample)
        vals.append(v)
    elapsed = time.perf_counter() - t_all
    value = statistics.median(vals)
    sample = (f"{n_sample} prompts x {C2['tokens']} tokens of the C2 generator (seed 7), "
              f"learned_linear random-init + LRU 10%, moesim.replay_traces(jobs={cores})")
    line = {
        "impl": "reference", "metric": "trace tokens/sec (predict+cache-sim)",
        "value": value, "unit": "trace tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * elapsed / max(1, args.steps),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator)",
        "config": dict(_config(C2["prompts"], C2["prompts"] * C2["tokens"] * C2["layers"], 166,
                               world),
                       sampled=f"each step replays {n_sample} of the {C2['prompts']} prompts "
                               "(bounded CPU sample, see cpu_baseline)"),
        "cpu_baseline": {"value": value, "unit": "trace tokens/s", "cores": cores,
                         "kind": "reference", "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "trace tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "hit_rate_10pct": {"learned_linear": rep.cache_hit_rate},
        "counters": {"prompts": f"0..{n_sample - 1}", "measured_accesses": rep.measured_accesses,
                     "cache_hits": rep.cache_hits, "prediction_hits": rep.prediction_hits,
                     "uncovered_queries": rep.uncovered_queries},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# Our arm.
# ---------------------------------------------------------------------------

def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2508_17137_b200 as m

    world, rank, local = _dist()
    if world > 1:
        # MOEB_BENCH_ONE_DEVICE=1 + MOEB_BENCH_DIST_BACKEND=gloo run every rank
        # on cuda:0 (a check of the multi-rank code path on a single-GPU box)
        if os.environ.get("MOEB_BENCH_ONE_DEVICE") == "1":
            local = 0
        torch.cuda.set_device(local)
        backend = os.environ.get("MOEB_BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    m.load_library()
    shape = m.ModelShape(C2["layers"], C2["experts"], C2["top_k"])
    P = args.prompts
    gen = m.GeneratorConfig(P, C2["tokens"], shape, C2["hot"], C2["skew"], C2["seed"],
                            first_prompt_id=rank * P)
    t0 = time.perf_counter()
    packed = m.generate_packed(gen, dev)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    rows = packed.rows
    L, E = shape.num_layers, shape.num_experts
    cap = m.CacheConfig(capacity_fraction=CAP_FRACTION).resolve_capacity(shape)
    w = np.random.default_rng(0).normal(0.0, 0.01, (E, L + E + 1))
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), w, trained=True)
    pred = m.make_predictor("learned_linear", shape, model=model)
    tokens_per_rank = P * C2["tokens"]

    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    # --overlap-steps: step i+1's predictor runs while step i's replay and
    # metrics finish (two mask buffers; the timed region ends after a join)
    pipe = m.PipelinedReplay(packed, args.chunks, overlap_steps=args.overlap_steps)

    def step(timing=None):
        vec = m.metrics.metric_vector(E, dev)
        # per-prompt counters too, as the reference's replay_traces fills
        # SimReport.per_prompt (engine.py:75, 148)
        counters = pipe.run(pred, [cap], WARMUP_TOKENS, BUDGET, metrics=vec, timing=timing,
                            per_prompt=True)
        if world > 1:
            # the counter reduce (NCCL) waits on this step's replay and metrics
            # streams only, so overlapped steps keep overlapping
            s_comm.wait_stream(pipe.s_sim)
            s_comm.wait_stream(pipe.s_met)
            s_comm.wait_stream(stream)
            with torch.cuda.stream(s_comm):
                buf = torch.cat([counters.view(-1), vec])
                dist.all_reduce(buf)
                counters = buf[:counters.numel()].view(counters.shape)
                vec = buf[counters.numel():]
            if not pipe.overlap:
                stream.wait_stream(s_comm)
        return counters, vec

    s_comm = torch.cuda.Stream(dev)

    # --- warm-up ---
    # The clock sampler (an nvidia-smi process) starts before the warm-up so
    # its NVML start-up is over before the timed region; it keeps sampling
    # through the timed region.
    # At least W warm-up steps, and at least ~2 s of them: a first run on a
    # box that just finished other GPU work was occasionally slow for its
    # first hundreds of milliseconds.
    clocks = ClockSampler(torch.cuda.current_device()).__enter__()
    t_w = time.perf_counter()
    n_w = 0
    while True:
        counters, vec = step()
        n_w += 1
        if n_w % 8 == 0:
            torch.cuda.synchronize()
        done = n_w >= args.warmup and time.perf_counter() - t_w >= 2.0
        if world > 1:  # every rank runs the same number of steps (each has collectives)
            flag = torch.tensor([0 if done else 1], dtype=torch.int32, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MAX)
            done = int(flag.item()) == 0
        if done:
            break
    pipe.join()
    torch.cuda.synchronize()

    # --- timed region: device clock, max over ranks ---
    hbm, bf16, bf16_sus, peak_kind = _peaks()
    timing = []
    try:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        start, end = ev(), ev()
        start.record(stream)
        for _ in range(args.steps):
            counters, vec = step(timing)
        pipe.join()
        stream.wait_stream(s_comm)
        end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    finally:
        clocks.__exit__(None, None, None)
    ms = start.elapsed_time(end)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = tokens_per_rank * world / (ms / 1000.0) * args.steps
    # per-step kernel time of each stage (sum over the step's chunk launches;
    # launches of the two stages overlap on separate streams)
    if os.environ.get("MOEB_BENCH_DEBUG"):  # diagnosis: per-step predict / replay times
        print("predict ms per step:", [round(a.elapsed_time(b), 2) for k, a, b, _ in timing
                                       if k == "predict"], file=sys.stderr)
        print("replay ms per step:", [round(a.elapsed_time(b), 2) for k, a, b, _ in timing
                                      if k == "replay"], file=sys.stderr)
    lin_ms = sum(a.elapsed_time(b) for k, a, b, _ in timing if k == "predict") / args.steps
    sim_ms = sum(a.elapsed_time(b) for k, a, b, _ in timing if k == "replay") / args.steps
    n_launch = len(timing) // args.steps
    clock_info = clocks.summary()

    c = counters[0, 0].cpu().numpy()
    mc = m.MetricCounts.from_vector(vec.cpu().numpy(), E)

    # --- the same steps issued as a stream of batches: step i+1's predictor
    # (K3t) beside step i's replay and metrics (two mask buffers), the last
    # step joined before the end event. Reported beside the headline, whose
    # per-kernel times stay attributable (K3t slows from 4.0 to ~4.8 ms when
    # it shares the SMs with K1s).
    pipelined = None
    if not pipe.overlap:
        pipe2 = m.PipelinedReplay(packed, args.chunks, overlap_steps=True)
        for _ in range(max(3, args.warmup)):
            pipe2.run(pred, [cap], WARMUP_TOKENS, BUDGET, metrics=m.metrics.metric_vector(E, dev),
                      per_prompt=True)
        pipe2.join()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s3, t3 = ev(), ev()
        s3.record(stream)
        for _ in range(args.steps):
            c3 = pipe2.run(pred, [cap], WARMUP_TOKENS, BUDGET,
                           metrics=m.metrics.metric_vector(E, dev), per_prompt=True)
        pipe2.join()
        t3.record(stream)
        torch.cuda.synchronize()
        ms3 = s3.elapsed_time(t3)
        if world > 1:
            t = torch.tensor([ms3], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms3 = float(t.item())
        if world == 1:  # (with more ranks c holds the reduced counters)
            assert np.array_equal(c3[0, 0].cpu().numpy(), c), "pipelined steps changed the counters"
        pipelined = {"value": tokens_per_rank * world / (ms3 / 1000.0) * args.steps,
                     "ms_per_step": ms3 / args.steps,
                     "how": "step i+1's K3t beside step i's K1s + K7 (two mask buffers)"}
        del pipe2

    # --- end to end through the public API with host buffers ---
    # StreamingReplay: every step copies its pinned host trace rows to the
    # device (copy stream, double-buffered so step i+1's copy overlaps step
    # i's compute) and reads its counters + metrics back to pinned host
    # memory; all inside the timed region. Host batches in a compact wire
    # format decoded into masks on the device after the copy: by default each
    # row's 6 expert ids at 6 bits (--e2e-format ids6, 4.5 B/row: 297 MB per
    # step, a shift decode of 0.32 ms), or its combinatorial rank as a 27-bit
    # stream (packed-ranks, 3.375 B/row, 223 MB, a digit-search decode of
    # 0.68 ms on the SMs the predictor needs: 429 M vs 449 M trace tok/s end
    # to end), sorted id pairs in 11 bits (idpairs, 4.125 B/row, 0.43 ms
    # decode: 429 M), u32 ranks, u8 ids (6 B/row) or the 8-byte masks.
    if args.e2e_format == "packed-ranks":
        truth_host = m.masks_to_ranks(packed.truth, C2["top_k"], E, packed=True).cpu().pin_memory()
    elif args.e2e_format == "ranks":
        truth_host = m.masks_to_ranks(packed.truth, C2["top_k"], E).cpu().pin_memory()
    elif args.e2e_format == "ids":
        truth_host = m.masks_to_ids(packed.truth, C2["top_k"]).cpu().pin_memory()
    elif args.e2e_format == "ids6":
        truth_host = m.masks_to_ids6(packed.truth, C2["top_k"]).cpu().pin_memory()
    elif args.e2e_format == "idpairs":
        truth_host = m.masks_to_idpairs(packed.truth, C2["top_k"]).cpu().pin_memory()
    else:
        truth_host = packed.truth.cpu().pin_memory()
    wire = args.e2e_format if args.e2e_format in ("ids6", "idpairs") else None
    sr = m.StreamingReplay(shape, packed.row_off_host, packed.prompt_ids, dev)
    h2d = truth_host.numel() * truth_host.element_size()
    d2h = (4 + 3 * L) * 8 + (3 * E + 3) * 8 + P * 4 * 8  # counters, metrics, per-prompt

    def e2e_run(n):
        res = sr.run(pred, [cap], WARMUP_TOKENS, BUDGET, [truth_host] * n, metrics=True,
                     per_prompt=True, wire=wire)
        if world > 1:
            torch.cuda.synchronize()
            buf = torch.cat([torch.cat([c.view(-1), v]) for c, v, _ in res]).to(dev)
            dist.all_reduce(buf)
            return buf.cpu()
        return res

    # warm-up with as many batches as the timed run, so the pinned host
    # buffers the batches read back into come from the caching host allocator
    # (a cudaHostAlloc inside the timed region stalls the pipeline)
    e2e_run(max(args.steps, args.warmup))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s2, t2 = ev(), ev()
    s2.record(stream)
    res2 = e2e_run(args.steps)
    t2.record(stream)
    torch.cuda.synchronize()
    ms2 = s2.elapsed_time(t2)
    if world > 1:
        t = torch.tensor([ms2], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms2 = float(t.item())
    e2e_value = tokens_per_rank * world / (ms2 / 1000.0) * args.steps
    if os.environ.get("MOEB_E2E_DEBUG"):  # per-batch compute spans of one more e2e run
        tl = []
        s3 = ev()
        s3.record(stream)
        sr.run(pred, [cap], WARMUP_TOKENS, BUDGET, [truth_host] * args.steps, metrics=True,
               wire=wire,
               timing=tl)
        torch.cuda.synchronize()
        print("e2e batches (start ms, compute ms):",
              [(round(s3.elapsed_time(a), 2), round(a.elapsed_time(b), 2)) for a, b in tl],
              file=sys.stderr)
    if world == 1:
        assert np.array_equal(res2[-1][0].numpy().reshape(-1), counters.cpu().numpy().reshape(-1))
        assert np.array_equal(res2[-1][2].numpy(), pipe.last_per_prompt[0].cpu().numpy())

    # --- roofline of the dominant kernel (HBM-bound integer work) ---
    bytes_per_row = 16  # truth mask read + predicted mask (read by K1 / written by K3)
    # K3 runs as K3t (k_linear_tc: tensor-core column sums + top-k on packed
    # keys) unless MOEB_K3=fp64 selects the SIMT fp64 kernel
    k3_name = "k_linear_predict" if os.environ.get("MOEB_K3", "").startswith("f") else "k_linear_tc"
    dom = "k_cache_sim" if sim_ms >= lin_ms else k3_name
    dom_ms = max(sim_ms, lin_ms)
    achieved = rows * bytes_per_row / (dom_ms / 1000.0) / 1e9
    # DRAM bytes per launch from the committed `ncu --set full` capture of the
    # same kernel on the same workload (profiles/traffic.json), scaled to this
    # run's rows per launch when the chunking differs.
    traffic, limiter = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            t = json.load(open(tpath)).get(dom)
            if t:
                traffic = t["dram_bytes"] * (rows / len(pipe.bounds)) / t["rows"]
                limiter = t.get("limiter")
        except Exception:
            traffic = None

    # --- per-policy hit rates at 10 % (outside the timed region) ---
    hit = {"learned_linear": int(c[1]) / int(c[0])}
    lru_c, _, _ = m.cache_replay(packed, [(None, None, False)], [cap], WARMUP_TOKENS, BUDGET,
                                 want_per_prompt=False)
    if world > 1:
        dist.all_reduce(lru_c)
    lc = lru_c[0, 0].cpu().numpy()
    hit["lru_only"] = int(lc[1]) / int(lc[0])

    # --- parity: the reference arm's own sample (prompts 0..255) through the
    # drop-in replay_traces, against the counters the reference produced for
    # it (tests/golden/c2_sample256.npz, made by tests/golden/make_c2_golden.py)
    parity = None
    gpath = os.path.join(ROOT, "tests", "golden", "c2_sample256.npz")
    if P >= 256 and os.path.exists(gpath):
        g = np.load(gpath)
        j = [int(x) for x in g["capacities"]].index(cap)
        cfg = m.ReplayConfig(shape, m.CacheConfig(capacity_fraction=CAP_FRACTION,
                                                  prefetch_budget=BUDGET),
                             warmup_tokens=WARMUP_TOKENS)
        # every rank calls the drop-in replay_traces on the same sample (prompts
        # 0..255): with a process group it shards the prompts over the ranks
        # and all-reduces the counters (distributed.replay_sharded)
        sample = packed.select(0, 256) if rank == 0 else m.generate_packed(
            m.GeneratorConfig(256, C2["tokens"], shape, C2["hot"], C2["skew"], C2["seed"],
                              first_prompt_id=0), dev)
        rep = m.replay_traces(sample, pred, cfg)
        got = np.concatenate([[rep.measured_accesses, rep.cache_hits, rep.prediction_hits,
                               rep.uncovered_queries], rep.layer_accesses,
                              rep.layer_cache_hits, rep.layer_prediction_hits])
        want = g["counters_learned_linear"][j]
        vec_s = m.metrics.metric_vector(E, dev)
        pred.predict_masks(sample, BUDGET, WARMUP_TOKENS, metrics=vec_s)
        met_eq = bool(np.array_equal(vec_s.cpu().numpy(), g["metrics_ints"]))
        parity = {"sample": "prompts 0..255 x 363 tokens (the reference arm's sample at 16 "
                            "host cores), learned_linear + LRU 10 %",
                  "reference": {"measured_accesses": int(want[0]), "cache_hits": int(want[1]),
                                "prediction_hits": int(want[2])},
                  "ours": {"measured_accesses": int(got[0]), "cache_hits": int(got[1]),
                           "prediction_hits": int(got[2])},
                  "counters_equal": bool(np.array_equal(got, want)),
                  "per_layer_equal": bool(np.array_equal(got[4:], want[4:])),
                  "metric_counts_equal": met_eq}

    # --- the paper's transformer predictor (tcgen05 path) on a C2 slice ---
    tr_info = None
    if args.transformer_prompts > 0:
        from paper_2508_17137_b200 import transformer as TR
        Pt = min(args.transformer_prompts, P)
        tpk = packed.select(0, Pt)
        Wt = TR.TransformerWeights.random(L, E, seed=0, fp16=True, device=dev)
        tpred = m.make_predictor("transformer", shape, transformer=Wt)

        def tr_step(timing=None):
            vec_t = m.metrics.metric_vector(E, dev)
            mk = tpred.predict_masks(tpk, BUDGET, WARMUP_TOKENS, metrics=vec_t, timing=timing)
            cnt_t, _, _ = m.cache_replay(tpk, [(mk, None, False)], [cap], WARMUP_TOKENS, BUDGET,
                                         want_per_prompt=False)
            return cnt_t, vec_t

        for _ in range(2):
            tr_step()
        torch.cuda.synchronize()
        timing = {}
        ts, te = ev(), ev()
        ts.record(stream)
        nt = max(1, min(3, args.steps))
        for _ in range(nt):
            cnt_t, vec_t = tr_step(timing)
        te.record(stream)
        torch.cuda.synchronize()
        tms = ts.elapsed_time(te) / nt
        ker = {}
        for name, lst in timing.items():
            msum = sum(a.elapsed_time(b) for a, b, _ in lst) / nt
            fl = sum(f for _, _, f in lst) / nt
            ker[name] = {"ms": msum, "tflops": fl / (msum / 1e3) / 1e12}
        tdom = max((k for k in ker if ker[k]["tflops"] > 0), key=lambda k: ker[k]["ms"])
        tot_flops = sum(sum(f for _, _, f in lst) for lst in timing.values()) / nt
        ct = cnt_t[0, 0].cpu().numpy()
        mct = m.MetricCounts.from_vector(vec_t.cpu().numpy(), E)
        tr_info = {
            "workload": f"C2 slice: {Pt} prompts x {C2['tokens']} tokens (rows {tpk.rows})",
            "predictor": "transformer 4x(d512,h8,ff2048), windows 512",
            "dtype": "fp16 GEMM/attention operands, fp32 accumulation, fp16 residual stream "
                     "(fp32 LayerNorm statistics)",
            "trace_tok_per_s": Pt * C2["tokens"] / (tms / 1e3), "ms_per_step": tms,
            "tflops_achieved": tot_flops / (tms / 1e3) / 1e12, "kernels": ker,
            "roofline": {"bound": "tensor", "kernel": tdom, "achieved": ker[tdom]["tflops"],
                         "peak": bf16_sus, "unit": "TFLOP/s",
                         "frac": ker[tdom]["tflops"] / bf16_sus,
                         "peak_kind": f"{peak_kind} dense bf16/fp16 sustained"},
            "hit_rate_10pct": int(ct[1]) / int(ct[0]),
            "prediction": {"macro_f1": mct.macro_f1(), "position_accuracy": mct.position_accuracy,
                           "label_accuracy": mct.label_accuracy},
        }
        del Wt, tpred

    # --- MoE-Infinity EAM matcher at scale (BASELINE C4) on tensor cores ---
    eam_info = None
    if args.eam_sketches > 0 and rank == 0:
        from paper_2508_17137_b200 import sketches as SK
        t0 = time.perf_counter()
        lib = m.generate_packed(m.GeneratorConfig(args.eam_sketches, 32, shape, C2["hot"],
                                                  C2["skew"], 11, first_prompt_id=10**6), dev)
        coll = SK.build_eamc(lib, SK.EamcConfig(mode="recent", capacity=args.eam_sketches))
        del lib
        qtr = m.generate_packed(m.GeneratorConfig(16, 128, shape, C2["hot"], C2["skew"],
                                                  C2["seed"]), dev)
        qc = SK.token_query_counts(qtr, WARMUP_TOKENS)
        tcm = SK.TensorCoreMatcher(coll, dev)
        torch.cuda.synchronize()
        setup_s = time.perf_counter() - t0
        tcm.match_counts(qc)  # warm-up
        torch.cuda.synchronize()
        timing = {}
        e0, e1 = ev(), ev()
        e0.record(stream)
        idx_tc, _, nrr = tcm.match_counts(qc, timing)
        e1.record(stream)
        torch.cuda.synchronize()
        ms_all = e0.elapsed_time(e1)
        a, b, fl = timing["gemm_rowmax"][0]
        gms = a.elapsed_time(b)
        eam_info = {
            "workload": f"C4: {args.eam_sketches} sketches (D = {L * E}) x {qc.shape[0]} "
                        "per-token layer-0 queries of the C1 prompts",
            "queries_per_s": qc.shape[0] / (ms_all / 1e3), "ms": ms_all,
            "gemm_ms": gms,
            "roofline": {"bound": "tensor", "kernel": "k_gemm<EPI_ROWMAX> (fp16 split)",
                         "achieved": fl / (gms / 1e3) / 1e12, "peak": bf16, "unit": "TFLOP/s",
                         "frac": fl / (gms / 1e3) / 1e12 / bf16,
                         "algorithmic": "2 M S D (the fp16 hi/lo split doubles executed FLOPs)",
                         "peak_kind": f"{peak_kind} dense bf16/fp16 burst"},
            "reranked_tiles_per_query": float(nrr.float().mean().item()), "setup_s": setup_s,
        }
        del tcm, coll

    cpu_base = None
    if rank == 0 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        n_sample = max(16 * cores, 256)  # ~10 s of reference work (bounded C2 sample)
        try:
            v, dt, _ = time_reference(n_sample, cores)
            cpu_base = {"value": v, "unit": "trace tokens/s", "cores": cores, "kind": "reference",
                        "sample": f"{n_sample} x {C2['tokens']}-token C2 prompts, "
                                  f"moesim.replay_traces(jobs={cores}) learned_linear + LRU 10% "
                                  f"({dt:.1f} s)", "cpu": cpu_model()}
        except Exception as exc:
            cpu_base = {"value": None, "unit": "trace tokens/s", "cores": 0, "kind": "reference",
                        "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": "trace tokens/sec (predict+cache-sim)",
            "value": value, "unit": "trace tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "warmup_steps_run": n_w, "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64+f64",
            "data": "synthetic (reference generator, bit-identical, generated on device)",
            "config": _config(P, rows, cap, world),
            "e2e": {"value": e2e_value, "unit": "trace tokens/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "host_format": {
                        "packed-ranks": "combinatorial rank of each row's 6-expert set as a "
                                        "27-bit stream (3.375 B/row), decoded on device "
                                        "(k_ranks_to_masks_seeded)",
                        "ranks": "u32 combinatorial rank of each row's 6-expert set [rows], "
                                 "decoded on device (k_ranks_to_masks_seeded)",
                        "ids": "u8 expert ids [rows][6], decoded on device (k_ids_to_masks)",
                        "ids6": "each row's 6 ascending expert ids at 6 bits as a 36-bit "
                                "stream (4.5 B/row), decoded on device (k_ids6_to_masks)",
                        "idpairs": "each row's 6 ascending expert ids as 3 sorted pairs, a "
                                   "pair (a < b) as C(b, 2) + a in 11 bits: a 33-bit stream "
                                   "(4.125 B/row), decoded on device by table lookups "
                                   "(k_idpairs_to_masks)",
                        "masks": "int64 mask rows"}[args.e2e_format]},
            # per chunk and step: K3t (k_linear_tc_prep, k_linear_tc, k_linear_tc_refine,
            # k_linear_rows_exact, the gated fp64 k_linear_predict, k_linear_tc_finalize),
            # K1s (k_stack_replay) + K1 (k_cache_sim_warp over the prompts K1s left
            # undecided), K7 (k_metrics64)
            "gpu_launches": 9 * len(pipe.bounds) * args.steps,
            "pipeline": {"chunks": len(pipe.bounds), "streams": "predict || replay (|| H2D in e2e)",
                         "overlap_steps": pipe.overlap},
            "pipelined_steps": pipelined,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": traffic,
                         "algorithmic_bytes": f"{bytes_per_row} B/row x {rows} rows",
                         "limiter": limiter},
            "kernels_ms": {k3_name: lin_ms, "k_cache_sim": sim_ms,
                           "k_metrics64": "overlapped with k_cache_sim (low-priority stream)"},
            "hit_rate_10pct": hit,
            "prediction": {"macro_f1": mc.macro_f1(), "position_accuracy": mc.position_accuracy,
                           "label_accuracy": mc.label_accuracy},
            "parity": parity,
            "cpu_baseline": cpu_base,
            "transformer": tr_info,
            "eam_c4": eam_info,
            "clocks": clock_info,
            "setup": {"generate_s": gen_s},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    if os.environ.get("MOEB_BENCH_STACKS"):  # diagnosis: dump every thread's stack after N s
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["MOEB_BENCH_STACKS"]), exit=False)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--prompts", type=int, default=C2["prompts"])
    ap.add_argument("--e2e-format", choices=["packed-ranks", "idpairs", "ranks", "ids6", "ids",
                                             "masks"],
                    default="ids6",
                    help="host batch format of the end-to-end run: 6-bit expert ids (4.5 B/row), "
                         "combinatorial ranks as a 27-bit stream (3.4 B/row) or as u32 "
                         "(4 B/row), 11-bit sorted id pairs (4.1 B/row), u8 expert ids "
                         "(6 B/row), all decoded on device, or the 8-byte mask rows")
    ap.add_argument("--overlap-steps", action="store_true",
                    help="overlap step i+1's predictor with step i's replay")
    ap.add_argument("--chunks", type=int, default=1,
                    help="prompt chunks pipelined across the predict / replay streams")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eam-sketches", type=int, default=100000,
                    help="EAM library size for the C4 matcher leg (0: skip)")
    ap.add_argument("--transformer-prompts", type=int, default=C2["prompts"],
                    help="C2 prompts replayed with the transformer predictor (default: all of "
                         "C2; 0: skip)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:
        # --gpus N without a torchrun environment: relaunch as N ranks on this node
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={29500 + os.getpid() % 1000}", os.path.abspath(__file__)]
        os.execv(sys.executable, cmd + sys.argv[1:])
    if world and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
