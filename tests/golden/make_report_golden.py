"""Golden CSV reports from the REFERENCE (moesim.engine report emitters) for a
small replay and sweep; the counters are stored next to the bytes so the CPU
test can rebuild the same SimReports.   python tests/golden/make_report_golden.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    import moesim
    from moesim import engine
    shape = moesim.ModelShape(4, 8, 2)
    traces = moesim.generate_synthetic(moesim.GeneratorConfig(5, 12, shape, 3, 0.8, 3))
    cfg = moesim.ReplayConfig(shape, moesim.CacheConfig(capacity_fraction=0.25,
                                                        prefetch_budget=2), warmup_tokens=2)
    rep = moesim.replay_traces(traces, moesim.make_predictor("oracle", shape, traces=traces), cfg)
    pts = moesim.sweep(traces, lambda: moesim.make_predictor("lru_only", shape), "lru_only",
                       [0.1, 0.25, 0.5], shape, 2, 2)

    def repvec(r):
        return dict(v=[r.measured_accesses, r.cache_hits, r.prediction_opportunities,
                       r.prediction_hits, r.uncovered_queries],
                    la=r.layer_accesses.tolist(), lc=r.layer_cache_hits.tolist(),
                    lp=r.layer_prediction_hits.tolist(),
                    pp={str(k): [c.measured_accesses, c.cache_hits, c.prediction_opportunities,
                                 c.prediction_hits] for k, c in r.per_prompt.items()})
    out = {"shape": [4, 8, 2], "report": repvec(rep),
           "points": [dict(f=p.capacity_fraction, kind=p.predictor_kind, report=repvec(p.report))
                      for p in pts],
           "summary": engine.report_summary_csv(rep, "oracle", 8).decode(),
           "layers": engine.report_layers_csv(rep).decode(),
           "prompts": engine.report_prompts_csv(rep).decode(),
           "sweep": engine.sweep_csv(pts).decode(),
           "sweep_layers": engine.sweep_layers_csv(pts).decode()}
    json.dump(out, open(os.path.join(HERE, "report_csv.json"), "w"))


if __name__ == "__main__":
    main()
