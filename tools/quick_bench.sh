#!/bin/bash
# GPU box: K1/K3 parity tests + the headline bench without the side legs.
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_streaming.py -q -x 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --eam-sketches 0 --transformer-prompts 0 "$@" 2>&1 | tail -1 | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', round(d['ms_per_step'],3), 'Mtok/s', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), d['kernels_ms'], d['hit_rate_10pct'])"
