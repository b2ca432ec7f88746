for c in 4 2 4 2 1; do
  MOEB_K7_CTAS=$c timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --eam-sketches 0 --transformer-prompts 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ctas $c', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,1), 'M dev', round(d['e2e']['value']/1e6,1), 'M e2e', round(d['kernels_ms']['k_cache_sim'],3))"
done
