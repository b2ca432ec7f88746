mkdir -p gpurun_out
for lib in base emu1 emu2 emu3 base emu2 emu1 emu3; do
  if [ $lib = base ]; then L=""; else L="$PWD/build_alt/libmoeb_$lib.so"; fi
  MOEB_LIB=$L timeout 300 python tools/bench_transformer.py --prompts 700 --steps 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms'],1), d['stages_ms'].get('attention'), round(d['trace_tok_per_s']))"
done 2>&1 | tee gpurun_out/ab_attn.log
for lib in emu1 emu2 emu3; do MOEB_LIB=$PWD/build_alt/libmoeb_$lib.so timeout 300 python -m pytest -q -x tests/test_gpu_transformer.py 2>&1 | tail -1; done
