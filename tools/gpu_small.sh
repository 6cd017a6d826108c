bash tools/gpu_check.sh
for cfg in C1 C2; do timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['roofline']['phase_ms'].items()}, d['gpu_launches']//20)"; done
