make -s -C oracle synth
for i in 1 2; do python bench.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','ms_per_step','ttft_p50_ms','ttft_p90_ms')}, d['e2e']['value'], d['saturated_load'], d['roofline']['frac'], d['roofline']['t_cap'], d['roofline']['forward_tflops'], d['clocks'])"; done
