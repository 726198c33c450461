make -s -C oracle synth
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','ms_per_step','ttft_p50_ms','ttft_p90_ms')}, d['e2e']['value'], d['roofline']['frac'], d['roofline']['achieved'], d['roofline']['forward_tflops'], d['clocks'])"
