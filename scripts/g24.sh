make -s -C oracle synth
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for s in "256 16" "16 1" "512 1"; do timeout 300 python scripts/prof_forward.py $s; done
timeout 300 python scripts/prof_forward.py 512 1 0 qwen2.5-32b
python bench.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','ms_per_step','ttft_p50_ms','ttft_p90_ms')}, d['e2e']['value'], d['roofline']['frac'], d['roofline']['forward_tflops'], d['clocks'])"
