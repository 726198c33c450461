make -s -C oracle synth
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python scripts/gemm_plans2.py qwen2.5-7b 4096:2800 2048:1500 1024:700 512:300 256:190 16:16 2>&1 | grep t_cap
for s in "256 16" "128 16" "64 16" "16 1"; do timeout 300 python scripts/prof_forward.py $s; done 2>&1 | grep shape
python bench.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','ms_per_step','ttft_p50_ms','ttft_p90_ms')}, d['e2e']['value'], d['roofline']['frac'], d['roofline']['forward_tflops'], d['clocks'])"
