# Bench after stream-K + epilogue rework: default (K=40) and the K=20 window, plus the GPU suite.
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02/gputest_b.log 2>&1
echo "rc=$?" >> gpurun_out/r02/gputest_b.log
tail -2 gpurun_out/r02/gputest_b.log
timeout 900 python bench.py > gpurun_out/r02/bench_b40.json 2> gpurun_out/r02/bench_b40.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_b20.json 2> gpurun_out/r02/bench_b20.err
python - <<'PY'
import json
for f in ("gpurun_out/r02/bench_b40.json", "gpurun_out/r02/bench_b20.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["e2e"]["value"], d["roofline"]["frac"], d.get("ttft_ms"), d["clocks"], d.get("extra_configs", {}).get("c2_short_7b", {}).get("value"))
    except Exception as e:
        print(f, "ERR", e)
PY
