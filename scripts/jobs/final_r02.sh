# Round-2 final measurement pass: GPU suite (incl. full depth), smoke, bench K=40 (default) and K=20, launch list.
mkdir -p gpurun_out/r02
export LP_PARITY_OUT=gpurun_out/r02/full_depth_parity_final.jsonl
rm -f $LP_PARITY_OUT
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02/gputest_final.log 2>&1
echo "rc=$?" >> gpurun_out/r02/gputest_final.log
tail -2 gpurun_out/r02/gputest_final.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke_final.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02/smoke_final.log
tail -2 gpurun_out/r02/smoke_final.log
LP_BENCH_OUT=gpurun_out/r02/bench_final_run timeout 900 python bench.py > gpurun_out/r02/bench_final40.json 2> gpurun_out/r02/bench_final40.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_final20.json 2> gpurun_out/r02/bench_final20.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02/bench_final_ref.json 2> gpurun_out/r02/bench_final_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02/launches_final.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r02/bench_ncu.log 2>&1
python scripts/summarize_ncu.py gpurun_out/r02/launches_final.csv > gpurun_out/r02/launches_final_summary.txt 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/r02/bench_final40.json", "gpurun_out/r02/bench_final20.json", "gpurun_out/r02/bench_final_ref.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("value"), d.get("e2e", {}).get("value"), d.get("roofline", {}).get("frac"), d.get("clocks"))
    except Exception as e:
        print(f, "ERR", e)
PY
head -12 gpurun_out/r02/launches_final_summary.txt
