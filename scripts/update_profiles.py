"""Copy a full GPU measurement pass (gpurun_out/) into profiles/ (r01_*) and
rewrite the generated sections of profiles/r01_summary.md: bench table, bucket
tables, ncu per-forward table, per-config table. Run after the pass in
.gpujobs-style: bench.py, ncu launch list, dominant-kernel ncu capture,
bucket_roofline.py (7B h0 / h1024, 32B), run_configs.py, ncu_forward.py."""
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
G, P = ROOT / "gpurun_out", ROOT / "profiles"


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    import csv
    rows = list(csv.reader(out.splitlines()))
    h, v = rows[0], rows[2]
    return {n: v[i] for i, n in enumerate(h)}


def bucket_table(fn, title):
    d = json.load(open(fn))
    bs = [b for b in d["buckets"] if b["kind"] == "graph"]
    Ls = sorted({b["l_pad"] for b in bs})
    Ds = sorted({b["depth"] for b in bs})
    out = [f"**{title}** — fraction of the forward's roofline floor (`h` HBM-bound, `t` tensor-bound)\n",
           "| depth \\ l_pad | " + " | ".join(map(str, Ls)) + " |", "|" + "---|" * (len(Ls) + 1)]
    for dp in Ds:
        row = []
        for lp in Ls:
            b = [x for x in bs if x["l_pad"] == lp and x["depth"] == dp]
            row.append(f"{b[0]['frac_roofline']:.2f}{b[0]['bound'][0]}" if b else "")
        out.append(f"| {dp} | " + " | ".join(row) + " |")
    ls = [b for b in d["buckets"] if b["kind"] == "long"]
    if ls:
        out.append("\nLong-prefill 512-token chunks (chunk graphs, tcgen05 attention): " + "; ".join(
            f"H={b['H']}: {b['ms']:.2f} ms, {b['tflops']:.0f} TF/s = {b['frac_tensor_sustained']:.2f} of sustained bf16"
            for b in ls))
    return "\n".join(out) + "\n"


def main():
    shutil.copy(G / "launches.csv", P / "r01_launches_bench_quick.csv")
    (P / "r01_launches_bench_quick_summary.txt").write_text(
        subprocess.run([sys.executable, str(ROOT / "scripts" / "summarize_ncu.py"), str(G / "launches.csv")],
                       capture_output=True, text=True).stdout)
    for src, dst in (("buckets_qwen2.5-7b_h0.json", "r01_buckets_7b_h0.json"),
                     ("buckets_qwen2.5-7b_h1024.json", "r01_buckets_7b_h1024.json"),
                     ("buckets_qwen2.5-32b_h0.json", "r01_buckets_32b_h0.json"), ("configs.json", "r01_configs.json")):
        shutil.copy(G / src, P / dst)
    bench = json.loads((G / "bench.log").read_text().strip().splitlines()[-1])
    (P / "r01_bench.json").write_text(json.dumps(bench, indent=1))
    raw = ncu_raw(G / "dom_full.ncu-rep")
    rd, wr = float(raw["dram__bytes_read.sum"]) * 1e6, float(raw["dram__bytes_write.sum"]) * 1e6
    dom = json.loads((P / "r01_dominant_kernel.json").read_text())
    dom["captures"] = [{"t_cap": 4096, "n_live": 2846, "gpu_time_us": float(raw["gpu__time_duration.sum"]),
                        "sm_clock_ghz": float(raw["sm__cycles_elapsed.avg.per_second"]),
                        "dram_bytes_read": int(rd), "dram_bytes_write": int(wr), "dram_bytes_per_launch": int(rd + wr),
                        "algorithmic_bytes": 2 * 18944 * 3584 * 2 + 2846 * 3584 * 2 + 2846 * 18944 * 2,
                        "tensor_pipe_pct_elapsed": float(raw["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]),
                        "note": "bench.py default run: most common step capacity 4096, median live tokens 2846"}]
    (P / "r01_dominant_kernel.json").write_text(json.dumps(dom, indent=1))
    tags = ["7b_16x1", "7b_16x1_h1024", "7b_64x4_h1024", "7b_256x1", "7b_chunk512_h1536", "7b_256x16", "32b_16x1",
            "32b_chunk512_h1536", "7b_8x64_h4000", "7b_16x16_h4000"]
    nf = json.loads((P / "r01_ncu_forwards.json").read_text())
    nf["forwards"] = {t: json.load(open(G / f"ncu_fwd_{t}.json")) for t in tags}
    (P / "r01_ncu_forwards.json").write_text(json.dumps(nf, indent=1))
    names = {"7b_16x1": "7B 16x1, H=0", "7b_16x1_h1024": "7B 16x1, H=1024", "7b_64x4_h1024": "7B 64x4, H=1024",
             "7b_256x1": "7B 256x1, H=0", "7b_chunk512_h1536": "7B 512-token chunk, H=1536",
             "7b_256x16": "7B 256x16, H=0", "32b_16x1": "32B 16x1, H=0", "32b_chunk512_h1536": "32B 512-token chunk, H=1536",
             "7b_8x64_h4000": "7B 8x64, H=4000", "7b_16x16_h4000": "7B 16x16, H=4000"}
    ncu_rows = []
    for t in tags:
        d = nf["forwards"][t]
        c = d["classes"]
        g, a = c["gemm"], c.get("attention", {"share": 0, "tensor_pct_time_weighted": 0})
        ncu_rows.append(f"| {names[t]} | {d['time_us'] / 1e3:.2f} ms | {d['dram_gbs']:.0f} | {g['share'] * 100:.0f} % / "
                        f"{g['gbs']:.0f} / {g['tensor_pct_time_weighted']:.0f} % | {a['share'] * 100:.0f} % / "
                        f"{a['tensor_pct_time_weighted']:.0f} % |")
    tables = (bucket_table(P / "r01_buckets_7b_h0.json", "Qwen2.5-7B, H=0") + "\n" +
              bucket_table(P / "r01_buckets_7b_h1024.json", "Qwen2.5-7B re-prefill, H=1024 per member") + "\n" +
              bucket_table(P / "r01_buckets_32b_h0.json", "Qwen2.5-32B, H=0") + "\n")
    s = (P / "r01_summary.md").read_text()
    # Generated bucket tables end where the hand-written KV-dominated section starts.
    i, j = s.index("**Qwen2.5-7B, H=0**"), s.index("**Qwen2.5-7B, KV-dominated re-prefill")
    s = s[:i] + tables + "\n" + s[j:]
    i = s.index("| 7B 16x1, H=0 |")
    j = s.index("\n\n", i)
    s = s[:i] + "\n".join(ncu_rows) + s[j:]
    (P / "r01_summary.md").write_text(s)
    cf = json.load(open(P / "r01_configs.json"))
    print("bench", bench["value"], bench["e2e"]["value"], bench["ttft_p50_ms"], bench["ttft_p90_ms"],
          bench["roofline"]["achieved"], bench["roofline"]["frac"], bench["roofline"]["forward_tflops"],
          bench["gpu_launches"], bench["clocks"])
    print("dominant", dom["captures"][0])
    for k, v in cf.items():
        print(k, v["frac_roofline"], round(v["gpu_req_per_s"], 1), v["live"])


if __name__ == "__main__":
    main()
