"""A/B two builds of the native library on the bench workloads (one process
per run, so the library is loaded fresh): BASELINE config 2's window (c2) or
the headline c4 window at K steps.
usage: LP_LIB=path/to/lib.so ab_bench.py c2|c4 [STEPS] [WARMUP]"""
import argparse
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_11589_b200 import _native as N  # noqa: E402

if os.environ.get("LP_LIB"):
    N.LIB_PATH = Path(os.environ["LP_LIB"]).resolve()
import bench  # noqa: E402

which = sys.argv[1]
a = argparse.Namespace(steps=int(sys.argv[2]) if len(sys.argv) > 2 else 40,
                       warmup=int(sys.argv[3]) if len(sys.argv) > 3 else 5, gpus=1)
lib = os.environ.get("LP_LIB", "product")
if which == "c2":
    r = bench.run_c2(a)
    print(f"{lib} c2: {r['value']:.1f} req/s (e2e {r['e2e']:.1f}), {r['ms_per_step']:.3f} ms/step", flush=True)
else:
    import tempfile

    from paper_2601_11589_b200 import engine as E
    from paper_2601_11589_b200 import scenarios as S
    from paper_2601_11589_b200.instance import MODELS, PrefillInstance
    inst = PrefillInstance(MODELS["qwen2.5-32b"], device=0, max_tokens=16384, max_members=64, kv_pages=0)
    inst.capture_graphs()
    cfg = bench.scenario(1, bench.LAMBDA_PER_GPU, bench.DURATION_MS)
    work = Path(tempfile.mkdtemp(prefix="laps_ab_"))
    st = E.simulate(S.text(cfg), "", work / "replay", mode=E.REPLAY, instances=[inst], token_seed=bench.TOKEN_SEED,
                    window=(a.warmup, a.steps), stop_after_window=True)
    reqs = bench.request_equivalents(bench.window_dispatches(work / "replay" / "events.log", a.warmup, a.steps))
    inst.close()
    print(f"{lib} c4 K={a.steps}: {reqs / (st.window_device_ms / 1000.0):.2f} req/s, "
          f"{st.window_device_ms / a.steps:.3f} ms/step", flush=True)
