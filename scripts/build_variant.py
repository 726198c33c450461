"""Build a variant of the native library with one source recompiled under
extra nvcc flags (A/B experiments; the product build is untouched).
usage: build_variant.py SOURCE.cu OUT.so [-DNAME=VALUE ...]"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_11589_b200 import build as B  # noqa: E402

src = B.CSRC / sys.argv[1]
out = Path(sys.argv[2]).resolve()
flags = sys.argv[3:]
B.build()
out.parent.mkdir(parents=True, exist_ok=True)
obj = out.with_suffix(".o")
subprocess.run([B._nvcc(), *B.ARCH, *B.NVCC_FLAGS, *flags, "-c", str(src), "-o", str(obj)], check=True)
live = [o for o in sorted(B.BUILD.glob("*.o")) if (B.CSRC / o.name[:-2].replace("__", "/")).exists()]
objs = [o for o in live if o.name != src.name + ".o"] + [obj]
cuda_lib = B._cuda_home() / "lib64"
subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", str(out), *map(str, objs), "-L", str(cuda_lib), "-lcudart",
                "-Xlinker", "-rpath," + str(cuda_lib)], check=True)
print("built", out)
