"""In-tree build of the native library ``liblaps_prefill.so``.

Compiles every ``csrc/*.cu`` with nvcc for sm_100a (``-gencode
arch=compute_100a,code=sm_100a -lineinfo``) and every ``csrc/host/*.cpp`` with
g++ -std=c++20 (the host engine; never -ffast-math), then
links one shared object next to this file. nvcc cross-compiles without a GPU,
so this runs in the CPU container; the .so travels to the GPU box with the
repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "native"
LIB = PKG / "liblaps_prefill.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-I", str(ROOT / "include"), "-I", str(CSRC)]
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-I", str(ROOT / "include"),
             "-I", str(CSRC), "-I", str(CSRC / "host")]


def _cuda_include() -> str:
    for cand in ("/usr/local/cuda/include",):
        if os.path.exists(os.path.join(cand, "nvtx3")):
            return cand
    return str(Path(shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc").resolve().parent.parent / "include")


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _cuda_home() -> Path:
    return Path(_nvcc()).resolve().parent.parent


def _header_digest() -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.rglob("*.h")) + list(CSRC.rglob("*.cuh")) + list(CSRC.rglob("*.hpp"))
                    + list((ROOT / "include").rglob("*.h*"))):
        h.update(p.read_bytes())
    h.update(" ".join(NVCC_FLAGS + CXX_FLAGS + ARCH).encode())
    return h.hexdigest()


def _compile(src: Path, obj: Path, force: bool) -> str:
    if not force and obj.exists() and obj.stat().st_mtime >= src.stat().st_mtime:
        return f"up-to-date {src.name}"
    obj.parent.mkdir(parents=True, exist_ok=True)
    if src.suffix == ".cu":
        cmd = [_nvcc(), *ARCH, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    else:
        cmd = [os.environ.get("CXX", "g++"), *CXX_FLAGS, "-isystem", _cuda_include(), "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return f"built {src.name}"


def build(verbose: bool = False, force: bool = False) -> Path:
    sources = sorted(CSRC.glob("*.cu")) + sorted((CSRC / "host").glob("*.cpp"))
    BUILD.mkdir(parents=True, exist_ok=True)
    stamp = BUILD / "headers.sha256"
    digest = _header_digest()
    if not stamp.exists() or stamp.read_text() != digest:
        force = True
    objs = [BUILD / (s.relative_to(CSRC).as_posix().replace("/", "__") + ".o") for s in sources]
    with cf.ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as ex:
        for msg in ex.map(lambda so: _compile(so[0], so[1], force), zip(sources, objs)):
            if verbose:
                print(msg, flush=True)
    newest = max(o.stat().st_mtime for o in objs)
    if force or not LIB.exists() or LIB.stat().st_mtime < newest:
        cuda_lib = _cuda_home() / "lib64"
        cmd = [_nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-L", str(cuda_lib),
               "-lcudart", "-Xlinker", "-rpath," + str(cuda_lib)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"linked {LIB}", flush=True)
    stamp.write_text(digest)
    build_examples(verbose)
    return LIB


EXAMPLES = ROOT / "examples"


def build_examples(verbose: bool = False) -> None:
    """Plain-C consumers of the C ABI (examples/*.c) -> build/examples/, linked
    against the in-tree liblaps_prefill.so (rpath to the package dir)."""
    out = ROOT / "build" / "examples"
    out.mkdir(parents=True, exist_ok=True)
    for src in sorted(EXAMPLES.glob("*.c")):
        exe = out / src.stem
        if exe.exists() and exe.stat().st_mtime >= max(src.stat().st_mtime, LIB.stat().st_mtime):
            continue
        cmd = [os.environ.get("CC", "gcc"), "-std=c11", "-O2", "-Wall", "-Wextra", "-I", str(ROOT / "include"),
               str(src), "-o", str(exe), "-L", str(PKG), "-llaps_prefill", "-Wl,-rpath," + str(PKG),
               "-Wl,-rpath,$ORIGIN/../../paper_2601_11589_b200"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"example build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"built {exe}", flush=True)


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
