"""SASS evidence from the shipped library: per kernel, how many tcgen05 /
TMA / TMEM / legacy-MMA instructions its code holds (cuobjdump -sass of
paper_2601_11589_b200/liblaps_prefill.so). Writes profiles/<round>_sass_mnemonics.txt.
usage: sass_mnemonics.py ROUND_TAG"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2601_11589_b200" / "liblaps_prefill.so"
KEEP = re.compile(r"^(UTCHMMA|UTCBAR|UTMALDG|UTMASTG|LDTM|STTM|HMMA|UTCCP|MUFU\.EX2|SYNCS|FFMA2|FADD2|FMNMX3)")
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
counts = collections.Counter()
func = None
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        dem = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        dem = dem.replace("lp::(anonymous namespace)::", "").replace("void ", "")
        func = re.sub(r"\(.*$", "", dem)
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?P\d+\s+)?([A-Z][A-Za-z0-9_.]+)", line)
    if func and m and KEEP.match(m.group(1)):
        counts[(func, m.group(1))] += 1
lines = [f"# SASS evidence (cuobjdump -sass {LIB.relative_to(ROOT)}, built from this commit), count per kernel per mnemonic",
         "# UTCHMMA(.2CTA) = tcgen05.mma cta_group::1/2; UTCBAR = tcgen05.commit; UTMALDG.nD = TMA tensor loads; "
         "LDTM/STTM = tcgen05.ld/st; HMMA.16816 = warp mma.sync; MUFU.EX2 = hardware exp2; FFMA2 / FADD2 = packed fp32x2; FMNMX3 = three-input max; SYNCS = mbarrier ops"]
for (f, mn), n in sorted(counts.items()):
    lines.append(f"{n:4d}  {mn:32s} {f}")
path = ROOT / "profiles" / f"{tag}_sass_mnemonics.txt"
path.write_text("\n".join(lines) + "\n")
print(path)
