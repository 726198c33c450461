"""Ordered-token overlap of our host sources against the reference's
(comments stripped, identifiers kept): difflib matching blocks / len(ours)
and / len(theirs). A self-check for "written, not copied" (reads
/root/reference only when it exists; not used by tests or the product)."""
import difflib
import re
import sys
from pathlib import Path

TOK = re.compile(r"[A-Za-z_]\w*|\d+\.?\d*|\S")


def tokens(path):
    s = Path(path).read_text()
    s = re.sub(r"//[^\n]*", " ", s)
    s = re.sub(r"/\*.*?\*/", " ", s, flags=re.S)
    s = re.sub(r'"(\\.|[^"\\])*"', '"S"', s)
    return TOK.findall(s)


def overlap(a, b):
    sm = difflib.SequenceMatcher(None, a, b, autojunk=False)
    m = sum(bl.size for bl in sm.get_matching_blocks() if bl.size >= 8)
    return m / max(1, len(a)), m / max(1, len(b))


ref = sorted(Path("/root/reference/proj/src").glob("*.cpp"))
ours = sys.argv[1:] or sorted(str(p) for p in Path("paper_2601_11589_b200/csrc/host").glob("*.cpp"))
for o in ours:
    ta = tokens(o)
    best = max(((overlap(ta, tokens(r)), r.name) for r in ref), key=lambda x: x[0][0])
    print(f"{Path(o).name:20s} vs {best[1]:16s} ours {best[0][0]:.2f} theirs {best[0][1]:.2f}")


def show(ours_path, ref_path, min_size=8):
    a, b = tokens(ours_path), tokens(ref_path)
    sm = difflib.SequenceMatcher(None, a, b, autojunk=False)
    for bl in sm.get_matching_blocks():
        if bl.size >= min_size:
            print(bl.size, " ".join(a[bl.a:bl.a + bl.size]))
