"""Per-source-line instruction and stall-sample shares of one kernel from an
ncu report (--import-source on, -lineinfo builds), for finding where a
kernel's issue slots go:  python tools/ncu_lines.py report.ncu-rep [kernel-regex] [top]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kre = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fn, hdr, path = None, None, ""
by = collections.defaultdict(collections.Counter)
st = collections.defaultdict(collections.Counter)
src = {}
cur = None
for r in rows:
    if len(r) >= 2 and r[0] == "Function Name":
        fn = r[1]
        continue
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < len(hdr) // 2:
        continue
    if r[0]:
        try:
            cur = (path, int(r[0]))
        except ValueError:
            continue
        src[cur] = r[1].strip()[:90]
        continue
    try:
        v = int(r[hdr.index("Instructions Executed")])
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    by[fn][cur] += v
    st[fn][cur] += s
for f in by:
    if kre and not kre.search(f):
        continue
    tot, tst = sum(by[f].values()), max(1, sum(st[f].values()))
    print(f"== {f}: {tot} warp instructions, {tst} stall samples")
    for ln, v in sorted(by[f].items(), key=lambda x: -x[1])[:top]:
        print(f"{ln[0][:14]:>14}:{ln[1]:<5d} {v / tot * 100:5.1f}% inst {st[f][ln] / tst * 100:5.1f}% stall  {src.get(ln, '')}")
