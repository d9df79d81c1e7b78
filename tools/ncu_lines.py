"""Per-source-line instruction and stall shares from an ncu report (source page, cuda+sass)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
func = fpath = hdr = None
agg = collections.defaultdict(lambda: collections.defaultdict(lambda: [0, 0]))
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fpath = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        ws = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if r[0] == "" or hdr is None:
        continue
    try:
        key = (fpath, int(r[0]), r[1][:100])
        agg[func][key][0] += int(r[ie] or 0)
        agg[func][key][1] += int(r[ws] or 0)
    except ValueError:
        pass
for func, items in agg.items():
    tot = sum(v[0] for v in items.values()) or 1
    tots = sum(v[1] for v in items.values()) or 1
    print("==", func[:110], "inst", tot, "samples", tots)
    for k, v in sorted(items.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{v[0] / tot * 100:5.1f}% inst {v[1] / tots * 100:5.1f}% stall  {k[0]}:{k[1]} {k[2]}")
