"""Per-source-line shared-memory wavefronts (total / ideal / excessive) from an
ncu report's source page: where the bank conflicts are.

    python tools/ncu_smem.py report.ncu-rep [top]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fpath, hdr, line, src = None, None, None, None
agg = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fpath = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        cw = hdr.index("L1 Wavefronts Shared")
        ci = hdr.index("L1 Wavefronts Shared Ideal")
        ce = hdr.index("L1 Wavefronts Shared Excessive")
        continue
    if r[0] == "Function Name" or hdr is None:
        continue
    if r[0]:  # a cuda source line row (aggregated)
        line, src = int(r[0]), r[1][:90]
        try:
            w, i, e = (float(r[c] or 0) for c in (cw, ci, ce))
        except ValueError:
            continue
        if w:
            k = (fpath, line, src)
            a = agg.setdefault(k, [0, 0, 0])
            a[0] += w; a[1] += i; a[2] += e
tot = sum(v[0] for v in agg.values()) or 1
exc = sum(v[2] for v in agg.values())
print(f"shared wavefronts {tot:.0f}, excessive {exc:.0f} ({exc / tot * 100:.1f}%)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
    print(f"{v[0]:10.0f} wf {v[1]:10.0f} ideal {v[2]:10.0f} exc  {k[0]}:{k[1]} {k[2]}")
