import json, sys
for o in ["deformation", "state"]:
    p = json.load(open(f"gpurun_out/prof_{o}.json"))["profile"]
    tot = sum(v[1] for v in p.values())
    print(o, f"total {tot:.3f} ms")
    for k, v in sorted(p.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:22s} n={v[0]:4d} {v[1]:8.3f} ms  {v[2]/v[1]/1e6 if v[1] else 0:8.1f} GB/s")
