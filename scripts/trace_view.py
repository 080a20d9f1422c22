"""Print the per-round device timeline of gpurun_out/round_trace_slim.json."""
import json
import sys

ev = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/round_trace_slim.json"))
gpu = [e for e in ev if e["cat"] in ("kernel", "gpu_memcpy", "gpu_memset")]
starts = [i for i, e in enumerate(gpu) if "elementwise" in e["name"]]
bounds = starts + [len(gpu)]
for r in range(len(starts)):
    seg = gpu[bounds[r] + 1:bounds[r + 1]]
    if not seg:
        continue
    t0 = gpu[bounds[r]]["ts"] + gpu[bounds[r]]["dur"]
    print(f"--- round {r}")
    for e in seg:
        if e["dur"] > 5 or "Memcpy" in e["name"]:
            print(f"{e['ts'] - t0:8.1f} {e['dur']:7.1f} s{e['stream']} {e['name'][:60]}")
    print("span", max(e["ts"] + e["dur"] for e in seg) - t0)
