"""Summarise a bench JSON line: python tools/bsum.py gpurun_out/x_bench.json"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("C2", round(d["value"] / 1e9, 3), "Gpairs/s", d["ms_per_step"], "ms",
      {k: v["ms_per_step"] for k, v in d.get("kernel_breakdown", {}).items()})
for k in ("roofline", "roofline_other"):
    r = d.get(k)
    r = r[0] if isinstance(r, list) else r
    if r:
        print(" ", k, r["kernel"][:40], r["achieved"], r["unit"], "frac", r["frac"], "share", r.get("kernel_share_of_step"))
for k in d:
    if k.startswith("secondary") and isinstance(d[k], dict):
        s = d[k]
        print(k, s["workload"][:3], round(s["value"], 1), s["ms_per_step"], s.get("kernel_breakdown"),
              {a: b for a, b in (s.get("gram_tc") or {}).items() if "frac" in a})
