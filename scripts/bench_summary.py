"""Print the essentials of a bench.py JSON line (ours or the reference arm)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
if d.get("impl") == "reference":
    print("reference:", round(d["value"], 2), d["unit"], "steps", d["steps"], "ms/step", round(d["ms_per_step"]), d["prep"])
    sys.exit()
print("value", round(d["value"]), "e2e", round(d["e2e"]["value"]), "ms/step", round(d["ms_per_step"], 3),
      "gteps", round(d["gteps"], 1), "launches", d["gpu_launches"])
print("clocks", d["clocks"])
print("parity", d["parity"])
r = d["roofline"]
print("roofline", r["kernel"], round(r["achieved"]), "GB/s frac", round(r["frac"], 3), "traffic", r["traffic"])
cb = d.get("cpu_baseline") or {}
print("cpu_baseline", round(cb.get("value", 0), 2), cb.get("cores"), cb.get("kind"))
for g in d["groups"]:
    print(" group", g["ks"], g["kernel"], "lanes", g["lanes"], round(g["ms_per_call"], 3), "ms frac", round(g["frac_of_peak"], 3),
          "GTEPS", round(g["gteps"], 1))
for c, v in (d.get("extra_configs") or {}).items():
    if c == "cfg5":
        print(c, {k: (round(x["ms"], 2), round(x["queries_per_s"]), x["engine"], x["lanes_per_batch"], round(x["gteps"], 1))
                  for k, x in v["k"].items()})
    else:
        cb = v.get("cpu_baseline", {})
        print(c, round(v["value"]), "e2e", round(v["e2e"]["value"]), "gteps", round(v["gteps"], 1),
              [(g["ks"], round(g["ms_per_call"], 3), round(g["frac_of_peak"], 3)) for g in v["groups"]],
              "cpu", round(cb.get("value", 0)), "parity", v["parity"]["checked"], v["parity"]["mismatches"])
