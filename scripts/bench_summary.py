"""Print the key numbers of a bench.py JSON line (and of a reference-arm line)."""
import json
import sys

d = json.load(open(sys.argv[1]))
oc = d.pop("other_configs", {})
print({k: d.get(k) for k in ("value", "ms_per_step", "assembly_ms", "matvec_ms", "matvecs_step_ms",
                             "pairs_evaluated_per_unique", "gpu_launches")})
r = d["roofline"]
print("roofline", {k: r.get(k) for k in ("achieved", "peak", "frac", "peak_burst", "frac_of_burst",
                                          "peak_at_kernel_clock", "frac_at_kernel_clock", "traffic")})
print("assembly alone", r.get("assembly_alone"), "| sustained-peak clocks", r["peak_clocks"])
m = d.get("roofline_matvec_multi") or {}
print("matvec single frac", d["roofline_matvec"]["frac"], "| multi", {k: m.get(k) for k in ("bound", "frac", "frac_hbm", "frac_fp64", "ms")})
print("clocks", d["clocks"])
e = d.get("e2e", {})
print("e2e", e.get("value"), e.get("s_per_step"), e.get("s_per_step_median"), "| cpu_baseline", d.get("cpu_baseline", {}).get("value"))
for c, v in oc.items():
    if "error" in v:
        print(c, v)
        continue
    print(c, "value %.3g ms %.3f asm %s roof %.3f e2e %.3g cpu %.3g clk %s" % (
        v["value"], v["ms_per_step"], v.get("assembly_ms"), v["roofline"]["frac"], v.get("e2e", {}).get("value", 0),
        v.get("cpu_baseline", {}).get("value", 0), v["clocks"]["sm_mhz"]))
    if v.get("nearfield_roofline"):
        print("   nearfield", v["nearfield_ms"], v["nearfield_roofline"]["frac"])
if len(sys.argv) > 2:
    ref = json.load(open(sys.argv[2]))
    print("reference", ref["value"], ref["ms_per_step"], ref["cpu_baseline"]["cores"], ref["cpu_baseline"]["kind"],
          "| same config", ref["config"] == d["config"], "| e2e ratio %.0f" % (e.get("value", 0) / ref["value"]),
          "| value ratio %.0f" % (d["value"] / ref["value"]))
