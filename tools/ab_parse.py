import json, sys
tag = sys.argv[1]
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    j = json.loads(line); r = j["roofline"]
    print(tag, round(j["value"] / 1e9, 1), "Gp/s  k2", round(r["achieved"]), "GB/s frac", round(r["frac"], 3),
          "k1", round(r["k1_gbs"]), "step_frac", round(r["step_frac"], 3), "clk", j["clocks"]["sm_mhz"], j["clocks"]["reasons"])
