import json, sys
v = None
for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep.log"):
    l = l.strip()
    if l.startswith("variant"):
        v = l.split()[1]
    elif l.startswith("{"):
        d = json.loads(l); r = d["roofline"]
        ach = r["achieved"] or 0
        print(v, round(d["value"], 1), "kernel", round(ach, 1), "frac", round(r["frac"] or 0, 3),
              "stream", round(d["config"].get("stream_2r1w_gbs") or 0, 1), "clk", d["clocks"]["sm_mhz"])
    elif "Error" in l:
        print(v, l)
