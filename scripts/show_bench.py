import json, sys
for f in sys.argv[1:]:
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); r = d.get("roofline") or {}
            tl = d.get("timeline_ms")
            tls = "" if not tl or not tl.get("steps") else " tl(b_done %.3f i_start %.3f i_done %.3f x_done %.3f)" % (
                tl["boundary_done"], tl["inner_start"], tl["inner_done"], tl["exchange_done"])
            print(f.split("/")[-1], "value", round(d["value"], 1), "per_gpu", round(d["config"].get("t_eff_per_gpu_gbs", 0), 1),
                  "ms", round(d["ms_per_step"], 4), "kernel", round(r.get("achieved") or 0, 1),
                  "exposed", d.get("exposed_halo") and round(d["exposed_halo"]["ms_per_step"], 4),
                  "e2e", d.get("e2e") and round(d["e2e"]["value"], 1),
                  "launches", d.get("gpu_launches"), "clk", (d.get("clocks") or {}).get("sm_mhz"), tls)
        elif "Error" in l or "error:" in l:
            print(f, l.strip()[:300])
