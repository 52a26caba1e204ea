"""One-line summary of an acoustic bench log: ms/step, V-kernel ms and fraction."""
import json
import sys

lines = [x for x in open(sys.argv[1]) if x.startswith("{")]
if not lines:
    print("no json")
else:
    d = json.loads(lines[-1])
    r = d.get("roofline") or {}
    print(f"ms_per_step {d.get('ms_per_step'):.4f} v_ms {r.get('avg_launch_ms', 0):.4f} v_frac {r.get('frac', 0):.4f}")
