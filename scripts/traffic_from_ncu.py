"""Write a profiles/traffic*.json summary (the DRAM bytes bench.py reports as roofline.traffic) from an
ncu --set full report: the first launch whose name matches KERNEL.  Usage:
  python scripts/traffic_from_ncu.py REP KERNEL ALG_BYTES OUT --n 512 --dims 1,1,1 [--ranks R] [--note ...]
ALG_BYTES: algorithmic bytes per launch (per rank); --ranks: the launch covers R ranks (virtual ranks
on one GPU): the DRAM bytes are divided by R."""
import argparse, csv, io, json, subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep"); ap.add_argument("kernel"); ap.add_argument("alg", type=int); ap.add_argument("out")
ap.add_argument("--n", type=int, default=512); ap.add_argument("--dims", default="1,1,1")
ap.add_argument("--ranks", type=int, default=1); ap.add_argument("--note", default="")
a = ap.parse_args()
txt = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3, "usecond": 1,
         "nsecond": 1e-3, "msecond": 1e3}
for r in rows[2:]:
    d = dict(zip(h, r))
    if a.kernel not in d["Kernel Name"]:
        continue
    u = dict(zip(h, units))
    val = lambda k: float(d[k].replace(",", "")) * scale[u[k]]
    rd, wr = val("dram__bytes_read.sum") / a.ranks, val("dram__bytes_write.sum") / a.ranks
    out = {"kernel": d["Kernel Name"][:120], "n": a.n, "dims": [int(x) for x in a.dims.split(",")],
           "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
           "algorithmic_bytes_per_launch": a.alg, "ratio": (rd + wr) / a.alg,
           "source": f"{a.rep} (ncu --set full, first matching launch, cold replay)"
                     + (f"; per rank of a {a.ranks}-rank launch" if a.ranks > 1 else "") + (f"; {a.note}" if a.note else ""),
           "ncu_duration_us": val("gpu__time_duration.sum")}
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out))
    break
else:
    raise SystemExit(f"no launch matching {a.kernel}")
