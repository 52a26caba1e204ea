"""bench.py's JSON contract on CPU: the --impl reference arm (the CPU oracle)
prints one line with the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--n", "48", "--steps", "2",
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=300,
                       env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_committed_traffic_summaries_match_the_algorithmic_bytes():
    """The ncu traffic files bench.py reads carry the algorithmic bytes of DESIGN.md's per-cell figures
    (heat 24 B, binary32 heat 12 B per updated cell of the 510^3 interior; the fused acoustic sweep 64 B
    per cell of 512^3) and a DRAM traffic within a few percent of them (no wasted re-reads).  The fused
    heat kernel (per rank of a two-rank launch, x data plane included) may exceed it by its short
    z chunks' plane re-reads and the staging traffic: < 5 %."""
    want = {"traffic.json": (24 * 510 ** 3, 1.03, [1, 1, 1]), "traffic_f32.json": (12 * 510 ** 3, 1.03, [1, 1, 1]),
            "traffic_acoustic.json": (64 * 512 ** 3, 1.03, [1, 1, 1]),
            "traffic_fused.json": (24 * 510 ** 3, 1.05, [2, 1, 1])}
    for name, (alg, tol, dims) in want.items():
        d = json.load(open(os.path.join(ROOT, "profiles", name)))
        assert d["n"] == 512 and d["dims"] == dims, name
        assert d["algorithmic_bytes_per_launch"] == alg, name
        assert abs(d["dram_read_bytes"] + d["dram_write_bytes"] - d["dram_bytes_per_launch"]) < 1e3, name
        assert 1.0 <= d["dram_bytes_per_launch"] / alg < tol, name


