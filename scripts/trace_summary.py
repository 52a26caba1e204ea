"""Summary of a fused_trace2.py capture: per rank, extra (sender) blocks' end times vs the tiles' end,
and the mean duration of x-face / other tiles.  Usage: python scripts/trace_summary.py DIR NEXTRA"""
import sys
import numpy as np

d, nx = sys.argv[1], int(sys.argv[2])
for r in (0, 1):
    for sk in (0, 1):
        a = np.load(f"{d}/trace2_r{r}_{sk}.npz")["a"]
        t0 = a[:, 0].min()
        s, e = (a[:, 0] - t0) / 1e3, (a[:, 3] - t0) / 1e3
        info = a[nx:, 2]
        tx = info & 255
        dur = e[nx:] - s[nx:]
        print(f"rank {r} skip {sk}: span {e.max():.1f} tiles end {e[nx:].max():.1f} "
              f"extra end {np.round(np.sort(e[:nx])[-4:], 1).tolist()} "
              f"x0 {dur[tx == 0].mean():.1f} xN {dur[tx == tx.max()].mean():.1f} "
              f"mid {dur[(tx > 0) & (tx < tx.max())].mean():.1f}")
for r in (0, 1):
    a = np.load(f"{d}/trace2_r{r}_0.npz")["a"]
    t0 = a[:, 0].min()
    x = (a[:nx] - t0) / 1e3
    act = x[:, 3] > 2
    print(f"rank {r} senders (last chunk): waited-until / copied-at / end", 
          np.round(x[act][:, [1, 2, 3]], 1).tolist())
