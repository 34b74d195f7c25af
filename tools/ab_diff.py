"""Scratch: where do two result dumps of tools/ab_batch.py differ?  python tools/ab_diff.py a.npz b.npz"""
import sys
import numpy as np
a, b = dict(np.load(sys.argv[1])), dict(np.load(sys.argv[2]))
for key in ("y", "z", "lam"):
    d = np.abs(a[key] - b[key])
    bad = d > 0
    cols = np.nonzero(bad.any(axis=0))[0]
    rows = np.nonzero(bad.any(axis=1))[0]
    print(f"{key}: shape {d.shape} differing entries {int(bad.sum())} max {d.max():.3e}; columns {len(cols)}: {cols[:40].tolist()}"
          f"{' ...' if len(cols) > 40 else ''}; rows {len(rows)}: min {rows.min() if len(rows) else -1} max {rows.max() if len(rows) else -1}")
    for c in cols[:3]:
        r = np.nonzero(bad[:, c])[0]
        print(f"   column {c}: {len(r)} rows differ: {r.tolist()[:200]}  |d| {d[r[:4], c]}")
