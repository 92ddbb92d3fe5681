"""Summarise a per-CTA timeline (bench.py --cta-times) including the marks.

usage: python tools/cta_marks.py gpurun_out/cta_cfg2.npz
"""
import sys

import numpy as np

z = np.load(sys.argv[1])
t0 = min(int(z[k][:, 0].min()) for k in z.files if len(z[k]))
for k in ["f3_gsort", "f3_fwd", "f3_srows_bwd2", "f3_bwd1", "f3_combine"]:
    if k not in z.files or not len(z[k]):
        continue
    a = z[k].astype(np.int64)
    st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
    print(f"{k:14s} ctas {len(a):4d} start {st.min():7.2f} end {en.max():7.2f} "
          f"dur mean {np.mean(en - st):6.2f} max {np.max(en - st):6.2f}")
    prev = a[:, 0]
    for m in range(4):
        col = a[:, 4 + m]
        ok = col > 0
        if not ok.any():
            continue
        d = (col[ok] - prev[ok]) / 1e3
        print(f"   mark{m}: from previous mean {d.mean():6.2f} p90 {np.percentile(d, 90):6.2f} max {d.max():6.2f}"
              f"  (abs mean {np.mean((col[ok] - t0) / 1e3):7.2f})")
        prev = np.where(ok, col, prev)
    d = (a[:, 1] - prev) / 1e3
    print(f"   exit : from previous mean {d.mean():6.2f} p90 {np.percentile(d, 90):6.2f} max {d.max():6.2f}")
