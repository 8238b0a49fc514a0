"""Reads an SSSVD_GEMM_DUMP file (one "start_ns end_ns flops" line per DMMA GEMM launch of a
shifted-solve pass, from the %globaltimer stamps) and reports, for the last pass in the file: the
GEMM-busy time (union of the launch intervals), the gaps with no GEMM running, the flops and
busy-time share per launch size class, and the aggregate rate in the time segments where only
launches of the largest class are active (the trailing updates running without small-GEMM company).
    python tools/gemm_timeline.py dump.txt"""
import sys

import numpy as np

passes, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = []
        passes.append(cur)
    elif cur is not None:
        a, b, f = line.split()
        cur.append((int(a), int(b), float(f)))
p = np.array(passes[-1], dtype=np.float64)
st, en, fl = p[:, 0], p[:, 1], p[:, 2]
t0, t1 = st.min(), en.max()
print(f"launches {len(p)}, span {(t1 - t0) * 1e-9:.3f} s, flops {fl.sum():.3e}")
# sweep line over all interval endpoints
ev = np.concatenate([np.stack([st, np.ones_like(st), np.arange(len(p))], 1), np.stack([en, -np.ones_like(en), np.arange(len(p))], 1)])
ev = ev[np.lexsort((-ev[:, 1], ev[:, 0]))]
edges = [1e9, 1e10, 1e11, 1e12]
cls = np.digitize(fl, edges)   # 0: < 1e9 ... 4: >= 1e12
names = ["<1e9", "1e9-1e10", "1e10-1e11", "1e11-1e12", ">=1e12"]
active = np.zeros(5, dtype=int)
busy = 0.0
only_big = 0.0
seg_by_top = np.zeros(5)
prev = ev[0, 0]
for t, d, i in ev:
    dt = t - prev
    if dt > 0 and active.sum() > 0:
        busy += dt
        top = max(k for k in range(5) if active[k] > 0)
        low = min(k for k in range(5) if active[k] > 0)
        seg_by_top[top] += dt
        if low == top == cls.max():
            only_big += dt
    prev = t
    active[cls[int(i)]] += int(d)
print(f"GEMM busy {busy * 1e-9:.3f} s ({100 * busy / (t1 - t0):.1f} % of the span), aggregate {fl.sum() / (busy * 1e-9) / 1e12:.2f} TF/s")
for k in range(5):
    m = cls == k
    if m.any():
        dur = (en[m] - st[m])
        print(f"  class {names[k]:>10}: {m.sum():6d} launches, {100 * fl[m].sum() / fl.sum():5.1f} % of the flops, "
              f"mean duration {dur.mean() * 1e-3:9.1f} us, busy time with this as the largest active class {seg_by_top[k] * 1e-9:.3f} s")
print(f"time with only largest-class launches active: {only_big * 1e-9:.3f} s")
