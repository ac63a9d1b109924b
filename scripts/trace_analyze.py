"""Critical-path view of one level's sweep from a CE_TRACE dump (development tool).

usage: CE_TRACE=6 CE_TRACE_FILE=/tmp/t6.bin python scripts/levels.py 2; python scripts/trace_analyze.py /tmp/t6.bin
Per wave: when its first task was claimed / started, when each stage (A1, A2, A3, B) of the
wave's rows started and finished (relative to the wave's start), in microseconds."""
import sys
import numpy as np

path = sys.argv[1]
raw = open(path, "rb").read()
o = 0
n, m = np.frombuffer(raw, np.int64, 2, o)
o += 16
row = np.frombuffer(raw, np.int32, n, o); o += 4 * n
part = np.frombuffer(raw, np.int32, n, o); o += 4 * n
nA1 = np.frombuffer(raw, np.int32, m, o); o += 4 * m
nA3 = np.frombuffer(raw, np.int32, m, o); o += 4 * m
wave = np.frombuffer(raw, np.int64, m, o); o += 8 * m
tr = np.frombuffer(raw, np.uint64, 4 * n, o).reshape(n, 4).astype(np.float64)
t0 = tr[:, 0].min()
claim, run, end = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, (tr[:, 2] - t0) / 1e3
a1 = nA1[row]
a3 = nA3[row]
stage = np.where(part < a1, 1, np.where(part == a1, 2, np.where(part <= a1 + a3, 3, 4)))
w = wave[row]
nw = int(w.max()) + 1
print(f"items {n}, rows {m}, waves {nw}, level time {end.max():.0f} us")
print("wave  rows | start  A1 run..end   A2 run..end   A3 run..end   B run..end   | wave len  A2 dur  B dur(mean task)")
prev_end = 0.0
lens = []
for k in list(range(0, min(nw, 6))) + list(range(nw // 2, nw // 2 + 6)):
    sel = w == k
    ws = run[sel].min()
    line = f"{k:4d} {len(np.unique(row[sel])):4d} | {ws:8.0f}"
    for st in (1, 2, 3, 4):
        ss = sel & (stage == st)
        if ss.any():
            line += f"  {run[ss].min() - ws:5.0f}..{end[ss].max() - ws:5.0f}"
        else:
            line += "        -    "
    b = sel & (stage == 4)
    a2 = sel & (stage == 2)
    line += f" | {end[sel].max() - ws:6.0f} {np.mean(end[a2] - run[a2]):6.0f} {np.mean(end[b] - run[b]) if b.any() else 0:6.0f}"
    print(line)
# average per-stage critical contributions over all waves
tot = {1: 0.0, 2: 0.0, 3: 0.0, 4: 0.0}
gap = 0.0
for k in range(nw):
    sel = w == k
    ws = run[sel].min()
    last = ws
    for st in (1, 2, 3, 4):
        ss = sel & (stage == st)
        if ss.any():
            e = end[ss].max()
            tot[st] += max(0.0, e - max(last, run[ss].min()))
            gap += max(0.0, run[ss].min() - last)
            last = max(last, e)
print("mean per wave (us): " + ", ".join(f"A{s if s < 4 else 'B'} {tot[s] / nw:.0f}" for s in (1, 2, 3)) + f", B {tot[4] / nw:.0f}, gaps {gap / nw:.0f}")
# time between consecutive waves' starts
starts = np.array([run[w == k].min() for k in range(nw)])
ends = np.array([end[w == k].max() for k in range(nw)])
print(f"mean wave-start spacing {np.mean(np.diff(starts)):.0f} us; mean (next start - this end) {np.mean(starts[1:] - ends[:-1]):.0f} us")
