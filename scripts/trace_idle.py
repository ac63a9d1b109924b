"""Where the SM time of one level's sweep goes, from a CE_TRACE dump (development tool).

usage: CE_TRACE=8 CE_TRACE_FILE=/tmp/t8.bin python scripts/ab_factor.py 3 reference 0; python scripts/trace_idle.py /tmp/t8.bin
Per stage: number of items, SM-seconds running (end - run) and parked (run - claim: the CTA holds
the ticket and polls its dependencies).  Then per wave (means): span, the parked time by stage."""
import sys
import numpy as np

path = sys.argv[1]
grid = int(sys.argv[2]) if len(sys.argv) > 2 else 148
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
# stage: 0 leaf (first tree level is unknown here: leaves = the row's first tickets), 1 other A1, 2 A2, 3 A3, 4 B
stage = np.where(part < a1, 1, np.where(part == a1, 2, np.where(part <= a1 + a3, 3, 4)))
total = end.max()
print(f"items {n}, rows {m}, waves {int(wave.max()) + 1}, level time {total / 1e3:.1f} ms, grid {grid}: {grid * total / 1e6:.1f} SM-s")
names = {1: "A1", 2: "A2", 3: "A3", 4: "B"}
busy_all = 0.0
for st in (1, 2, 3, 4):
    s = stage == st
    if not s.any():
        continue
    busy = (end[s] - run[s]).sum() / 1e6
    parked = (run[s] - claim[s]).sum() / 1e6
    busy_all += busy + parked
    print(f"  {names[st]:2s}: {int(s.sum()):8d} items, running {busy:7.2f} SM-s (mean {np.mean(end[s] - run[s]):7.1f} us), parked {parked:7.2f} SM-s "
          f"(mean {np.mean(run[s] - claim[s]):6.1f} us, p99 {np.percentile(run[s] - claim[s], 99):7.1f} us)")
print(f"  unaccounted (ticket fetch, kernel tail): {grid * total / 1e6 - busy_all:.2f} SM-s")
# ticket-order position of the parked time: which tickets hold CTAs longest
order = np.argsort(claim, kind="stable")
w = wave[row]
nw = int(w.max()) + 1
# per wave: span between consecutive wave A2 ends
a2end = np.zeros(nw)
for k in range(nw):
    s = (w == k) & (stage == 2)
    a2end[k] = end[s].max() if s.any() else 0
print(f"mean spacing of consecutive waves' A2 ends: {np.mean(np.diff(a2end)):.0f} us")
# parked time of B items split by whether the item was claimed before its row's last strip ended
print("wave | A1: first claim, first run, last end | A2: claim run end | A3: first claim, first run, last end | B: first claim, first run, median end, last end   (us, relative to the previous wave's A2 end)")
for k in list(range(nw // 2, min(nw, nw // 2 + 8))):
    sel = w == k
    ref = a2end[k - 1] if k > 0 else 0.0
    line = f"{k:5d} |"
    for st in (1, 2, 3, 4):
        s = sel & (stage == st)
        if not s.any():
            line += "      -      |"
            continue
        if st == 4:
            line += f" {claim[s].min() - ref:6.0f} {run[s].min() - ref:6.0f} {np.median(end[s]) - ref:6.0f} {end[s].max() - ref:6.0f} |"
        else:
            line += f" {claim[s].min() - ref:6.0f} {run[s].min() - ref:6.0f} {end[s].max() - ref:6.0f} |"
    print(line)
