"""Turn scripts/round_profiles.sh outputs (gpurun_out/) into the committed profiles/ files and
print the summary numbers (development tool).

usage: python scripts/process_profiles.py [round tag, default r1]"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
NCU = "/usr/local/cuda/bin/ncu"


def rows(path):
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) >= len(hdr):
            yield dict(zip(hdr, r))


def ms(v, unit):
    return float(v.replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)


for src, dst in [("bench.json", "bench_cfg2"), ("bench_cfg3.json", "bench_cfg3"), ("bench_cfg4_64.json", "bench_cfg4_64cubed")]:
    if os.path.exists(os.path.join(OUT, src)):
        shutil.copy(os.path.join(OUT, src), os.path.join(PROF, f"{tag}_{dst}.json"))
        d = json.load(open(os.path.join(OUT, src)))
        print(dst, round(d["value"]), "unknowns/s; factor", round(d["factor_ms"], 1), "ms; pcg", round(d["pcg_solve_ms"], 1),
              "ms; e2e", round(d["e2e"]["value"]), "; roofline", d["roofline"]["bound"], round(d["roofline"]["frac"], 4))
shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(PROF, f"{tag}_launches_cfg2.csv"))

per = {}
for r in rows(os.path.join(OUT, "sweep_traffic.csv")):
    d = per.setdefault(int(r["ID"]), {})
    if r["Metric Name"].startswith("dram__bytes"):
        d["dram"] = d.get("dram", 0.0) + float(r["Metric Value"].replace(",", "")) * \
            {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r["Metric Unit"], 1)
    elif r["Metric Name"] == "gpu__time_duration.sum":
        d["ms"] = ms(r["Metric Value"], r["Metric Unit"])
levels = [{"level": k + 1, "dram_bytes": per[i]["dram"], "ncu_ms": per[i]["ms"]} for k, i in enumerate(sorted(per))]
traffic = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none "
           "-k regex:sweep_kernel -c 9, python scripts/levels.py 2 (cfg2 full, one factorization; scripts/round_profiles.sh)",
           "levels": levels, "total_dram_bytes": sum(x["dram_bytes"] for x in levels),
           "total_ncu_ms": sum(x["ncu_ms"] for x in levels)}
json.dump(traffic, open(os.path.join(PROF, f"{tag}_sweep_traffic_cfg2.json"), "w"), indent=1)
print("sweep DRAM per level (GB, ncu ms):", [(x["level"], round(x["dram_bytes"] / 1e9, 1), round(x["ncu_ms"], 1)) for x in levels])
print("sweep DRAM total GB", round(traffic["total_dram_bytes"] / 1e9, 1))

agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows(os.path.join(OUT, "launches.csv")):
    k = r["Kernel Name"].split("(")[0].replace("void ", "")[:70]
    agg[k][0] += 1
    agg[k][1] += ms(r["Metric Value"], r["Metric Unit"])
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:8]:
    print(f"  {100 * v[1] / tot:6.2f}%  {v[0]:5d}  {k}")

rep = os.path.join(OUT, "sweep_L6.ncu-rep")
if os.path.exists(rep):
    with open(os.path.join(PROF, f"{tag}_sweep_L6_ncu_details.csv"), "w") as f:
        subprocess.run([NCU, "-i", rep, "--page", "details", "--csv"], stdout=f, stderr=subprocess.DEVNULL, check=False)
    raw = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
    rr = list(csv.reader(raw))
    d = {rr[0][i]: (rr[2][i], rr[1][i]) for i in range(len(rr[0]))}
    st = {k: float(d[k][0].replace(",", "")) for k in d
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and d[k][0] not in ("", "n/a")}
    s = sum(st.values())
    print("L6 stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / s:.1f}%"
                                  for k, v in sorted(st.items(), key=lambda t: -t[1])[:5]))
    for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
              "sm__throughput.avg.pct_of_peak_sustained_elapsed"):
        if k in d:
            print(" ", k, d[k])
