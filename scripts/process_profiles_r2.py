"""File scripts/round2_profiles.sh outputs (gpurun_out/) as profiles/r2_* and print the numbers
(development tool)."""
import collections
import csv
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
NCU = "/usr/local/cuda/bin/ncu"


def rows(path):
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) >= len(hdr):
            yield dict(zip(hdr, r))


def to_ms(v, unit):
    return float(v.replace(",", "")) * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
                                        "msecond": 1.0, "s": 1e3, "second": 1e3}.get(unit, 1e-6)


def to_bytes(v, unit):
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


if os.path.exists(os.path.join(OUT, "bench.json")):
    shutil.copy(os.path.join(OUT, "bench.json"), os.path.join(PROF, "r2_bench_cfg3.json"))
    d = json.load(open(os.path.join(OUT, "bench.json")))
    print("bench", round(d["value"]), "unknowns/s; factor", round(d["factor_ms"], 1), "ms; pcg", round(d["pcg_solve_ms"], 1),
          "; e2e", d["e2e"]["value"], "; sweep frac", round(d["roofline"]["frac"], 4), "; apply frac",
          round(d["roofline_apply"]["frac"], 4))

if os.path.exists(os.path.join(OUT, "launches_cfg3.csv")):
    shutil.copy(os.path.join(OUT, "launches_cfg3.csv"), os.path.join(PROF, "r2_launches_cfg3.csv"))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows(os.path.join(OUT, "launches_cfg3.csv")):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            k = r["Kernel Name"].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").split("(")[0].split("<")[0][-60:]
            agg[k][0] += 1
            agg[k][1] += to_ms(r["Metric Value"], r["Metric Unit"])
    tot = sum(v[1] for v in agg.values())
    summ = [{"kernel": k, "launches": v[0], "ms": round(v[1], 2), "share": round(v[1] / tot, 4)}
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    json.dump({"source": "ncu --metrics gpu__time_duration.sum --clock-control none, python scripts/ab_factor.py 3 "
               "reference 1 (2 factorizations + PCG of cfg3)", "total_ms": tot, "kernels": summ},
              open(os.path.join(PROF, "r2_launches_cfg3_summary.json"), "w"), indent=1)
    for x in summ[:12]:
        print(x)

if os.path.exists(os.path.join(OUT, "sweep_traffic_cfg3.csv")):
    per = {}
    for r in rows(os.path.join(OUT, "sweep_traffic_cfg3.csv")):
        d = per.setdefault(int(r["ID"]), {})
        if r["Metric Name"].startswith("dram__bytes"):
            d["dram"] = d.get("dram", 0.0) + to_bytes(r["Metric Value"], r["Metric Unit"])
        elif r["Metric Name"] == "gpu__time_duration.sum":
            d["ms"] = to_ms(r["Metric Value"], r["Metric Unit"])
    levels = [{"level": k + 1, "dram_bytes": per[i]["dram"], "ncu_ms": per[i]["ms"]} for k, i in enumerate(sorted(per))]
    tr = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control "
          "none -k regex:sweep_kernel -c 10, python scripts/level_table.py 3 reference (cfg3 full, one factorization)",
          "levels": levels, "total_dram_bytes": sum(x["dram_bytes"] for x in levels),
          "total_ncu_ms": sum(x["ncu_ms"] for x in levels)}
    json.dump(tr, open(os.path.join(PROF, "r2_sweep_traffic_cfg3.json"), "w"), indent=1)
    print("sweep DRAM per level (GB, ms):", [(x["level"], round(x["dram_bytes"] / 1e9, 1), round(x["ncu_ms"], 1)) for x in levels])
    print("total GB", round(tr["total_dram_bytes"] / 1e9, 1))

rep = os.path.join(OUT, "sweep_cfg3_L8.ncu-rep")
if os.path.exists(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    open(os.path.join(PROF, "r2_sweep_cfg3_L8_ncu_details.csv"), "w").write(out)
    raw = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = raw.splitlines()
    if len(lines) >= 3:
        hdr = next(csv.reader([lines[0]]))
        val = next(csv.reader([lines[2]]))
        want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "smsp__average_warp_latency_issue_stalled_barrier", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]
        got = {h: v for h, v in zip(hdr, val) if h in want}
        json.dump(got, open(os.path.join(PROF, "r2_sweep_cfg3_L8_ncu_raw.json"), "w"), indent=1)
        print(got)
