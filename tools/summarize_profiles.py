"""Summarise ncu artefacts from gpurun_out/ into committed profiles/.

usage: python tools/summarize_profiles.py TAG [WORKLOAD_KEY]
  (WORKLOAD_KEY, e.g. config4/tf32: the bench workload the traffic list was
   taken on; bench.py looks the dominant kernel's traffic up under it)
  reads  gpurun_out/launches_TAG.csv        (ncu --metrics gpu__time_duration.sum list)
         gpurun_out/traffic_TAG.csv         (optional: dram bytes per launch, all launches)
         gpurun_out/prof_TAG_*.ncu-rep      (ncu --set full captures)
  writes profiles/ncu_summary_TAG.md, profiles/ncu_traffic.json
"""
import csv
import glob
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

FAMILY = [("igemm_kernel", "igemm_kernel (KB-CONV / KB-KS)"), ("wgrad_row_kernel", "wgrad_row_kernel (KB-WGRAD-ROW)"),
          ("fwd_row_kernel", "fwd_row_kernel (KB-CONV-ROW)"), ("wgrad_kernel", "wgrad_kernel (KB-WGRAD)"),
          ("ks_split", "ks_split_kernel (KB-SPLIT)"), ("reduce_partials", "reduce_partials (KB-REDUCE)"),
          ("pad_channels", "pad_channels (KB-PAD)")]


def fam(name):
    for key, label in FAMILY:
        if key in name:
            return label
    return "other: " + name[:50]


def read_ncu_csv(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def to_us(v, unit):
    v = float(v.replace(",", ""))
    return {"nsecond": v / 1e3, "usecond": v, "msecond": v * 1e3, "ns": v / 1e3, "us": v}.get(unit, v)


def launches(tag):
    p = os.path.join(OUT, f"launches_{tag}.csv")
    if not os.path.exists(p):
        return None
    rows = [r for r in read_ncu_csv(p) if r["Metric Name"] == "gpu__time_duration.sum"]
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        v = to_us(r["Metric Value"], r["Metric Unit"])
        if v != v:  # nan: launch not measured
            continue
        f = fam(r["Kernel Name"])
        per[f][0] += 1
        per[f][1] += v
    return per


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {h[i]: (v[i], u[i]) for i in range(min(len(h), len(v)))}
        res.append(d)
    return res


def num(d, k):
    if k not in d:
        return None
    v, u = d[k]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
    return x * scale.get(u, 1)


def main(tag, key="config4/tf32"):
    os.makedirs(PROF, exist_ok=True)
    md = [f"# ncu summary -- round {tag}\n",
          "Captured on one B200 with `--clock-control none` (see tools/ncu_full.sh, bench.py).  ncu times are",
          "cold-cache and serialised: compare SHARES of the step, not absolute times.\n"]
    per = launches(tag)
    if per:
        tot = sum(v[1] for v in per.values())
        md += ["## Launch list (one bench step incl. warm-up launches)\n", "| kernel family | launches | total us | share |",
               "|---|---|---|---|"]
        for f, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            md.append(f"| {f} | {n} | {t:.1f} | {t / tot:.1%} |")
        md.append("")
    traffic = {}
    tp = os.path.join(OUT, f"traffic_{tag}.csv")
    if os.path.exists(tp):
        rows = read_ncu_csv(tp)
        by = defaultdict(lambda: defaultdict(float))
        for r in rows:
            lk = (r["ID"], r["Kernel Name"])
            v = float(r["Metric Value"].replace(",", ""))
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r["Metric Unit"], 1)
            by[lk][r["Metric Name"]] += v * mult
        agg = defaultdict(list)
        for (i, name), m in by.items():
            b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
            if b != b:  # nan: launch not measured
                continue
            agg[name.split("<")[0].split("(")[0].replace("void ", "").replace("cks::", "")].append(b)
        for k, v in agg.items():
            traffic[k] = {"dram_bytes_per_launch": sum(v) / len(v), "launches": len(v)}
        md += ["## DRAM traffic per launch (all launches of one step)\n", "| kernel | launches | mean dram bytes/launch |",
               "|---|---|---|"]
        for k, v in traffic.items():
            md.append(f"| {k} | {v['launches']} | {v['dram_bytes_per_launch'] / 1e6:.2f} MB |")
        md.append("")
    reps = sorted(glob.glob(os.path.join(OUT, f"prof_{tag}_*.ncu-rep")))
    if reps:
        md += ["## Full captures (`ncu --set full`)\n",
               "| capture | kernel | us | DRAM MB (r+w) | tensor pipe % (active) | L2 thru % | SM thru % | regs |",
               "|---|---|---|---|---|---|---|---|"]
        for rep in reps:
            for d in raw_metrics(rep):
                name = d.get("Kernel Name", ("?",))[0]
                dur = num(d, "gpu__time_duration.sum")
                dram = (num(d, "dram__bytes_read.sum") or 0) + (num(d, "dram__bytes_write.sum") or 0)
                tens = num(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
                l2 = num(d, "lts__throughput.avg.pct_of_peak_sustained_elapsed")
                sm = num(d, "sm__throughput.avg.pct_of_peak_sustained_elapsed")
                regs = num(d, "launch__registers_per_thread")
                cap = os.path.basename(rep).replace(".ncu-rep", "")
                md.append(f"| {cap} | {re.sub(r'[(<].*', '', name)[:40]} | {dur:.2f} | {dram / 1e6:.2f} | "
                          f"{tens if tens is not None else float('nan'):.1f} | {l2 or 0:.1f} | {sm or 0:.1f} | "
                          f"{regs or 0:.0f} |")
        md.append("")
    with open(os.path.join(PROF, f"ncu_summary_{tag}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    if traffic:
        tj = os.path.join(PROF, "ncu_traffic.json")
        try:
            allt = json.load(open(tj))
        except Exception:
            allt = {}
        allt = {k: v for k, v in allt.items() if "/" in k}  # drop the round-1 flat layout
        allt[key] = {k.split("_kernel")[0] + "_kernel": v for k, v in traffic.items()}
        with open(tj, "w") as f:
            json.dump(allt, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02", *sys.argv[2:3])
