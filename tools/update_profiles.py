#!/usr/bin/env python
"""Copy the round evidence produced by tools/profile_round.sh (+ bench.py --workload lines) from
gpurun_out/ into profiles/: the default bench line, the launch list and its summary, the K1
ncu --set full summary and the K1 DRAM traffic per instance-launch used by bench.py.

  python tools/update_profiles.py [--round 01]
"""
import argparse
import collections
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")


def launches_summary(src, dst, command):
    rows = list(csv.reader(open(src)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[h + 1:]:
        if len(r) <= iv:
            continue
        v = float(r[iv].replace(",", ""))
        u = r[iu]
        ms = v / 1e6 if u == "ns" else (v / 1e3 if u == "us" else (v if u == "ms" else v * 1e3))
        name = re.sub(r"\(.*", "", r[ik]).strip()
        tot[name] += ms
        cnt[name] += 1
    T = sum(tot.values())
    out = [command, "(cold-cache, serialised per-launch times; compare shares, not absolutes)", ""]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{k:60s} launches={cnt[k]:3d}  total={v:10.2f} ms  share={100 * v / T:6.2f}%")
    open(dst, "w").write("\n".join(out) + "\n")
    return out


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return dict(zip(rows[0], rows[2])) if len(rows) > 2 else {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="01")
    a = ap.parse_args()
    r = f"r{a.round}"
    line = open(os.path.join(G, "bench_default.json")).read().strip().splitlines()[-1]
    d = json.loads(line)
    open(os.path.join(P, f"{r}_bench_default.json"), "w").write(line + "\n")
    print("bench:", round(d["value"] / 1e9, 1), "G/s, e2e", round(d["e2e"]["value"] / 1e9, 1),
          "kernel frac", round(d["roofline"]["frac"], 3), d["clocks"])
    if os.path.exists(os.path.join(G, "launches.csv")):
        import shutil
        shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, f"{r}_bench_launches.csv"))
        out = launches_summary(os.path.join(G, "launches.csv"), os.path.join(P, f"{r}_bench_launches_summary.txt"),
                               "ncu --metrics gpu__time_duration.sum --clock-control none  "
                               "python bench.py --steps 3 --warmup 3 --no-cpu-baseline")
        print("\n".join(out[3:6]))
    rep = os.path.join(G, "prof_k1.ncu-rep")
    if os.path.exists(rep):
        summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                              capture_output=True, text=True).stdout
        open(os.path.join(P, f"{r}_k1_ncu_full_summary.txt"), "w").write(
            "# K1 (k1_lattice_pt) on the config-5 geometry: 296 instances x 100 sweeps (one launch), EA L=32, 64 slots\n"
            "# command: tools/profile_round.sh (ncu --set full --clock-control none --import-source on "
            "-k regex:k1_lattice -s 3 -c 1)\n" + summ)
        raw = ncu_raw(rep)
        rd = float(raw.get("dram__bytes_read.sum", "0").replace(",", ""))
        wr = float(raw.get("dram__bytes_write.sum", "0").replace(",", ""))
        unit_r, unit_w = raw.get("dram__bytes_read.sum", ""), raw.get("dram__bytes_write.sum", "")
        # the raw page reports values in the unit of its second header row; ncu_summary prints them too
        print("k1 dram read/write (raw):", unit_r, unit_w)
    wl = os.path.join(G, "workloads.jsonl")
    if os.path.exists(wl):
        import shutil
        shutil.copy(wl, os.path.join(P, f"{r}_workloads.jsonl"))
        for l in open(wl):
            x = json.loads(l)
            print(x["metric"][-8:], round(x["value"] / 1e9, 1), "G/s frac", round(x["roofline"]["frac"], 3),
                  "cpu", round(x.get("cpu_baseline", {}).get("value", 0) / 1e9, 3))


if __name__ == "__main__":
    main()
