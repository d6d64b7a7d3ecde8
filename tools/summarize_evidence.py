"""Copies one evidence run (tools/evidence_1gpu.sh -> gpurun_out/ev/) into profiles/:
bench line, launch list, ncu summaries, GEMM DRAM traffic and a per-kernel launch table.

    python tools/summarize_evidence.py [gpurun_out/ev] [prefix=r1]
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "ev")
PFX = sys.argv[2] if len(sys.argv) > 2 else "r1"
OUT = os.path.join(ROOT, "profiles")


def ncu_summary(rep, dst):
    with open(dst, "w") as f:
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep], stdout=f, check=True)


def gemm_traffic(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u, rows = r[0], r[1], r[2:]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    launches = []
    for row in rows:
        d, uu = dict(zip(h, row)), dict(zip(h, u))
        b = sum(float(d[k]) * scale[uu[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        t = float(d["gpu__time_duration.sum"])
        t = {"ns": t / 1e3, "us": t, "ms": t * 1e3}[uu["gpu__time_duration.sum"]]
        launches.append({"kernel": d["Kernel Name"][:48], "dram_bytes": b, "us": t})
    return {"workload": "1.3b", "source": "ncu --set full --clock-control none of bench.py --steps 3 --warmup 3 "
            "(the 6 gemm2 launches of one step)", "dram_bytes_per_launch": sum(x["dram_bytes"] for x in launches) /
            max(len(launches), 1), "launches": launches}


def launch_table(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot, n = defaultdict(float), defaultdict(int)
    for r in rows[start + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("moe::<unnamed>::", "")
        if name.startswith("at::"):
            continue
        tot[name] += float(r[vi].replace(",", ""))
        n[name] += 1
    allt = sum(tot.values())
    lines = ["| kernel | launches | mean us / launch | share of our kernel time |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| `{k}` | {n[k]} | {v / n[k] / 1e3:.1f} | {100 * v / allt:.1f}% |")
    return "\n".join(lines)


def main():
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(SRC, "bench.json")) as f:
        line = f.read().strip().splitlines()[-1]
    json.loads(line)
    open(os.path.join(OUT, f"{PFX}_bench_1gpu.json"), "w").write(line + "\n")
    if os.path.exists(os.path.join(SRC, "launches.csv")):
        subprocess.run(["cp", os.path.join(SRC, "launches.csv"), os.path.join(OUT, f"{PFX}_launches.csv")], check=True)
        open(os.path.join(OUT, f"{PFX}_launch_table.md"), "w").write(launch_table(os.path.join(SRC, "launches.csv")) + "\n")
    for rep, name in (("gemm_full", "gemm"), ("other_full", "other"), ("small_full", "small"), ("optim_full", "optim")):
        p = os.path.join(SRC, rep + ".ncu-rep")
        if os.path.exists(p):
            ncu_summary(p, os.path.join(OUT, f"{PFX}_{name}_ncu_summary.txt"))
    p = os.path.join(SRC, "gemm_full.ncu-rep")
    if os.path.exists(p):
        json.dump(gemm_traffic(p), open(os.path.join(OUT, "gemm_traffic.json"), "w"), indent=1)
    print("ok")


if __name__ == "__main__":
    main()
