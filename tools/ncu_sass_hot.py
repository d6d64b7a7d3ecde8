"""Hottest SASS lines of one kernel in an ncu report (stall samples + exec counts).

    python tools/ncu_sass_hot.py report.ncu-rep <kernel-regex> [N]
"""
import csv
import io
import subprocess
import sys


def main(path, kern, n=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r != hdr]
    data = [d for d in data if (d["Warp Stall Sampling (All Samples)"] or "0").isdigit()]
    tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
    print(f"{len(data)} SASS lines, {tot} stall samples")
    # window view: print hot lines in address order with their samples
    hot = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:int(n)]
    hot_addr = {d["Address"] for d in hot}
    for d in data:
        if d["Address"] in hot_addr:
            print(f'{d["Address"][-5:]} {int(d["Warp Stall Sampling (All Samples)"]):6d} '
                  f'{int(d["Instructions Executed"] or 0):9d}  {d["Source"].strip()}')


if __name__ == "__main__":
    main(*sys.argv[1:])
