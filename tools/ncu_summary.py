"""Summarise an ncu report: duration, throughput, stall reasons, DRAM bytes per kernel.

    python tools/ncu_summary.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_op_hmma.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units, rows = r[0], r[1], r[2:]
    for row in rows:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        print("==", d.get("Kernel Name", "?")[:100])
        for k in KEYS:
            if k in d:
                print(f"    {k} = {d[k]} {u.get(k, '')}")
        tensor = [(k, d[k]) for k in h if "tensor" in k and "pct" in k and d[k] not in ("", "n/a")]
        for k, v in tensor[:6]:
            print(f"    {k} = {v}")
        st = []
        for k in h:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(d[k])))
                except ValueError:
                    pass
        st.sort(key=lambda x: -x[1])
        print("    stalls/issue:", ", ".join(f"{k}={v:.2f}" for k, v in st[:7]))


if __name__ == "__main__":
    main(sys.argv[1])
