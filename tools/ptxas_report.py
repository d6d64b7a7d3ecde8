"""Per-kernel registers / spills / smem from `nvcc -Xptxas -v` (one source file).

    python tools/ptxas_report.py paper_2305_13525_b200/csrc/route.cu
"""
import re
import subprocess
import sys

sys.path.insert(0, ".")
from paper_2305_13525_b200.build import ARCH, NVCC, ROOT, nccl_dirs  # noqa: E402


def main(src):
    inc, _ = nccl_dirs()
    cmd = [NVCC, "-O3", "-std=c++17", *ARCH, "-I", f"{ROOT}/include", "-I", inc, "-Xptxas", "-v",
           "-c", src, "-o", "/dev/null"]
    err = subprocess.run(cmd, capture_output=True, text=True).stderr
    name = None
    spill = ""
    for line in err.splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            raw = m.group(1)
            dm = subprocess.run(["c++filt", raw], capture_output=True, text=True).stdout.strip()
            name = re.sub(r"\(.*", "", dm.replace("moe::(anonymous namespace)::", ""))
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            spill = f"spill st/ld {m.group(1)}/{m.group(2)}"
        m = re.search(r"Used (\d+) registers(.*)", line)
        if m and name:
            print(f"{name:60s} regs={m.group(1):>4s} {spill} {m.group(2).strip(', ')}")
            name = None
    if "error" in err:
        print(err)


if __name__ == "__main__":
    for s in sys.argv[1:]:
        main(s)
