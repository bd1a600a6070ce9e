"""Per-kernel SASS census of the engine library: tcgen05 MMA (UTCHMMA / UTCQMMA), TMEM loads/stores
(LDTM / STTM), TMA (UTMALDG / UBLKCP), mma.sync (HMMA) and cluster barriers, from cuobjdump -sass.

    python tools/sass_census.py > profiles/r2_sass_census.txt
"""
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_2408_12526_b200" / "_lib" / "libstudentpar_b200.so"
OPS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMAPF", "UBLKCP", "HMMA", "SYNCS", "UCGABAR"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    kernels, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = Counter()
            continue
        if cur is None:
            continue
        for op in OPS:
            if re.search(r"\b" + op + r"(\.|\s)", line):
                kernels[cur][op] += 1
    names = subprocess.run(["c++filt"], input="\n".join(kernels), capture_output=True, text=True).stdout.splitlines()
    total = Counter()
    print(f"# {LIB.name}: SASS instruction census per kernel (cuobjdump -sass)")
    print(f"{'kernel':70s} " + " ".join(f"{o:>8s}" for o in OPS))
    for (mangled, cnt), name in zip(kernels.items(), names):
        total.update(cnt)
        print(f"{name[:70]:70s} " + " ".join(f"{cnt[o]:8d}" for o in OPS))
    print(f"{'TOTAL':70s} " + " ".join(f"{total[o]:8d}" for o in OPS))


if __name__ == "__main__":
    sys.exit(main())
