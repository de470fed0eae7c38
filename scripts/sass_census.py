"""Per-kernel SASS census of the built objects (Blackwell-native evidence): counts of the tcgen05 / TMA
instructions in every kernel of build/*.o.   python scripts/sass_census.py > profiles/<tag>_sass_census.txt

UTCHMMA / UTCQMMA  tcgen05.mma (TMEM accumulator)     LDTM / STTM   tcgen05.ld / tcgen05.st
UTMALDG / UTMASTG  TMA tensor load / store            UTMAPF        TMA prefetch
UBLKCP             cp.async.bulk (non-tensor)         HMMA          legacy mma.sync (should be 0)"""
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ("UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "SYNCS", "HMMA")


def census(obj):
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True, check=True).stdout
    out, name, counts = [], None, None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if name:
                out.append((name, counts))
            name, counts = m.group(1), dict.fromkeys(OPS, 0)
            continue
        if name:
            for op in OPS:
                if re.search(r"\b" + op + r"\b", line):
                    counts[op] += 1
    if name:
        out.append((name, counts))
    return out


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines() if r.returncode == 0 else names


def main():
    print("# SASS census (cuobjdump -sass build/*.o), sm_100a")
    print("# " + " ".join(OPS))
    for obj in sorted(glob.glob(os.path.join(ROOT, "build", "*.o"))):
        rows = census(obj)
        if not rows:
            continue
        pretty = demangle([n for n, _ in rows])
        print(f"\n## {os.path.basename(obj)}")
        for (n, c), p in zip(rows, pretty):
            short = p.split("(")[0]
            print(f"{short:60s} " + " ".join(f"{op}={c[op]}" for op in OPS if c[op]))


if __name__ == "__main__":
    sys.exit(main())
