"""SASS instruction summary of every kernel in the built objects (cuobjdump
-sass): counts of the mnemonics that show which hardware path a kernel uses —
tcgen05 MMA / TMEM loads (UTCHMMA, LDTM), TMA (UTMALDG, UTMASTG, UBLKCP),
cp.async (LDGSTS), plain global loads / stores, shuffles, spills (LDL/STL).

  python tools/sass_summary.py > profiles/r02_sass_summary.md
"""
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMASTG", "UBLKCP", "LDGSTS", "LDG", "STG", "LDS", "STS",
        "SHFL", "VOTE", "ATOMS", "RED", "LDL", "STL"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return out[:len(names)]


def main():
    objs = sorted(glob.glob(os.path.join(ROOT, "paper_2507_16991_b200", "csrc", "build", "*.o")))
    print("# SASS instruction summary (sm_100a, cuobjdump -sass of the built objects)\n")
    print("Counts are static instructions in each kernel's SASS (not executions). "
          "UTCHMMA = tcgen05.mma, LDTM = tcgen05.ld, UTMALDG/UTMASTG = TMA tensor load/store, "
          "LDGSTS = cp.async, LDL/STL = local-memory spills.\n")
    for o in objs:
        sass = subprocess.run(["cuobjdump", "-sass", o], capture_output=True, text=True).stdout
        funcs = re.split(r"\n\s*Function : ", sass)[1:]
        rows = []
        for f in funcs:
            name = f.split("\n", 1)[0].strip()
            body = f
            cnt = {k: len(re.findall(r"\b" + k + r"(\.|\s)", body)) for k in KEYS}
            rows.append((name, cnt))
        if not rows:
            continue
        names = demangle([r[0] for r in rows])
        print(f"## {os.path.basename(o)}\n")
        print("| kernel | " + " | ".join(KEYS) + " |")
        print("|---|" + "---|" * len(KEYS))
        for (raw, cnt), nm in zip(rows, names):
            nm = nm.replace("void ", "").split("(")[0]
            if len(nm) > 90:
                nm = nm[:87] + "..."
            print(f"| `{nm}` | " + " | ".join(str(cnt[k]) for k in KEYS) + " |")
        print()


if __name__ == "__main__":
    sys.exit(main())
