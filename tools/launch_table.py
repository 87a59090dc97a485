"""Per-launch table of an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv` log: kernel, duration (us), DRAM read / write (MB)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
d = defaultdict(dict)
for r in rows[1:]:
    d[(int(r[0]), r[ki].split("(")[0])][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
print("| kernel | us | DRAM read MB | DRAM write MB |\n|---|---|---|---|")
for (i, k), m in sorted(d.items()):
    print(f"| `{k}` | {m.get('gpu__time_duration.sum', 0):.1f} | {m.get('dram__bytes_read.sum', 0):.1f} | "
          f"{m.get('dram__bytes_write.sum', 0):.1f} |")
