"""Average duration per kernel from an ncu --metrics gpu__time_duration.sum --csv launch list.

    python tools/launch_summary.py gpurun_out/launches.csv [...]
"""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    d = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ik].replace("void ", "").replace("ef::", "").replace("<unnamed>::", "")
        k = name.split("(")[0].split("<")[0] or "(memset/other)"
        d.setdefault(k, []).append(float(r[iv]))
    print("==", path)
    for k, v in d.items():
        print(f"  {k:32s} n={len(v):3d} avg={sum(v) / len(v) / 1000:9.2f} us")
