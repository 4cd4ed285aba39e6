"""Per-source-line instructions and stall samples of one kernel from an ncu
--set full report: ncu's SASS page (metrics per instruction, in address order)
zipped with nvdisasm -g line info of the same function from the built object.

    python tools/ncu_lines.py REPORT KERNEL_REGEX OBJECT MANGLED_NAME [TOP]
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_lines(obj, mangled):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    out, cur, inside = [], None, False
    for line in txt.splitlines():
        if line.startswith(".text."):
            inside = line[len(".text."):-1] == mangled
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            out.append((cur, m.group(2).strip()))
    return out


def main(rep, kern, obj, mangled, top=40):
    csvt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                           "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(csvt)))
    h = next(r for r in rows if "Instructions Executed" in r)
    start = rows.index(h) + 1
    ie, sa = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    prof = []
    for r in rows[start:]:
        if len(r) <= ie:
            continue
        if not (r[ie] or "0").isdigit():
            break  # the next kernel's table
        prof.append((r[1].strip(), int(r[ie] or 0), int(r[sa] or 0)))
    lines = sass_lines(obj, mangled)
    if len(lines) != len(prof):
        print(f"warning: {len(lines)} disassembled vs {len(prof)} profiled instructions", file=sys.stderr)
    agg = {}
    for (src, _), (s, n, sm) in zip(lines, prof):
        a = agg.setdefault(src, [0, 0])
        a[0] += n
        a[1] += sm
    T = sum(v[0] for v in agg.values()) or 1
    S = sum(v[1] for v in agg.values()) or 1
    print(f"{'line':28s} {'instr%':>7s} {'stall%':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[: int(top)]:
        print(f"{str(k):28s} {v[0] / T * 100:6.1f}% {v[1] / S * 100:6.1f}%")
    print(f"total instructions {T}, samples {S}")


if __name__ == "__main__":
    main(*sys.argv[1:])
