"""K1 instruction / stall-sample breakdown by phase from an ncu --set full report.

    python tools/k1_phases.py gpurun_out/prof_v11.ncu-rep

Segments are the SASS ranges between K1's block barriers (phase 1 ends at the
barrier before phase 2, etc.; phase 3, the classifier, is the segment after
the last barrier; code placed after the kernel's EXIT is reported separately).  Uses `ncu -i ... --page source --print-source sass --csv`.
"""
import csv
import io
import subprocess
import sys


def main(rep, kernel="k1v3"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ie, sa = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    data = [(r[1].strip(), int(r[ie] or 0), int(r[sa] or 0)) for r in rows[2:] if len(r) > ie]
    T, S = sum(d[1] for d in data), sum(d[2] for d in data)
    segs, cur, name = [], [0, 0], "prologue"
    nbar = 0
    for s, n, sm in data:
        op = s.split()[1] if s.startswith("@") else (s.split()[0] if s else "")
        if n > 0 and (op.startswith("BAR") or op == "EXIT"):
            segs.append((name, *cur))
            cur = [0, 0]
            nbar += op.startswith("BAR")
            name = "after EXIT (out-of-line code)" if op == "EXIT" else f"after barrier {nbar}"
        cur[0] += n
        cur[1] += sm
    segs.append((name, *cur))
    print(f"{'segment':40s} {'warp-instr':>12s} {'share':>7s} {'samples':>8s}")
    for name, n, sm in segs:
        if n or sm:
            print(f"{name:40s} {n:12d} {n / T * 100:6.1f}% {sm / S * 100:7.1f}%")
    print(f"{'total':40s} {T:12d}")


if __name__ == "__main__":
    main(*sys.argv[1:])
