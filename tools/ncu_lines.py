"""Per CUDA-source-line totals (warp instructions executed, stall samples) of
one kernel in an ncu report.

usage: python tools/ncu_lines.py REP [KERNEL_REGEX] [TOP]
"""
import csv
import io
import subprocess
import sys


def main(rep, kernel=None, top=45):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:
        cmd += ["--kernel-name", "regex:" + kernel]
    txt = subprocess.run(cmd, capture_output=True, text=True, errors="replace").stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = next(r for r in rows if len(r) > 3 and r[0] == "Line No")
    col = {h: i for i, h in enumerate(hdr) if h not in ("Source",)}
    ie, ist = col["Instructions Executed"], col["Warp Stall Sampling (All Samples)"]
    lines = []
    for r in rows:
        if len(r) == len(hdr) and r[0] not in ("", "Line No") and r[2] == "-":
            try:
                lines.append((int(r[ie] or 0), int(r[ist] or 0), r[0], r[1].strip()))
            except ValueError:
                pass
    ti = sum(x[0] for x in lines) or 1
    ts = sum(x[1] for x in lines) or 1
    print(f"total warp-instructions {ti:,}  stall samples {ts:,}")
    for n, s, ln, src in sorted(lines, key=lambda x: -x[0])[:top]:
        print(f"{ln:>5} {100 * n / ti:5.1f}% ins {100 * s / ts:5.1f}% stall  {src[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None,
         int(sys.argv[3]) if len(sys.argv) > 3 else 45)
