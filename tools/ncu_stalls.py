"""Stall reasons per CUDA source line (sampled) of one kernel in an ncu report.

usage: python tools/ncu_stalls.py REP [KERNEL_REGEX] [TOP]
"""
import csv
import io
import subprocess
import sys

REASONS = ["long_sb", "short_sb", "wait", "mio", "lg", "barrier", "branch_resolving", "math",
           "not_selected", "selected", "drain", "membar", "no_inst", "dispatch", "misc"]


def main(rep, kernel=None, top=30):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:
        cmd += ["--kernel-name", "regex:" + kernel]
    txt = subprocess.run(cmd, capture_output=True, text=True, errors="replace").stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = next(r for r in rows if len(r) > 3 and r[0] == "Line No")
    col = {h: i for i, h in enumerate(hdr) if h != "Source"}
    tot_i = col["Warp Stall Sampling (All Samples)"]
    lines, totals = [], {k: 0 for k in REASONS}
    for r in rows:
        if len(r) == len(hdr) and r[0] not in ("", "Line No") and r[2] == "-":
            try:
                d = {k: int(r[col["stall_" + k]] or 0) for k in REASONS}
            except (KeyError, ValueError):
                continue
            for k in REASONS:
                totals[k] += d[k]
            lines.append((int(r[tot_i] or 0), r[0], r[1].strip(), d))
    T = sum(totals.values()) or 1
    print("totals:", ", ".join(f"{k} {100 * v / T:.1f}%" for k, v in
                               sorted(totals.items(), key=lambda x: -x[1]) if v))
    for n, ln, src, d in sorted(lines, key=lambda x: -x[0])[:top]:
        det = " ".join(f"{k}={100 * v / T:.1f}" for k, v in sorted(d.items(), key=lambda x: -x[1])[:3] if v)
        print(f"{ln:>5} {100 * n / T:5.1f}%  {src[:70]:70s} {det}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None,
         int(sys.argv[3]) if len(sys.argv) > 3 else 30)
