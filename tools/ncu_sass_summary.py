"""Summarise an ncu SASS source page (csv) by opcode and hottest instructions.

usage: ncu -i rep --page source --csv [--kernel-name ...] > x.csv; python tools/ncu_sass_summary.py x.csv
"""
import csv
import collections
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    col = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
    ex = col["Instructions Executed"]
    st = col["Warp Stall Sampling (All Samples)"]
    by_op = collections.Counter()
    stall_op = collections.Counter()
    tot = 0
    tot_st = 0
    for r in data:
        op = r[1].split()[0] if r[1].split() else "?"
        if op.startswith("@"):
            op = r[1].split()[1]
        op = op.split(".")[0]
        n = int(r[ex] or 0)
        s = int(r[st] or 0)
        by_op[op] += n
        stall_op[op] += s
        tot += n
        tot_st += s
    print(f"total warp-instructions executed {tot:,}; stall samples {tot_st:,}")
    for op, n in by_op.most_common(25):
        print(f"  {op:10s} {n:14,} {100*n/tot:5.1f}%  stall {100*stall_op[op]/max(tot_st,1):5.1f}%")
    print("hottest instructions by stall samples:")
    for r in sorted(data, key=lambda r: -int(r[st] or 0))[:top]:
        print(f"  {r[0][-5:]} {int(r[st] or 0):7d} ex={int(r[ex] or 0):10,}  {r[1].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
