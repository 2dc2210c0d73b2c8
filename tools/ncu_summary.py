"""Summarise an ncu report (.ncu-rep) into JSON: per kernel duration, DRAM
bytes, throughput, pipe utilisation, occupancy, top stall reasons.

usage: python tools/ncu_summary.py report.ncu-rep > profiles/xxx.json
"""
import csv
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "ns": 1, "us": 1e3, "ms": 1e6,
              "msecond": 1e6}


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:80]}
        stalls = {}
        for i, name in enumerate(hdr):
            val = r[i].replace(",", "")
            if name in KEYS:
                try:
                    v = float(val) * UNIT_SCALE.get(units[i], 1)
                except ValueError:
                    continue
                d[KEYS[name]] = v
            if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
                try:
                    stalls[name.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(val)
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1
        d["top_stalls_pct"] = {k: round(100 * v / tot, 1)
                               for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:5]}
        res.append(d)
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
