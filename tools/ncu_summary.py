"""Summarise an ncu report (stage kernel) into a small text/JSON file.

    python tools/ncu_summary.py gpurun_out/<tag>_stage.ncu-rep profiles/<round>/<name>
writes <name>.txt (key metrics + stall breakdown) and <name>.json.
"""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.max", "smsp__inst_executed.avg",
    "smsp__cycles_active.avg", "sm__warps_active.avg.per_cycle_active",
]


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        rec = {"kernel": d[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                rec[k] = d[hdr.index(k)] + (" " + units[hdr.index(k)] if units[hdr.index(k)] else "")
        stalls = {}
        for i, h in enumerate(hdr):
            m = re.match(r"smsp__pcsamp_warps_issue_stalled_(\w+)$", h)
            if m and not h.endswith("_not_issued"):
                try:
                    stalls[m.group(1)] = int(float(d[i]))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1
        rec["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in
                            sorted(stalls.items(), key=lambda kv: -kv[1]) if v}
        res.append(rec)
    json.dump(res, open(out + ".json", "w"), indent=1)
    with open(out + ".txt", "w") as fh:
        for i, r in enumerate(res):
            fh.write(f"--- launch {i}: {r['kernel']}\n")
            for k in KEYS:
                if k in r:
                    fh.write(f"  {k:70s} {r[k]}\n")
            fh.write("  stalls (% of samples): " + ", ".join(f"{k} {v}" for k, v in
                                                            r["stall_pct"].items()) + "\n")
    print(open(out + ".txt").read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
