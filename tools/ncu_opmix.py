"""Executed SASS opcode counts per CUDA source line (ncu source page,
sass+cuda correlation) for one kernel section of a report.

    python tools/ncu_opmix.py <report.ncu-rep> [section] [opcode-prefix ...]
"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, sec=1, ops=("DMUL", "IMAD", "DFMA")):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True).stdout
    secs, cur, line, fname = [], None, None, ""
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
        elif r and r[0] == "Function Name":
            if not secs or secs[-1][0] != r[1] or fname == "dgswe_kernels.cuh" and secs[-1][2]:
                secs.append((r[1], collections.defaultdict(collections.Counter), set()))
            cur = secs[-1][1]
            secs[-1][2].add(fname)
        elif r and r[0] == "Line No":
            hdr = r
        elif cur is not None and len(r) > 8:
            if r[0]:
                line = (fname[:10] + ":" + r[0], r[1].strip()[:80])
            elif r[2].startswith("0x"):
                ie = int(r[7] or 0)
                toks = r[3].split()
                if toks and toks[0].startswith("@"):
                    toks = toks[1:]
                if toks:
                    cur[line][toks[0].split(".")[0]] += ie
    name, data, _ = secs[min(sec, len(secs) - 1)]
    print(name)
    for op in ops:
        tot = sum(c[op] for c in data.values())
        print(f"== {op}: {tot}")
        for ln, c in sorted(data.items(), key=lambda kv: -kv[1][op])[:14]:
            if c[op]:
                print(f"  {c[op]:9d}  L{ln[0]:>5} {ln[1]}")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], int(a[1]) if len(a) > 1 else 1, tuple(a[2:]) or ("DMUL", "IMAD", "DFMA"))
