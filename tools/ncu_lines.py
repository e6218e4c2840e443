"""Top CUDA source lines of an ncu report by warp-stall samples.

    python tools/ncu_lines.py <report.ncu-rep> [section_index] [top]
"""
import csv
import io
import subprocess
import sys


def main(rep, sec=1, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "sass,cuda"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    secs, cur, hdr = [], None, None
    launch = -1
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1]
            if fname.endswith("dgswe_kernels.cuh"):
                launch += 1
        if r and r[0] == "Function Name":
            cur = [] if fname.endswith("dgswe_kernels.cuh") else None
            if cur is not None:
                secs.append(cur)
        elif r and r[0] == "Line No":
            hdr = r
        elif cur is not None and r and r[0].isdigit() and len(r) > 5 and r[2] == "-":
            cur.append(r)
    data = secs[min(sec, len(secs) - 1)]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    tot = sum(int(r[si] or 0) for r in data) or 1
    toti = sum(int(r[ie] or 0) for r in data) or 1
    print(f"{len(secs)} sections; samples {tot}; warp-instr {toti}")
    for r in sorted(data, key=lambda r: -int(r[si] or 0))[:top]:
        print(f"{100*int(r[si] or 0)/tot:5.1f}% smp {100*int(r[ie] or 0)/toti:5.1f}% ins  L{r[0]:>4} {r[1].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1,
         int(sys.argv[3]) if len(sys.argv) > 3 else 40)
