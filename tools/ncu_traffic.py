"""Write profiles/ncu_traffic.json from an ncu --set full capture of the
stage kernel: DRAM bytes (read + write) per launch, averaged over the
captured launches (one SSPRK3 step = 3 launches), for bench.py's
roofline.traffic field.

    python tools/ncu_traffic.py <report.ncu-rep> <config> [source-note]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep, config, note=""):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = []
    for d in data:
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(k)
            tot += float(d[i]) * scale[units[i]]
        per.append(tot)
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    out[config] = sum(per) / len(per)
    out[config + "_per_launch"] = per
    out[config + "_source"] = note or os.path.basename(rep)
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
