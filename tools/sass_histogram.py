"""SASS instruction histogram of the stage kernels (evidence for the
TMA / mbarrier / FP64 claims in DESIGN.md).

    python tools/sass_histogram.py [build/dgswe_obj/deg_p3.o ...] > profiles/r02/sass_histogram.txt
Counts static SASS opcodes (first mnemonic, predicates and modifiers
stripped to the base op plus its first modifier) per kernel, including the
non-inlined face-flux subroutine it calls.
"""
import collections
import re
import subprocess
import sys

KEEP = ("stage_kernel", "face_flux_noinline")


def functions(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True, check=True).stdout
    cur, body = None, {}
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            body[cur] = []
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if cur and m:
            body[cur].append(m.group(1))
    return body


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()


def main():
    objs = sys.argv[1:] or ["build/dgswe_obj/deg_p3.o", "build/dgswe_obj/deg_p4.o"]
    groups = {"FP64": ("DFMA", "DMUL", "DADD", "DSETP", "DMMA", "MUFU.RCP64H", "MUFU.RSQ64H"),
              "TMA/bulk": ("UBLKCP", "UBLKPF", "UTMALDG", "UTMASTG", "UBLKRED"),
              "mbarrier": ("SYNCS",), "async copy": ("LDGSTS",), "barrier": ("BAR",),
              "shared": ("LDS", "STS"), "global": ("LDG", "STG", "LD", "ST")}
    for obj in objs:
        body = functions(obj)
        names = [n for n in body if any(k in n for k in KEEP)]
        for n, d in zip(names, demangle(names)):
            ops = body[n]
            full = collections.Counter(ops)
            base = collections.Counter(o.split(".")[0] for o in ops)
            print(f"== {d}  [{obj}]  {len(ops)} SASS instructions")
            for g, pref in groups.items():
                cnt = sum(c for o, c in full.items() if any(o == p or o.startswith(p + ".") for p in pref))
                print(f"   {g:11s} {cnt}")
            print("   top: " + ", ".join(f"{o} {c}" for o, c in base.most_common(24)))
            detail = sorted((o, c) for o, c in full.items()
                            if o.split(".")[0] in ("UBLKCP", "UBLKPF", "SYNCS", "LDGSTS", "MUFU", "DMMA", "BAR"))
            print("   detail: " + ", ".join(f"{o} {c}" for o, c in detail))


if __name__ == "__main__":
    main()
