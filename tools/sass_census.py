"""SASS census of the built libsalus.so: counts of the Blackwell-specific
instructions that prove the tcgen05 / TMA / TMEM path (B200_PROFILING.md's
mnemonics), with one example line each.

usage: python tools/sass_census.py [out.txt]   (default profiles/r02_sass_census.txt)
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
LIB = os.path.join(ROOT, "paper_1902_04610_b200", "libsalus.so")
PAT = re.compile(r"\b(UTC[A-Z0-9_.]*|UTMA[A-Z0-9_.]*|UBLKCP[A-Z0-9_.]*|UBLKRED[A-Z0-9_.]*|LDTM[A-Z0-9_.]*|"
                 r"STTM[A-Z0-9_.]*|SYNCS[A-Z0-9_.]*|FENCE\.VIEW\.ASYNC[A-Z0-9_.]*)")
MEANING = {
    "UTCHMMA": "tcgen05.mma kind::f16 (bf16 -> fp32 TMEM accumulator)",
    "UTCBAR": "tcgen05.commit -> mbarrier (multicast to both CTAs of the pair)",
    "UTMALDG": "cp.async.bulk.tensor load (TMA, 2-D tensor map)",
    "UTMASTG": "cp.async.bulk.tensor store (TMA)",
    "UBLKCP": "cp.async.bulk (non-tensor bulk copy)",
    "UBLKRED": "cp.reduce.async.bulk",
    "LDTM": "tcgen05.ld (TMEM -> registers)",
    "STTM": "tcgen05.st",
    "UTCATOMSWS": "tcgen05.alloc / dealloc (TMEM allocator)",
    "SYNCS": "mbarrier operations",
    "FENCE.VIEW.ASYNC": "fence.proxy.async",
}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02_sass_census.txt")
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    counts, example = collections.Counter(), {}
    for line in sass.splitlines():
        for m in PAT.finditer(line):
            counts[m.group(1)] += 1
            example.setdefault(m.group(1), line.strip()[:140])
    funcs = re.findall(r"Function : (\S+)", sass)
    lines = [f"SASS census of {os.path.relpath(LIB, ROOT)} ({len(sass.splitlines())} lines of SASS)",
             "functions: " + ", ".join(funcs), ""]
    for mn, c in sorted(counts.items(), key=lambda kv: (-kv[1], kv[0])):
        fam = next((k for k in MEANING if mn.startswith(k)), "")
        lines.append(f"{c:6d}  {mn:<40} {MEANING.get(fam, '')}")
    lines.append("")
    lines.append("examples:")
    for mn in sorted(example):
        lines.append(f"  {example[mn]}")
    txt = "\n".join(lines) + "\n"
    with open(out, "w") as f:
        f.write(txt)
    print(txt)


if __name__ == "__main__":
    main()
