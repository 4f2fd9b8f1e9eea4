"""Per-kernel SASS opcode summary of libmoe_b200.so (cuobjdump -sass): the
tcgen05 / TMA / TMEM opcodes that prove which kernels run on the 5th-gen
tensor cores, plus instruction counts.  Writes profiles/<name>.md.

  python scripts/sass_summary.py [profiles/r02_sass_summary.md]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2109_10465_b200", "libmoe_b200.so")
WATCH = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMACMDFLUSH", "UBLKCP", "LDTM", "STTM",
         "SYNCS", "DFMA", "DMUL", "DADD", "FFMA", "HMMA", "ELECT"]


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02_sass_summary.md")
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    arch = sorted(set(re.findall(r"arch = (sm_\w+)", sass)))
    kern = None
    counts = collections.OrderedDict()
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            kern = m.group(1)
            counts[kern] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if kern and m:
            op = m.group(1)
            full = op + (m.group(2) or "")
            counts[kern]["_total"] += 1
            for w in WATCH:
                if op == w:
                    key = full if w in ("UTCHMMA", "UTMALDG", "UTMASTG") else w
                    counts[kern][key] += 1
    demangled = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.split("\n")
    lines = [f"# SASS opcode summary of `paper_2109_10465_b200/libmoe_b200.so` ({', '.join(arch)})", "",
             "`python scripts/sass_summary.py` (cuobjdump -sass).  Tensor-core / TMA / TMEM opcodes per kernel;",
             "`UTCHMMA` = tcgen05.mma, `.2CTA` = cta_group::2, `UTMALDG` / `UTMASTG` = TMA tensor load / store,",
             "`LDTM` = tcgen05.ld.  Kernels without any of them run on the SIMT pipes.", "",
             "| kernel | instructions | tcgen05 / TMA / TMEM | other |", "|---|---|---|---|"]
    for (k, c), name in zip(counts.items(), demangled):
        name = (name or k).replace("|", "\\|")
        tc = ", ".join(f"{op} {n}" for op, n in sorted(c.items()) if op.startswith(("UTC", "UTMA", "LDTM", "STTM", "UBLK")))
        other = ", ".join(f"{op} {n}" for op, n in sorted(c.items())
                          if op in ("DFMA", "DMUL", "DADD", "FFMA", "HMMA", "SYNCS", "ELECT"))
        lines.append(f"| `{name[:110]}` | {c['_total']} | {tc or '-'} | {other or '-'} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print(f"wrote {out}: {len(counts)} kernels")


if __name__ == "__main__":
    main()
