"""Per-kernel SASS evidence of the product library (cuobjdump -sass of the
sm_100a objects): TMA loads/stores (UTMALDG / UTMASTG), mbarrier operations
(SYNCS.*), tensor-core MMAs (IMMA), async copies (LDGSTS), and the
register / spill figures ptxas reported.  YIELD counts the forward-progress
yields ptxas inserted (in fnv_kernel only the out-of-line mbarrier retry
stubs should have them: one at a look-back loop head costs ~8 %, DESIGN 3.2).

  python scripts/sass_summary.py r02      -> profiles/r02_sass_summary.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_2412_15411_b200", "_build")
OPS = ["UTMALDG", "UTMASTG", "UBLKCP", "UTCIMMA", "UTCBAR", "UTMACMDFLUSH", "SYNCS.ARRIVE", "SYNCS.PHASECHK", "IMMA", "HMMA", "LDGSTS",
       "LDG", "STG", "LDS", "STS", "MUFU", "SHFL", "BAR", "YIELD"]


def demangle(name):
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except OSError:
        return name


def short(name):
    d = demangle(name).replace("(anonymous namespace)", "anon")
    d = re.sub(r"\(.*", "", d)
    return d.split("::")[-1] if "<" not in d else d[d.rfind("::", 0, d.find("<")) + 2:]


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"
    rows = []
    for obj in ("kernels.o", "engine.o", "log.o"):
        path = os.path.join(BUILD, obj)
        if not os.path.exists(path):
            continue
        text = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
        cur, counts = None, None
        for line in text.splitlines():
            m = re.search(r"Function : (\S+)", line)
            if m:
                if cur:
                    rows.append((obj, cur, counts))
                cur, counts = short(m.group(1)), collections.Counter()
                continue
            m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if m and cur:
                ins = m.group(1)
                counts["total"] += 1
                for op in OPS:
                    if ins == op or ins.startswith(op + "."):
                        counts[op] += 1
        if cur:
            rows.append((obj, cur, counts))
    out = [f"# SASS summary ({rnd})", "",
           "`cuobjdump -sass` of `paper_2412_15411_b200/_build/*.o` (sm_100a), static instruction counts per "
           "kernel (`scripts/sass_summary.py`). UTMALDG / UTMASTG = TMA tensor loads / stores, UBLKCP = bulk copies, UTCIMMA = tcgen05 integer MMA, UTCBAR = tcgen05.commit, SYNCS.* = "
           "mbarrier arrive / try-wait, IMMA = integer tensor-core MMA (mma.sync u8), YIELD = forward-progress yields ptxas inserted.", "",
           "| object | kernel | instr | " + " | ".join(OPS) + " |",
           "|---|---|---|" + "---|" * len(OPS)]
    for obj, k, c in rows:
        out.append(f"| {obj} | `{k}` | {c['total']} | " + " | ".join(str(c[o]) for o in OPS) + " |")
    dst = os.path.join(ROOT, "profiles", f"{rnd}_sass_summary.md")
    open(dst, "w").write("\n".join(out) + "\n")
    print(dst)


if __name__ == "__main__":
    main()
