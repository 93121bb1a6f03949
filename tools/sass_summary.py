"""Per-kernel SASS instruction summary of the built library (Blackwell
evidence: tcgen05 MMAs, TMA loads, TMEM loads/stores, bulk copies, fp64 MMAs).

    python tools/sass_summary.py > profiles/r02_sass_summary.md
"""

import re
import subprocess
import sys
from collections import Counter, OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2301_03047_b200" / "libglr_b200.so"
# mnemonic families (prefix match on the opcode)
FAMILIES = OrderedDict([
    ("UTCQMMA / UTCOMMA (tcgen05.mma fp8/fp4/mxf4)", ("UTCQMMA", "UTCOMMA")),
    ("UTCIMMA (tcgen05.mma kind::i8)", ("UTCIMMA",)),
    ("UTCHMMA (tcgen05.mma kind::f16)", ("UTCHMMA",)),
    ("UTMALDG (TMA tensor load)", ("UTMALDG",)),
    ("UBLKCP (bulk copy)", ("UBLKCP",)),
    ("LDTM (tcgen05.ld)", ("LDTM",)),
    ("STTM (tcgen05.st)", ("STTM",)),
    ("UTCBAR (tcgen05.commit)", ("UTCBAR",)),
    ("DMMA (fp64 mma.sync)", ("DMMA",)),
    ("DFMA", ("DFMA",)),
    ("LDGSTS (cp.async)", ("LDGSTS",)),
    ("SYNCS (mbarrier)", ("SYNCS",)),
])


def main():
    out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    kernels = OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            op, mods = m.group(1), m.group(2) or ""
            for fam, prefixes in FAMILIES.items():
                if op.startswith(prefixes):
                    kernels[cur][fam] += 1
                    if op.startswith("UTC") and ".2CTA" in mods:
                        kernels[cur][fam + " [.2CTA]"] += 1
    demangle = {}
    try:
        names = "\n".join(kernels)
        dm = subprocess.run(["c++filt"], input=names, capture_output=True, text=True).stdout
        demangle = dict(zip(kernels, dm.splitlines()))
    except Exception:
        pass
    print("# SASS instruction summary (cuobjdump -sass of libglr_b200.so, sm_100a)\n")
    print("Static instruction counts per kernel (not executed counts); only kernels with at least")
    print("one tensor-core, TMA, TMEM, bulk-copy or fp64 instruction are listed.\n")
    print("| kernel | instructions |")
    print("|---|---|")
    for k, c in kernels.items():
        if not c:
            continue
        name = demangle.get(k, k)
        name = re.sub(r"\(.*", "", name)
        print(f"| `{name}` | " + ", ".join(f"{f} x{n}" for f, n in c.items()) + " |")


if __name__ == "__main__":
    sys.exit(main())
