"""Per-kernel SASS opcode summary of the built engine (cuobjdump -sass): the Blackwell
instructions that prove the tcgen05 / TMEM / TMA / bulk-copy paths. Usage:
sass_summary.py [lib.so] > profiles/round2_sass_summary.md"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2210_09147_b200", "libpartime_b200.so")
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = [("UTCHMMA", "tcgen05.mma (tensor core)"), ("UTCBAR", "tcgen05.commit"), ("LDTM", "tcgen05.ld (TMEM)"),
        ("STTM", "tcgen05.st (TMEM)"), ("UTCATOMSWS", "tcgen05.alloc/dealloc"), ("UTMALDG", "TMA tensor load"),
        ("UTMASTG", "TMA tensor store"), ("UTMAPF", "TMA tensor L2 prefetch"), ("UBLKCP", "bulk copy (TMA engine)"),
        ("UBLKPF", "bulk L2 prefetch"), ("SYNCS", "mbarrier ops"), ("FFMA", "fp32 FMA"), ("LDS", "shared load"),
        ("STS", "shared store"), ("LDG", "global load"), ("STG", "global store")]
print("# SASS opcode summary (cuobjdump -sass " + os.path.basename(lib) + ", sm_100a)\n")
print("| kernel | " + " | ".join(k for k, _ in KEYS) + " |")
print("|---" * (len(KEYS) + 1) + "|")
for part in re.split(r"\n\s*Function : ", txt)[1:]:
    name = part.split("\n", 1)[0].strip()
    name = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip().split("(")[0]
    ops = collections.Counter(re.findall(r"\s([A-Z][A-Z0-9]+)(?:\.\S*)?\s", part))
    print(f"| `{name}` | " + " | ".join(str(ops.get(k, 0)) for k, _ in KEYS) + " |")
print("\n" + "; ".join(f"{k} = {v}" for k, v in KEYS))
