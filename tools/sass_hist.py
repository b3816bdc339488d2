"""SASS opcode histogram per kernel of libccq_b200.so (cuobjdump -sass; no GPU
needed): the instructions that prove the tensor-core / TMA / bulk-copy paths
(UTCHMMA, UTMALDG, LDTM/STTM, UBLKCP, HMMA, FFMA2, DFMA/DADD, ...).

  python tools/sass_hist.py [lib] > profiles/r02_sass_hist.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2507_07145_b200", "libccq_b200.so")
KEYS = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "HMMA", "FFMA2", "FFMA", "HFMA2",
        "LOP3", "PRMT", "IMAD", "DFMA", "DADD", "LDS", "STS", "LDG", "STG", "SHFL", "SYNCS", "BAR"]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
func = None
hist = collections.defaultdict(collections.Counter)
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        func = m.group(1)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and func:
        hist[func][m.group(1)] += 1


def short(name):
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    d = re.sub(r"ccqb::\(anonymous namespace\)::", "", d)
    return d[:110]


print(f"# SASS opcode counts per kernel ({os.path.basename(lib)}, sm_100a); static counts, not executed")
print("kernel," + ",".join(KEYS))
for f in sorted(hist, key=lambda n: short(n)):
    c = hist[f]
    if not any(c[k] for k in ("UTCHMMA", "HMMA", "FFMA2", "UBLKCP", "UTMALDG", "DFMA", "LOP3")):
        continue
    print(short(f).replace(",", ";") + "," + ",".join(str(c[k]) for k in KEYS))
