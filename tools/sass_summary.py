"""Per-kernel SASS instruction summary of libbfly.so (math, memory, TMA / barrier mnemonics):
python tools/sass_summary.py > profiles/r02_sass_summary.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "paper_1502_01379_b200", "libbfly.so")
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
KEEP = re.compile(r"^(DFMA|DMUL|DADD|DMMA|FFMA|HMMA|UTC|LDTM|STTM|LDS|STS|LDG|STG|UBLKCP|UTMA|SYNCS|BAR|MUFU|SHFL|LDL|STL|ATOM|RED|MEMBAR|"
                  r"ACQBULK|ERRBAR|UCGABAR)")
counts = collections.OrderedDict()
name = None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        sym = m.group(1)
        dem = subprocess.run(["c++filt", sym], capture_output=True, text=True).stdout.strip()
        mm = re.search(r"(?:bfly::)?(?:\(anonymous namespace\)::)?(\w+)\s*[<(]", dem)
        name = mm.group(1) if mm else dem
        counts.setdefault(name, collections.Counter())
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Za-z0-9_.]+)", line)
    if m and name:
        op = m.group(1)
        if KEEP.match(op):
            counts[name][op] += 1
for k, c in counts.items():
    print("==", k)
    for op, n in c.most_common(12):
        print("%7d %s" % (n, op))
