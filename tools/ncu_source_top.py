"""Top SASS instructions by warp-stall samples from an `ncu --page source --csv` export,
with each one's dominant stall reasons, plus totals per stall reason and per opcode.
Usage: python tools/ncu_source_top.py export.source.csv [top]"""
import collections
import csv
import gzip
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
op = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
rows = list(csv.reader(op))
i = 0
while i < len(rows):
    if rows[i] and rows[i][0] == "Kernel Name":
        name = rows[i][1].split("(")[0].replace("void ", "").replace("bfly::", "")
        h = rows[i + 1]
        j = i + 2
        body = []
        while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
            if len(rows[j]) >= len(h) - 2:
                body.append(rows[j])
            j += 1
        i = j
        si = h.index("# Samples")
        stall = [(c, k) for c, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
        tot = sum(int(r[si] or 0) for r in body)
        if tot == 0:
            continue
        print(f"== {name}: {tot} samples, {len(body)} instructions")
        by = collections.Counter()
        byop = collections.Counter()
        for r in body:
            for c, k in stall:
                by[k] += int(r[c] or 0)
            byop[r[1].split()[0] if not r[1].startswith("@") else r[1].split()[1]] += int(r[si] or 0)
        print("  stalls:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in by.most_common(8)))
        print("  opcodes:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in byop.most_common(10)))
        for idx, r in sorted(enumerate(body), key=lambda x: -int(x[1][si] or 0))[:top]:
            st = sorted(((int(r[c] or 0), k[6:]) for c, k in stall), reverse=True)[:2]
            print(f"  {100 * int(r[si]) / tot:5.1f}%  #{idx:5d} {r[1][:70]:70s} {st[0][1]}:{st[0][0]} {st[1][1]}:{st[1][0]}")
    else:
        i += 1
