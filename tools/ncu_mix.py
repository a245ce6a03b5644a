"""Executed-instruction mix per opcode from an ncu source page (SASS)."""
import collections
import csv
import subprocess
import sys

rep, kidx = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
        continue
    if r and r[0] == "Address":
        cur["hdr"] = r
        continue
    if cur is not None:
        cur["rows"].append(r)
b = blocks[kidx]
h = {k: i for i, k in enumerate(b["hdr"])}
mix = collections.Counter()
for r in b["rows"]:
    src = r[h["Source"]].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1] if " " in src else src
    op = src.split()[0] if src else "?"
    mix[op] += int(r[h["Instructions Executed"]] or 0)
tot = sum(mix.values())
print(b["name"], f"total {tot:.3e}")
for op, n in mix.most_common(40):
    print(f"{op:28s} {n:14d} {100 * n / tot:5.1f}%")
