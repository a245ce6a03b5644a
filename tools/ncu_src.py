"""Summarise an ncu source page (SASS): top stall instructions with reasons and context."""
import csv
import subprocess
import sys

rep, kidx = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 12
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
R = b["rows"]
reasons = [k for k in b["hdr"] if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(int(r[h["Warp Stall Sampling (All Samples)"]] or 0) for r in R)
print(b["name"], "total samples", tot)
agg = {k: sum(int(r[h[k]] or 0) for r in R) for k in reasons}
print("by reason:", sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:10])
order = sorted(range(len(R)), key=lambda i: -int(R[i][h["Warp Stall Sampling (All Samples)"]] or 0))
for i in order[:topn]:
    r = R[i]
    rs = sorted(((int(r[h[k]] or 0), k[6:]) for k in reasons), reverse=True)[:3]
    print(f"{r[h['Warp Stall Sampling (All Samples)']]:>7} {rs}  @{i}: {r[h['Source']].strip()[:60]}")
    for j in range(max(0, i - 3), i):
        print(f"{'':>10} prev {R[j][h['Source']].strip()[:70]}")
