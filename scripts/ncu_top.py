"""Summarise an ncu --page source --csv dump: top stall instructions + reasons."""
import csv
import sys

path = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(open(path)))
# the file may hold several kernels (each starts with "Kernel Name"); take the first block
blocks = []
cur = None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r]
        blocks.append(cur)
    elif cur is not None:
        cur.append(r)
blk = blocks[0]
hdr = blk[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in blk[2:] if len(r) == len(hdr)]
col = "Warp Stall Sampling (All Samples)"
f = lambda r, c: float(r[idx[c]] or 0)
tot = sum(f(r, col) for r in data)
ie = sum(f(r, "Instructions Executed") for r in data)
print(blk[0][1][:100], "samples", tot, "warp-instr", ie)
for r in sorted(data, key=lambda r: -f(r, col))[:ntop]:
    print(f'{f(r, col):8.0f} {r[idx["Instructions Executed"]]:>10}  {r[idx["Source"]][:100]}')
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
sums = {h: sum(f(r, h) for r in data) for h in reasons}
print([(k, round(v / max(tot, 1), 3)) for k, v in sorted(sums.items(), key=lambda kv: -kv[1])[:8]])
