"""Summarise an `ncu --page source --csv --print-source sass` dump: executed
warp-instructions and stall samples per basic-block-ish region (split at
branch targets), top regions first.  python tools/ncu_hot.py src.csv [kernel_idx]"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
kidx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
# split into kernels
kernels, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        kernels.append(cur)
    elif cur is not None and r and r[0].startswith("0x"):
        cur["rows"].append(r)
    elif cur is not None and r and r[0] == "Address":
        cur["hdr"] = r
k = kernels[kidx]
h = k["hdr"]
ie = h.index("Instructions Executed")
ss = h.index("Warp Stall Sampling (All Samples)")
ins = [(int(r[0], 16), r[1].strip(), int(r[ie] or 0), int(r[ss] or 0)) for r in k["rows"]]
base = ins[0][0]
targets = set()
for a, s, _, _ in ins:
    m = re.search(r"BRA\S*\s+(?:\S+, )?0x([0-9a-f]+)", s)
    if m:
        targets.add(int(m.group(1), 16))
regions, start = [], 0
for i, (a, s, _, _) in enumerate(ins):
    if i > start and (a in targets or a - base in targets):
        regions.append((start, i))
        start = i
regions.append((start, len(ins)))
tot_i = sum(x[2] for x in ins)
tot_s = sum(x[3] for x in ins)
print(k["name"][:100], "total warp-instr", tot_i, "stall samples", tot_s)
stats = []
for s0, s1 in regions:
    body = ins[s0:s1]
    n = sum(x[2] for x in body)
    st = sum(x[3] for x in body)
    stats.append((n, st, body[0][0] - base, body[-1][0] - base, len(body)))
for n, st, a0, a1, L in sorted(stats, reverse=True)[:25]:
    print(f"  {a0:#07x}-{a1:#07x} len {L:4d}  instr {n / tot_i * 100:5.1f}%  stalls {st / max(tot_s, 1) * 100:5.1f}%")
