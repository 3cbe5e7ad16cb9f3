"""Summarise an ncu `--page source --print-source sass --csv` export:
executed warp-instructions per opcode and the top stall-sampled instructions."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
tot = collections.Counter(); stall = collections.Counter()
lines = []
for r in data:
    if len(r) < len(hdr): continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"): op = src.split()[1]
    try:
        n = int(r[ix["Instructions Executed"]] or 0)
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    tot[op.split(".")[0]] += n; stall[op.split(".")[0]] += s
    lines.append((s, n, r[ix["Address"]], src))
T = sum(tot.values()); S = sum(stall.values())
print(f"total warp-instr {T:.4g}  stall samples {S}")
for op, n in tot.most_common(30):
    print(f"{op:12s} {n:12d} {100*n/T:6.2f}%  stall {100*stall[op]/max(S,1):6.2f}%")
print("--- top stalled instructions")
for s, n, a, src in sorted(lines, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{s:7d} {n:11d} {a} {src[:90]}")
