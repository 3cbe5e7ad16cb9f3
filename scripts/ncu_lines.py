"""Per-CUDA-source-line executed instructions from an ncu
`--page source --print-source sass,cuda --csv` export."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
lines = []
for r in rows:
    if r and r[0].isdigit():
        try:
            lines.append((int(r[ie] or 0), int(r[st] or 0), int(r[0]), r[1]))
        except ValueError:
            pass
T = sum(l[0] for l in lines); S = sum(l[1] for l in lines)
print(f"total warp-instr {T:.4g} stall samples {S}")
for n, s, ln, src in sorted(lines, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{ln:5d} {100*n/T:6.2f}% st {100*s/max(S,1):5.1f}% {src.strip()[:95]}")
