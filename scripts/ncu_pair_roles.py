"""Split an ncu `--page source --print-source sass --csv` export of the
frame-pair kernel (k_chain_pair) into code regions by address: the stencil
role (from the first LDS.128 to the last SHFL-bearing loop), the IIR role
(after it), set-up and recheck code.  Prints executed warp instructions,
opcode mix, a dispatch-cycle estimate (FFMA2/FADD2/PRMT/LOP3 2 cycles, SHFL
4, the rest 1: the B200 rates of scripts/micro/pipe_rates.cu) and stall
samples per region.

    python scripts/ncu_pair_roles.py gpurun_out/pair0_sass.csv
"""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
recs = []
for r in rows[2:]:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    d = dict(zip(hdr, r))
    n = int(d["Instructions Executed"] or 0)
    op = re.sub(r"^@!?U?P\w+\s+", "", d["Source"].strip()).split()[0] if d["Source"].strip() else "?"
    st = {k: int(v) for k, v in d.items()
          if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
    recs.append((int(r[0], 16), op, n, st, d["Source"].strip()))
recs.sort()
# regions: the stencil march = the span of SHFL instructions; the IIR role =
# the span of STS.128 + UTMALDG; everything else "other"
shfl = [a for a, op, n, *_ in recs if op.startswith("SHFL") and n > 0]
sts = [a for a, op, n, *_ in recs if (op.startswith("STS.128") or op.startswith("UTMALDG")) and n > 0]
s0, s1 = min(shfl), max(shfl)
i0, i1 = min(sts), max(sts)
cost2 = ("FFMA2", "FADD2", "FMUL2", "PRMT", "LOP3", "FSEL", "SEL", "FMNMX3", "IMAD", "HFMA2")


def cyc(op, n):
    b = op.split(".")[0]
    if b == "SHFL":
        return 4 * n
    return (2 if b in cost2 else 1) * n


def region(a):
    if s0 - 0x400 <= a <= s1 + 0x200:
        return "stencil"
    if i0 - 0x200 <= a <= i1 + 0x100:
        return "iir"
    return "other"


agg = collections.defaultdict(lambda: [0, 0, collections.Counter(), collections.Counter()])
for a, op, n, st, src in recs:
    g = agg[region(a)]
    g[0] += n
    g[1] += cyc(op, n) if not op.startswith("SHFL") else n
    g[2][op.split(".")[0] if not op.startswith("IMAD") else op] += n
    g[3].update(st)
T = sum(g[0] for g in agg.values())
for k, (n, c, ops, st) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    S = sum(st.values()) or 1
    print(f"== {k}: {n:.4g} warp-instr ({100 * n / T:.1f}%), est. dispatch cycles {c:.4g}, "
          f"stall samples {S}")
    print("   ops: " + ", ".join(f"{o} {v / n * 100:.1f}%" for o, v in ops.most_common(16)))
    print("   stalls: " + ", ".join(f"{s[6:]} {v / S * 100:.1f}%" for s, v in st.most_common(9)))
