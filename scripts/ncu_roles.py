"""Split an ncu `--page source --print-source cuda,sass --csv` export of the
pipe kernel into warp roles by SASS address range (the role functions are
inlined into separate code regions) and sum executed instructions and stall
reasons per role."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; cur_file = None; cur_line = None
recs = []  # (addr, file, line, op, n, stalls{})
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if r[0] == "Function Name" or hdr is None: continue
    if r[0].isdigit(): cur_line = int(r[0]); continue
    if r[0] == "" and r[2].startswith("0x"):
        d = dict(zip(hdr, r))
        try: n = int(d["Instructions Executed"] or 0)
        except ValueError: continue
        st = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
        recs.append((int(r[2], 16), cur_file, cur_line, r[3].strip(), n, st))
recs.sort()
# an inlined instruction is listed under every source line of its inline
# chain: keep one record per address, preferring a fc_pipe.cu line
by = {}
for rec in recs:
    a = rec[0]
    if a not in by or (rec[1] == "fc_pipe.cu" and by[a][1] != "fc_pipe.cu"):
        by[a] = rec
recs = sorted(by.values())
# role of an address: by the source line of the role-specific code
def role(f, l):
    if f == "fc_pipe.cu":
        if 282 <= l <= 470: return "iir"
        if 593 <= l <= 850: return "stencil"
        if 540 <= l <= 580: return "exact"
        if 950 <= l <= 980: return "producer"
    return None
# propagate: helper lines inherit the role of the nearest role-tagged neighbour
tags = [role(f, l) for _, f, l, *_ in recs]
last = None
for i, t in enumerate(tags):
    if t: last = t
    else: tags[i] = ("~" + last) if last else "?"
agg = collections.defaultdict(lambda: [0, collections.Counter(), collections.Counter()])
for (a, f, l, op, n, st), t in zip(recs, tags):
    t = t.lstrip("~")
    agg[t][0] += n
    agg[t][1].update(st)
    agg[t][2][op.split()[0] if not op.startswith("@") else op.split()[1]] += n
T = sum(v[0] for v in agg.values())
for t, (n, st, ops) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    S = sum(st.values())
    print(f"== {t}: {n:.4g} warp-instr ({100*n/T:.1f}%), stall samples {S}")
    print("   ops: " + ", ".join(f"{o.split('.')[0]} {c/n*100:.1f}%" for o, c in ops.most_common(12)))
    print("   stalls: " + ", ".join(f"{k[6:]} {v/S*100:.1f}%" for k, v in st.most_common(9)))
