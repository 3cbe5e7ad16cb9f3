"""Deduplicated per-SASS-instruction rows (address order) from an ncu
`--page source --print-source cuda,sass --csv` export: executed count, the
source line, and the top stall reasons.  Usage: ncu_sass_dump.py CSV
[min_count] [first_addr last_addr]."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
mn = int(sys.argv[2]) if len(sys.argv) > 2 else 1
hdr = None; f = None; line = None; by = {}
for r in rows:
    if not r: continue
    if r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if r[0] == "Function Name" or hdr is None: continue
    if r[0].isdigit(): line = int(r[0]); continue
    if r[0] == "" and r[2].startswith("0x"):
        d = dict(zip(hdr, r))
        try: n = int(d["Instructions Executed"] or 0)
        except ValueError: continue
        st = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v)}
        a = int(r[2], 16)
        rec = (a, f, line, r[3].strip(), n, st)
        if a not in by or (f.startswith("fc_pipe") and not by[a][1].startswith("fc_pipe")): by[a] = rec
recs = sorted(by.values())
base = recs[0][0]
for a, f, l, op, n, st in recs:
    if n < mn: continue
    tops = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{a-base:6x} {n:9d} {f[:9]:9s}{l:5d}  {op[:64]:64s} " + " ".join(f"{k}:{v}" for k, v in tops))
