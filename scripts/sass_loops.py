"""Backward-branch loops of a kernel in a built object with their opcode mix
(no GPU needed).  python scripts/sass_loops.py OBJ MANGLED_SUBSTR [min_len]"""
import collections, re, subprocess, sys
obj, pat = sys.argv[1], sys.argv[2]
mn = int(sys.argv[3]) if len(sys.argv) > 3 else 40
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
parts = sass.split("Function : ")
blk = next(p for p in parts if p.split("\n")[0].strip().find(pat) >= 0)
ins = []
for line in blk.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
print("function", blk.split("\n")[0].strip(), "instructions", len(ins))
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA\S*.*?(0x[0-9a-f]+)\s*$", t)
    if not m: continue
    tgt = int(m.group(1), 16)
    if tgt >= a or tgt not in addr: continue
    body = [x for _, x in ins[addr[tgt]:i + 1]]
    if len(body) < mn: continue
    ops = collections.Counter()
    for x in body:
        x = re.sub(r"^@!?U?P\w+\s+", "", x)
        ops[x.split()[0]] += 1
    fma = sum(c for o, c in ops.items() if o.split(".")[0] in ("FFMA2", "FADD2", "FMUL2"))
    print(f"loop {tgt:#x}-{a:#x}: {len(body)} instr, packed f32x2 {fma}")
    print("   " + ", ".join(f"{o} {c}" for o, c in ops.most_common(22)))
