"""Opcode mix of the hottest loop of k_chain_pipe<OH, SRC_F32> from the built
object (no GPU needed): the rolled 6-step march body = the largest backward-
branch loop of the stencil role.

    python scripts/sass_body.py [OH] [0|1]
"""
import collections, re, subprocess, sys
oh = sys.argv[1] if len(sys.argv) > 1 else "15"
f32 = sys.argv[2] if len(sys.argv) > 2 else "0"
obj = ("paper_1509_04394_b200/_build/kernels_fc_pipe_cfg63.cu.o" if len(sys.argv) > 3
       else "paper_1509_04394_b200/_build/kernels_fc_pipe.cu.o")
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
ns = sys.argv[3] if len(sys.argv) > 3 else "6fcpipe"
name = f"_ZN{ns}12k_chain_pipeILi{oh}ELb{f32}EEEv14CUtensorMap_stNS_4ArgsE"
blk = sass.split("Function : " + name)[1].split("Function : ")[0]
ins = []
for line in blk.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
best = None
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA\S* (?:`\()?\.?L?_?x?_?(0x[0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in addr:
            body = [x for _, x in ins[addr[tgt]:i + 1]]
            n = i - addr[tgt] + 1
            # the march body: the smallest backward loop holding the Sobel shuffles
            if sum("SHFL.UP" in x for x in body) >= 12 and (best is None or n < best[0]):
                best = (n, addr[tgt], i)
n, lo, hi = best
mix = collections.Counter()
for _, t in ins[lo:hi + 1]:
    op = t.split()[1] if t.startswith("@") else t.split()[0]
    mix[op] += 1
print(f"{name}: {len(ins)} instructions; hottest loop {n} instructions")
print(dict(mix.most_common(30)))
