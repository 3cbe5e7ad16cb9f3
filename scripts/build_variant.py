"""Link a variant of the product library with one kernel source recompiled
under extra -D flags (A/B experiments on the GPU box via FUSEPLAN_LIB):

    python scripts/build_variant.py libX.so kernels/fc_pipe2.cu -DFP2_NSF=2 ...
"""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04394_b200 import build as B

name, src, flags = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()
objs = [os.path.join(B.OBJ, s.replace("/", "_") + ".o") for s in B.HOST_SRCS + B.CUDA_SRCS]
var = os.path.join(B.OBJ, "variant_" + name + ".o")
cmd = [B.NVCC] + B.NVCC_FLAGS + flags + ["-c", os.path.join(B.CSRC, src), "-o", var]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
objs = [var if o.endswith(src.replace("/", "_") + ".o") else o for o in objs]
out = os.path.join(os.path.dirname(B.LIB), name)
subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-cudart", "static", "-o", out] + objs +
               ["-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"], check=True)
print(out)
