"""A/B of frame-pair pipeline builds (FUSEPLAN_LIB per process): parity on a
few shapes + 800x600x1000 and 2048x2048x200 timing."""
import os, sys, subprocess
libs = sys.argv[1:]
code = r'''
import os, sys
sys.path.insert(0, os.getcwd())
from scripts.pair_check import run, timeit
bad = 0
for (W, H, F) in [(800, 600, 24), (192, 432, 31), (132, 40, 9)]:
    bad += run(W, H, F, 2)[3]
bad += run(800, 600, 20, 2, th=20.0, band=64.0)[3]
ms = sorted(timeit(800, 600, 1000, 2) for _ in range(3))[1]
ms2 = timeit(2048, 2048, 200, 2)
ex = run(800, 600, 64, 2, check=False)[0]
rc = ex.describe().get("exact_rechecks_total")
print(f"mismatches {bad}  800x600x1000 {ms:.3f} ms {1e6/ms:.0f} fps  2048x2048x200 {ms2:.3f} ms {2e5/ms2:.0f} fps  rechecks(total so far) {rc}", flush=True)
'''
for rnd in range(2):
    for lib in libs:
        env = dict(os.environ, FUSEPLAN_LIB=os.path.abspath(f"paper_1509_04394_b200/{lib}"))
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(f"== {lib}: {r.stdout.strip()} {r.stderr.strip()[-300:] if r.returncode else ''}", flush=True)
