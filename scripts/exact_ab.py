"""A/B of library builds (FUSEPLAN_LIB per process) on the exact frame-pair
pipeline: 800x600x1000 and 192x432x600 timing, rounds interleaved."""
import os, subprocess, sys
for rnd in range(3):
    for lib in sys.argv[1:]:
        env = dict(os.environ, FUSEPLAN_VARIANT="exact",
                   FUSEPLAN_LIB=os.path.abspath(f"paper_1509_04394_b200/{lib}"))
        outs = []
        for shape in (["800", "600", "1000"], ["192", "432", "600"]):
            r = subprocess.run([sys.executable, "scripts/tile_sweep.py"] + shape, env=env,
                               capture_output=True, text=True)
            outs.append(r.stdout.strip().split(": ")[-1] if r.returncode == 0 else r.stderr[-200:])
        print(f"== {lib}: " + " | ".join(outs), flush=True)
