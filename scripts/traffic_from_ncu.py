"""Records the dominant kernel's DRAM traffic per launch from an ncu raw-page
CSV export into profiles/traffic.json (read by bench.py's roofline.traffic).

    python scripts/traffic_from_ncu.py <raw.csv> <workload, e.g. 800x600x1000>
"""
import csv, json, os, sys

rows = list(csv.reader(open(sys.argv[1])))
h, u, v = rows[0], rows[1], rows[2]
ix = {n: i for i, n in enumerate(h)}


def val(name):
    x = float(v[ix[name]])
    unit = u[ix[name]].lower()
    return x * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(unit, 1)


rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                   "traffic.json")
j = json.load(open(out)) if os.path.exists(out) else {}
j[sys.argv[2]] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                  "kernel": v[ix["Kernel Name"]] if "Kernel Name" in ix else "",
                  "duration_us_under_ncu": float(v[ix["gpu__time_duration.sum"]]),
                  "source": os.path.basename(sys.argv[1])}
json.dump(j, open(out, "w"), indent=1)
print(json.dumps(j[sys.argv[2]]))
