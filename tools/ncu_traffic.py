"""Write profiles/ncu_traffic.json from an `ncu --set full` report of one forward + inverse
call (tools/prof_once.py): DRAM bytes (read + write) summed over the kernels of each C-ABI
call, which bench.py reports as roofline.traffic.  Dev tool, no GPU needed:
    python tools/ncu_traffic.py report.ncu-rep cfg4 profiles/ncu_traffic.json"""
import csv, io, json, subprocess, sys

rep, cfg, out = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot = {"slicq_forward": 0.0, "slicq_inverse": 0.0}
kern = {"slicq_forward": [], "slicq_inverse": []}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    d = "slicq_forward" if ("fwd_" in name) else "slicq_inverse" if ("inv_" in name) else None
    if d is None:
        continue
    b = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(m)
        b += float(r[i]) * scale[units[i]]
    tot[d] += b
    kern[d].append(name.split("(")[0])
try:
    data = json.load(open(out))
except (OSError, ValueError):
    data = {}
data[cfg] = {k: int(v) for k, v in tot.items()}
data[cfg]["_source"] = (f"{rep.split('/')[-1]}: ncu --set full, dram__bytes_read.sum + "
                        "dram__bytes_write.sum per kernel, summed over the kernels of each C-ABI "
                        f"call ({', '.join(kern['slicq_forward'] + kern['slicq_inverse'])})")
json.dump(data, open(out, "w"), indent=1)
print(json.dumps(data[cfg], indent=1))
