"""Dev tool: per-kernel table from an `ncu --csv --metrics ...` launch list (no GPU needed)."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
d = collections.OrderedDict()
for r in rows[1:]:
    k = (r[h.index("ID")], r[h.index("Kernel Name")][:70], r[h.index("Grid Size")])
    d.setdefault(k, {})[r[h.index("Metric Name")]] = r[h.index("Metric Value")] + " " + r[h.index("Metric Unit")]
for k, v in d.items():
    print(k[0], k[1], k[2], " | ".join(f"{a.split('.')[0].split('__')[-1]}={b}" for a, b in v.items()))
