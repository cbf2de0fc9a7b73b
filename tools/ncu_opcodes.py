"""Executed-instruction histogram by SASS opcode from an ncu report (no GPU)."""
import collections, csv, io, subprocess, sys
rep, kname = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kname}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
cnt = collections.Counter()
for r in rows:
    if r and r[0] == "Address":
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        op = r[1].strip().split()
        if not op: continue
        o = op[0]
        if o.startswith("@"): o = op[1]
        o = o.split(".")[0]
        try: cnt[o] += int(float(r[hdr.index("Instructions Executed")] or 0))
        except ValueError: pass
tot = sum(cnt.values())
print("total", tot)
for o, v in cnt.most_common(40):
    print(f"{o:12s} {v:12d} {100*v/tot:5.1f}%")
