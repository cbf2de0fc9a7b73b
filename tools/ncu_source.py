"""Per-source-line hot spots from an ncu report (no GPU needed):
    python tools/ncu_source.py report.ncu-rep <kernel-regex> [top] [regions]
Aggregates executed instructions and warp-stall samples (with reasons) per CUDA source line;
`regions` = "name:file:lo-hi,..." sums lines of a file range."""
import collections
import csv
import io
import subprocess
import sys

rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
# kernel "name" or "name@i": the i-th matching launch (template variants share a base name)
kname, _, idx = kname.partition("@")
sel = ["-s", idx, "-c", "1"] if idx else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kname}", *sel,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
inst = collections.Counter()
samp = collections.Counter()
reasons = collections.defaultdict(collections.Counter)
text = {}
cur_file = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    key = (cur_file, ln)
    text[key] = r[1][:70]
    try:
        inst[key] += int(float(r[hdr.index("Instructions Executed")] or 0))
        samp[key] += int(float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0))
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                v = int(float(r[i] or 0))
                if v:
                    reasons[key][h[6:]] += v
    except (ValueError, IndexError):
        pass
tot_i = sum(inst.values()) or 1
tot_s = sum(samp.values()) or 1


def rs(c, n=3):
    t = sum(c.values()) or 1
    return " ".join(f"{k}:{100*v/t:.0f}%" for k, v in c.most_common(n))


print(f"total warp-instructions {tot_i}, stall samples {tot_s}")
allr = collections.Counter()
for c in reasons.values():
    allr.update(c)
print("all stall reasons:", rs(allr, 8))
if top:
    print("-- by stall samples")
    for k, v in samp.most_common(top):
        print(f"{100*inst[k]/tot_i:5.1f}% inst {100*v/tot_s:5.1f}% samp  {k[0]}:{k[1]}  "
              f"{text.get(k,'')[:50]:50s} [{rs(reasons[k])}]")

if len(sys.argv) > 4:
    for spec in sys.argv[4].split(","):
        name, f, rng = spec.split(":")
        lo, hi = map(int, rng.split("-"))
        keys = [k for k in inst if k[0] == f and lo <= k[1] <= hi]
        si = sum(inst[k] for k in keys)
        ss = sum(samp[k] for k in keys)
        rr = collections.Counter()
        for k in keys:
            rr.update(reasons[k])
        print(f"region {name:10s} inst {100*si/tot_i:5.1f}%  samples {100*ss/tot_s:5.1f}%  [{rs(rr, 4)}]")
