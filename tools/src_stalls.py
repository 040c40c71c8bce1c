"""Top source lines per warp-stall reason of an ncu report:
python tools/src_stalls.py rep [reason,...] [n]"""
import collections, csv, subprocess, sys

rep = sys.argv[1]
reasons = (sys.argv[2] if len(sys.argv) > 2 else "long_sb,barrier,wait,short_sb").split(",")
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr = None
file = None
agg = collections.defaultdict(collections.Counter)
src = {}
total = 0
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ix = {name: i for i, name in enumerate(hdr)}
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    line = (file, int(r[0]))
    src[line] = r[1][:80]
    try:
        total += int(r[ix["# Samples"]])
        for c in reasons:
            agg[c][line] += int(r[ix["stall_" + c]])
    except (ValueError, KeyError):
        pass
print("samples", total)
for c in reasons:
    print(f"== {c}: {sum(agg[c].values())} ({100.0 * sum(agg[c].values()) / max(total, 1):.1f} %)")
    for l, k in agg[c].most_common(n):
        print(f"  {k:7d}  {l[0]}:{l[1]}  {src[l]}")
