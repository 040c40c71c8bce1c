"""Source-line hot spots (warp stall samples) of an ncu report:
python tools/src_hot.py rep [n]"""
import csv, subprocess, sys, collections
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
file = None
agg = collections.Counter(); src = {}; inst = collections.Counter()
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        file = r[1].split("/")[-1]
        continue
    if len(r) > 7 and r[0].isdigit():
        key = (file, int(r[0]))
        try:
            agg[key] += float(r[4]); inst[key] += float(r[7])
        except ValueError:
            pass
        src[key] = r[1][:90]
tot = sum(agg.values()) or 1
ti = sum(inst.values()) or 1
for k, v in agg.most_common(n):
    print(f"{v / tot * 100:5.1f}% stall {inst[k] / ti * 100:5.1f}% inst  {k[0]}:{k[1]}  {src[k]}")
