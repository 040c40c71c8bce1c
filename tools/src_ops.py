"""Per-source-line dynamic opcode mix of an ncu report (warp instructions per
warp-cell when `cells` is given): python tools/src_ops.py rep [cells] [ops,...]"""
import collections, csv, re, subprocess, sys

rep = sys.argv[1]
cells = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
want = sys.argv[3].split(",") if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
file = None
line = None
per = collections.defaultdict(collections.Counter)
src = {}
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        file = r[1].split("/")[-1]
        continue
    if len(r) < 8:
        continue
    if r[0].isdigit():
        line = (file, int(r[0]))
        src[line] = r[1][:80]
        continue
    if r[0] == "" and r[2].startswith("0x"):
        s = re.sub(r"^@!?U?P\d+\s+", "", r[3].strip())
        op = s.split()[0].split(".")[0]
        try:
            per[line][op] += int(r[7])
        except ValueError:
            pass
tot = collections.Counter()
for l, c in per.items():
    tot.update(c)
if want:
    rows = sorted(per.items(), key=lambda kv: -sum(kv[1][o] for o in want))[:25]
    for l, c in rows:
        print(f"{sum(c[o] for o in want) / cells:8.2f}  {l[0]}:{l[1]}  {src[l]}")
else:
    rows = sorted(per.items(), key=lambda kv: -sum(kv[1].values()))[:40]
    for l, c in rows:
        top = " ".join(f"{o}:{n / cells:.1f}" for o, n in c.most_common(5))
        print(f"{sum(c.values()) / cells:8.2f}  {l[0]}:{l[1]}  {src[l][:60]}  | {top}")
