"""Warp-stall breakdown (cycles per issued instruction) of an ncu report."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(out.splitlines()))
h, v = r[0], r[2]
st = []
for i, n in enumerate(h):
    if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
        st.append((float(v[i]), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
print(", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:8]))
