"""Summarise the round's ncu captures (tools/profile_r1.sh -> gpurun_out/) into
profiles/ (tracked):

  profiles/<tag>_kernels.csv        key metrics per captured kernel
  profiles/<tag>_launch_share.csv   per-kernel device time and share of the
                                    timed region (ncu launch list, serialised)
  profiles/<tag>_launches.csv       the launch list itself (ncu --csv)
  profiles/<tag>_ncu_details_<k>.csv  ncu --page details of each kernel
  profiles/<tag>_roofline_inputs.json  DRAM bytes per launch of the advance and
                                    limiter tile pass, limiter FP64 inst per cell
                                    (read by bench.py)

usage: python tools/summarize_profiles.py [tag] [gpurun_out]
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r1"
SRC = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
OUT = os.path.join(ROOT, "profiles")
KERNELS = ["k_theta_tiled", "k_theta_hard", "k_bisect_cert", "k_bisect_unc", "k_bisect_tail",
           "k_advance_tiled",
           "k_sched", "k_w1_tile", "k_ordered_sum", "k_strong_partials"]
# units of work per launch for the per-item columns: cells of the C2 batch
# (64 x 1000 x 200) for the march tile kernels, coarse cells (2000 x 400)
# for the W1 / L1 kernels of configs[3]; the hard-path kernels get None.
ITEMS = {"k_theta_tiled": 64 * 200000, "k_advance_tiled": 64 * 200000,
         "k_w1_tile": 800000, "k_strong_partials": 800000}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    d = {}
    for n, un, val in zip(h, u, v):
        try:
            d[n] = float(val.replace(",", "")) * SCALE.get(un, 1.0)
        except ValueError:
            d[n] = val
    return d


def summarize_kernel(k):
    rep = os.path.join(SRC, f"{TAG}_{k}.ncu-rep")
    if not os.path.exists(rep):
        return None
    d = raw(rep)
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    with open(os.path.join(OUT, f"{TAG}_ncu_details_{k}.csv"), "w") as f:
        f.write(det)
    cyc = d.get("smsp__cycles_elapsed.avg", 0.0)
    fp64 = sum(d.get(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed", 0.0)
               for op in ("dadd", "dmul", "dfma")) * cyc
    ms = d.get("gpu__time_duration.sum", float("nan"))
    rd, wr = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
    items = ITEMS.get(k)
    return {
        "kernel": k, "duration_ms": round(ms, 4),
        "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size"),
        "regs": d.get("launch__registers_per_thread"),
        "dram_read_GB": round(rd / 1e9, 4), "dram_write_GB": round(wr / 1e9, 4),
        "dram_GBps": round((rd + wr) / (ms * 1e-3) / 1e9, 1),
        "issue_active_pct": round(d.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0), 1),
        "warps_active_pct": round(d.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0), 1),
        "fp64_pipe_pct": round(d.get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 0), 1),
        "threads_per_warp_inst": round(d.get("smsp__thread_inst_executed_per_inst_executed.ratio", 0), 2),
        "warp_inst": d.get("smsp__inst_executed.sum"),
        "fp64_thread_inst": round(fp64),
        "items": items,
        "fp64_inst_per_item": round(fp64 / items, 1) if items else None,
        "dram_bytes_per_item": round((rd + wr) / items, 1) if items else None,
    }


def launch_share(suffix=""):
    path = os.path.join(SRC, f"{TAG}_launches{suffix}.csv")
    if not os.path.exists(path):
        return None
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    with open(os.path.join(OUT, f"{TAG}_launches{suffix}.csv"), "w") as f:
        f.write("\n".join(lines[start:]) + "\n")
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        name = r[ki].split("(")[0].split("<")[0].split("::")[-1].replace("void ", "")
        tot[name] += float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        cnt[name] += 1
    all_ms = sum(tot.values())
    out = [{"kernel": k, "launches": cnt[k], "total_ms": round(tot[k], 3),
            "avg_ms": round(tot[k] / cnt[k], 4), "share_pct": round(100 * tot[k] / all_ms, 1)}
           for k in sorted(tot, key=lambda k: -tot[k])]
    with open(os.path.join(OUT, f"{TAG}_launch_share{suffix}.csv"), "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(out[0]))
        w.writeheader()
        w.writerows(out)
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    rows = [r for r in (summarize_kernel(k) for k in KERNELS) if r]
    if rows:
        with open(os.path.join(OUT, f"{TAG}_kernels.csv"), "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=list(rows[0]))
            w.writeheader()
            w.writerows(rows)
    share = launch_share()
    late = launch_share("_late")
    by = {r["kernel"]: r for r in rows}
    if "k_theta_tiled" in by and "k_advance_tiled" in by:
        tt, adv = by["k_theta_tiled"], by["k_advance_tiled"]
        fp = {"k_theta_tiled_fp64_inst_per_cell": tt["fp64_inst_per_item"],
              "k_theta_tiled_dram_bytes_per_launch": round(1e9 * (tt["dram_read_GB"]
                                                                  + tt["dram_write_GB"])),
              "k_advance_tiled_dram_bytes_per_launch": round(1e9 * (adv["dram_read_GB"]
                                                                    + adv["dram_write_GB"])),
              "source": f"profiles/{TAG}_kernels.csv (ncu --set full, C2 64 samples at t=5e-4, "
                        "default build)"}
        with open(os.path.join(OUT, f"{TAG}_roofline_inputs.json"), "w") as f:
            json.dump(fp, f, indent=1)
    for r in rows:
        print(r)
    for r in (share or []) + (late or []):
        print(r)


if __name__ == "__main__":
    main()
