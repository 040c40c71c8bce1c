#!/usr/bin/env python
"""bench.py — the VLBM hot path on B200, one JSON line on rank 0.

Workload (N=1): BASELINE.json configs[1], the Mach-2000 jet at 1000x200 with
M=64 Monte-Carlo samples per GPU (weak scaling: rank r marches samples
r*64 .. r*64+63, no data-path collective).  One bench "step" = one VLBM time
step of every sample of the batch (each sample with its own adaptive dt, as
run_sample marches it).  Metric: sample-cell updates/s (whole job).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Timing: W untimed steps, then EXACTLY K steps bracketed by barrier +
synchronize, CUDA events on the library's stream, max over ranks.  The state
(64 x 20 planes x 200k cells x 8 B x 2 buffers = 4.1 GB) is far larger than
L2 (126 MB): "inputs larger than L2".

Extra keys: e2e (the same march through the public API from host buffers,
H2D of the initial fields and D2H of the final fields inside the timed
region), roofline (dominant kernel, live CUDA events), cpu_baseline (the
reference CPU path on this host), clocks (nvidia-smi during the timed
region), postproc (W1/L1 on BASELINE configs[3]'s synthetic ensembles).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NX, NY, M_PER_GPU = 1000, 200, 64
BYTES_PER_UPDATE = 320      # read u(4)+pops(16) f64, write the same
THETA_BYTES_PER_CELL = 168  # k_theta_tiled: read u + pops (160 B), write theta (8 B)
# FP64 peak of the non-tensor pipe, counting DADD/DMUL/DFMA as one
# instruction (the march is built with --fmad=false): measured by
# tools/fp64_peak.cu (profiles/fp64_peak.json, DADD/DMUL/DFMA instructions/s,
# the best of the three); fallback 148 SMs x 64 FP64 lanes x 1.965 GHz.
FP64_PEAK_THEORY = 148 * 64 * 1.965e9 / 1e12


def fp64_peak():
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            d = json.load(f)
        return max(d["dadd_per_s"], d["dmul_per_s"], d["dfma_per_s"]) / 1e12, "measured"
    except Exception:
        return FP64_PEAK_THEORY, "theoretical"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.rows = []  # (arrival time, fields)
        self.proc = None
        self.t0 = self.t1 = None

    def begin(self):
        """The timed region starts (the sampler itself is started earlier, under
        the untimed run_to / warm-up load, so that nvidia-smi is already
        streaming: a 20-step region lasts 60 ms, less than its start-up)."""
        self.t0 = time.monotonic()

    def end(self):
        self.t1 = time.monotonic()

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append((time.monotonic(), parts))

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        # the samples of the timed region; the sampling period is 100 ms, so a
        # short region also takes the samples within 150 ms of it (the GPU
        # runs the same kernels, warm-up steps, right before it)
        rows = [r for t, r in self.rows
                if self.t0 is None or (self.t0 - 0.15 <= t <= (self.t1 or t) + 0.15)]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({n for r in rows for n, v in zip(self.NAMES, r[2:])
                          if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def fp64_profile():
    """Per-launch DRAM bytes of the advance and limiter kernels and the
    limiter's FP64 instructions per cell, from the committed ncu capture
    (profiles/r<N>_roofline_inputs.json, the latest round's:
    tools/profile_round.sh + summarize_profiles.py)."""
    for tag in ("r2", "r1"):
        try:
            with open(os.path.join(ROOT, "profiles", f"{tag}_roofline_inputs.json")) as f:
                d = json.load(f)
            d["source"] = f"profiles/{tag}_kernels.csv"
            return d
        except Exception:
            continue
    return None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_reference(args, n_gpus, threads=None, seconds=None, max_steps=None):
    """The reference CPU march (oracle/_ref = the unmodified reference
    headers) on this host's cores, one sample per thread (run_ensemble's
    worker pool minus file I/O), on the SAME window the GPU arm times: every
    sample marched untimed to --t-start with run_sample's loop, then a bounded
    number of steps timed (about `seconds` of CPU work)."""
    seconds = seconds or getattr(args, "ref_seconds", 15.0)
    from oracle import oracle
    threads = threads or os.cpu_count() or 1
    kind = "reference" if oracle.available("ref") else "port"
    o = oracle.Oracle("ref" if kind == "reference" else "vo")
    g, p, pp = oracle.make_grid(NX, NY), oracle.make_params(), oracle.make_pert()
    n_samples = min(args.samples, threads)
    # ~2e6 updates/s per core mid-run (survey: 1.3-1.4e6 averaged to t = 0.003)
    steps = max(2, int(seconds * 2.0e6 / (NX * NY)))
    if max_steps:
        steps = max(2, min(steps, max_steps))
    pre = 0.0
    if kind == "reference":
        sec, upd, pre = o.march_window(g, p, pp, 42, 0, n_samples, args.t_start, steps, 0.02,
                                       threads)
    else:  # the C restatement (only when the reference could not be built)
        import concurrent.futures as cf

        def one(m):
            s = o.jet_sim(g, p, pp, 42, m)
            while s.time < args.t_start - 1e-12:
                s.step(min(s.suggest_dt(), args.t_start - s.time))
            return s

        with cf.ThreadPoolExecutor(threads) as ex:
            sims = list(ex.map(one, range(n_samples)))

        def run(s):
            for _ in range(steps):
                s.step(s.suggest_dt())
            return steps * NX * NY

        t0 = time.perf_counter()
        with cf.ThreadPoolExecutor(threads) as ex:
            upd = sum(ex.map(run, sims))
        sec = time.perf_counter() - t0
    used = min(threads, n_samples)
    return {"value": upd / sec, "unit": "sample-cell-updates/s", "cores": used, "kind": kind,
            "cpu_model": cpu_model(), "host_threads": os.cpu_count(),
            "sample": f"{n_samples} jet samples at {NX}x{NY}, each marched untimed to "
                      f"t={args.t_start:g} ({pre:.0f} s), then {steps} timed steps "
                      f"({upd:.3g} updates, {sec:.1f} s wall, {used} threads)"}


def postproc_cpu_baseline(M=1000, nxc=2000, rows=2):
    """The reference's restrict_field + wasserstein1 + strong_error
    (compute_metrics' calls, single-threaded as the reference runs them) on a
    configs[3] slice: `rows` coarse rows of 2000x400 (and the 2*rows fine rows
    of 4000x800), M = 1000 log-normal density samples (other components 0)."""
    import numpy as np
    from oracle import oracle
    if not oracle.available("ref"):
        return None
    rng = np.random.default_rng(3)
    coarse = np.zeros((M, 4, rows, nxc))
    fine = np.zeros((M, 4, 2 * rows, 2 * nxc))
    coarse[:, 0] = rng.lognormal(-0.125, 0.5, size=(M, rows, nxc))
    fine[:, 0] = rng.lognormal(-0.125, 0.5, size=(M, 2 * rows, 2 * nxc))
    sec, w1, es = oracle.Oracle("ref").postproc_timed(coarse, fine)
    nc = rows * nxc
    return {"value": nc / sec, "unit": "coarse cells/s (W1 + L1 + restriction, M=1000)",
            "cores": 1, "kind": "reference", "cpu_model": cpu_model(),
            "sample": f"{rows} coarse rows x {nxc} ({nc} cells), M={M}: restrict_field of "
                      f"the fine ensemble + wasserstein1 + strong_error in {sec:.2f} s"}


def postproc_bench(torch, dev, M=1000, nxc=2000, nyc=400, reps=3):
    """BASELINE configs[3]: W1 + L1 of M synthetic log-normal density
    ensembles (mu = -sigma^2/2, sigma = 0.5, so E[rho] = 1), coarse
    nxc x nyc vs the restriction of fine 2nxc x 2nyc, on device.  Other
    components are identically zero, so the density-only L1 equals the
    reference's 4-component strong_error bit-for-bit."""
    from paper_2605_25282_b200 import post
    nc, nf = nxc * nyc, 4 * nxc * nyc
    need = 8 * M * (nc + nf) + (1 << 30)
    free, _ = torch.cuda.mem_get_info(dev)
    if need > free:
        M = max(32, int(M * free / need) // 32 * 32)
    gen = torch.Generator(device=f"cuda:{dev}")
    coarse = torch.empty((M, nyc, nxc), dtype=torch.float64, device=f"cuda:{dev}")
    fine = torch.empty((M, 2 * nyc, 2 * nxc), dtype=torch.float64, device=f"cuda:{dev}")
    gen.manual_seed(1)
    coarse.normal_(-0.125, 0.5, generator=gen).exp_()
    gen.manual_seed(2)
    fine.normal_(-0.125, 0.5, generator=gen).exp_()
    terms = torch.empty(nc, dtype=torch.float64, device=coarse.device)
    res = torch.empty(1, dtype=torch.float64, device=coarse.device)
    part = torch.empty((M, 10), dtype=torch.float64, device=coarse.device)
    post.w1_cell_terms(torch, coarse, fine, terms)
    post.ordered_mean(torch, terms, res)
    post.strong_partials(torch, coarse, fine, part)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    w1_ms, mean_ms, l1_ms = [], [], []
    for _ in range(reps):
        ev[0].record()
        post.w1_cell_terms(torch, coarse, fine, terms)
        ev[1].record()
        post.ordered_mean(torch, terms, res)
        ev[2].record()
        post.strong_partials(torch, coarse, fine, part)
        ev[3].record()
        torch.cuda.synchronize()
        w1_ms.append(ev[0].elapsed_time(ev[1]))
        mean_ms.append(ev[1].elapsed_time(ev[2]))
        l1_ms.append(ev[2].elapsed_time(ev[3]))
    w1 = float(res.item())
    es = post.strong_finish(part.cpu().numpy())
    # the production call: terms and the storage-order mean overlapped
    wm = torch.empty(2, dtype=torch.float64, device=coarse.device)
    post.w1_mean(torch, coarse, fine, wm, terms)
    fused_ms = []
    for _ in range(reps):
        ev[0].record()
        post.w1_mean(torch, coarse, fine, wm, terms)
        ev[1].record()
        torch.cuda.synchronize()
        fused_ms.append(ev[0].elapsed_time(ev[1]))
    assert float(wm[0].item()) == w1, "overlapped W1 differs from terms + ordered mean"
    w1t = statistics.median(fused_ms)
    l1t = statistics.median(l1_ms)
    hbm, src = peaks()
    w1_bytes = 40.0 * M * nc  # M coarse + 4M fine values per coarse cell
    l1_bytes = 40.0 * M * nc
    del coarse, fine
    torch.cuda.empty_cache()
    return {
        "workload": f"C4 synthetic log-normal rho, M={M}, coarse {nxc}x{nyc} vs restricted "
                    f"fine {2 * nxc}x{2 * nyc}",
        "w1_cells_per_s": nc / (w1t * 1e-3), "w1_ms": w1t,
        "w1_kernel_ms": statistics.median(w1_ms), "ordered_mean_ms": statistics.median(mean_ms),
        "w1_note": "w1_ms: vlbm_d_w1_restrict_mean (the mean overlapped with the terms); "
                   "w1_kernel_ms + ordered_mean_ms: the two phases run back to back",
        "w1_values_sorted_per_s": 2 * M * nc / (statistics.median(w1_ms) * 1e-3),
        "w1_roofline": {"bound": "hbm", "achieved": w1_bytes / (statistics.median(w1_ms) * 1e-3)
                        / 1e9, "peak": hbm, "unit": "GB/s",
                        "frac": w1_bytes / (statistics.median(w1_ms) * 1e-3) / 1e9 / hbm,
                        "bytes_per_cell": 40 * M, "peak_source": src},
        "l1_sample_cells_per_s": M * nc / (l1t * 1e-3), "l1_ms": l1t,
        "l1_roofline_frac": l1_bytes / (l1t * 1e-3) / 1e9 / hbm,
        "W1": w1, "E_strong": es,
    }


def postproc_bench_dist(torch, dist, dev, ws, rank, M=1000, nxc=2000, nyc=400, reps=3):
    """BASELINE configs[3] sharded over the ranks: rank r holds
    its contiguous share of the M synthetic sample pairs (log-normal density,
    seeded per rank), restricts its fine samples locally, then
    distributed_wasserstein1 re-shards both ensembles by cell with one NCCL
    all_to_all each, computes the per-cell terms of its cell range and gathers
    them to rank 0 in storage order for the sequential mean.  Timed with CUDA
    events on each rank (max over ranks) around the whole sharded W1."""
    from paper_2605_25282_b200 import dist as vd
    from paper_2605_25282_b200 import vlbm as v
    s0, m_loc = vd.shard_range(M, ws, rank)
    nc = nxc * nyc
    d = f"cuda:{dev}"
    gen = torch.Generator(device=d)
    coarse = torch.empty((m_loc, nc), dtype=torch.float64, device=d)
    fine = torch.empty((m_loc, 4 * nc), dtype=torch.float64, device=d)
    gen.manual_seed(1000 + 2 * rank)
    coarse.normal_(-0.125, 0.5, generator=gen).exp_()
    gen.manual_seed(1001 + 2 * rank)
    fine.normal_(-0.125, 0.5, generator=gen).exp_()
    restricted = torch.empty((m_loc, nc), dtype=torch.float64, device=d)
    valid = torch.ones(m_loc, dtype=torch.bool, device=d)
    stream = torch.cuda.current_stream(dev).cuda_stream

    def once():
        for m in range(m_loc):  # one density plane per sample (var 0 of a 1-plane field)
            v._check(v.lib().vlbm_d_restrict_var(1, nxc, nyc, fine[m].data_ptr(), 0,
                                                 restricted[m].data_ptr(), stream))
        return vd.distributed_wasserstein1(torch, dist, coarse, restricted, valid)

    host = dist.get_backend() == "gloo"

    def timed(fn):
        fn()
        ts = []
        for _ in range(reps):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = fn()
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64,
                             device="cpu" if host else d)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ts.append(float(t.item()))
        return r, statistics.median(ts)

    out = {"workload": f"C4 synthetic log-normal rho, M={M} sharded over {ws} ranks, coarse "
                       f"{nxc}x{nyc} vs restricted fine {2 * nxc}x{2 * nyc}; restriction + "
                       "2 NCCL all_to_all + per-cell terms + ordered gather + sequential mean",
           "n_gpus": ws}
    w1 = None
    try:
        w1, ms = timed(once)
        out.update({"w1_cells_per_s": nc / (ms * 1e-3), "w1_ms": ms, "W1": w1})
    except Exception as exc:  # e.g. all_to_all on a gloo group of ranks sharing a GPU
        out["error"] = f"{type(exc).__name__}: {exc}"
    # the fused alternative: no re-shard, each rank's kernel reads the other
    # ranks' planes through CUDA-IPC peer mappings (NVLink) while it sorts
    try:
        w1p, msp = timed(lambda: vd.peer_wasserstein1(torch, dist, coarse, fine, valid, nxc))
        out["peer"] = {"how": "vlbm_d_w1_rows over CUDA-IPC peer mappings (no all_to_all)",
                       "w1_cells_per_s": nc / (msp * 1e-3), "w1_ms": msp, "W1": w1p,
                       "identical": (w1p == w1) if rank == 0 and w1 is not None else None}
    except Exception as exc:
        out["peer"] = {"error": f"{type(exc).__name__}: {exc}"}
    return out


METRIC = "VLBM sample-cell updates/s (GLUPS) & % HBM roofline; W1 post-proc cells/s"


def workload_config(args, M, ws):
    """The config object of both arms (same workload, metric and unit)."""
    return {"workload": f"{'C2 ' if (NX, NY) == (1000, 200) else ''}jet {NX}x{NY}, "
                        f"M={M}/GPU, RLMP, fp64, {args.steps} steps of each sample "
                        f"after run_to(t={args.t_start:g}) + {args.warmup} warm-up steps",
            "t_start": args.t_start,
            "nx": NX, "ny": NY, "samples_per_gpu": M, "parallelism": f"samples/{ws}",
            "l2": f"inputs larger than L2 ({2 * 20 * 8 * M * NX * NY / 1e9:.1f} GB "
                  "state per GPU)"}


def run_reference_arm(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    cb = cpu_reference(args, ws, max_steps=args.steps)
    line = {"impl": "reference", "metric": METRIC,
            "value": cb["value"], "unit": "sample-cell-updates/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (jet IC from splitmix64 seeds, base_seed 42)",
            "config": workload_config(args, args.samples, args.gpus),
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "sample-cell-updates/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(args) -> int:
    """--gpus N without a launcher: re-run this script under
    torch.distributed.run with N ranks on this node (rank r on cuda:r,
    rendezvous on 127.0.0.1); rank 0 prints the line.  On a box with fewer
    GPUs than N (a test of the multi-rank path) the ranks share the GPUs
    round-robin over gloo, and the line says so."""
    env = dict(os.environ)
    try:
        import torch
        ngpu = torch.cuda.device_count()
    except Exception:
        ngpu = 0
    if ngpu < args.gpus:
        env.setdefault("VLBM_BENCH_BACKEND", "gloo")
        print(f"bench.py: {args.gpus} ranks on {ngpu} GPU(s): ranks share GPUs, backend "
              f"{env['VLBM_BENCH_BACKEND']}", file=sys.stderr)
    env.setdefault("NCCL_DEBUG", "INFO")  # NCCL's init lines (ranks, transports) on stderr
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # default window: 200 steps of every sample from t = 0.0005, the middle
    # of configs[1]'s run to t = 0.001 (the limiter's work grows with time, so
    # the first steps would overstate the run's rate)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--samples", type=int, default=M_PER_GPU)
    ap.add_argument("--t-start", type=float, default=0.0005,
                    help="march every sample to this time (untimed, run_sample's loop) "
                         "before the warmup")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-postproc", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-late", action="store_true",
                    help="skip the late-time window (t >= 0.002) measurement")
    ap.add_argument("--late-steps", type=int, default=200)
    ap.add_argument("--grid", default=None,
                    help="NXxNY instead of configs[1]'s 1000x200 (e.g. 4000x800 = configs[2])")
    ap.add_argument("--no-roofline", action="store_true",
                    help="omit the roofline objects")
    ap.add_argument("--ref-seconds", type=float, default=15.0,
                    help="target CPU seconds of the reference-CPU sample")
    ap.add_argument("--no-first-order", action="store_true",
                    help="skip the theta = 0 (Limiter::FirstOrder) march line")
    args = ap.parse_args()
    global NX, NY
    if args.grid:
        NX, NY = (int(x) for x in args.grid.lower().split("x"))
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)

    import numpy as np
    import torch

    ws, rank, local = dist_env()
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
        return 2
    # one GPU per rank; on a box with fewer GPUs than ranks (a test of the
    # multi-rank path only) ranks share them round-robin
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        backend = os.environ.get("VLBM_BENCH_BACKEND", "nccl")  # gloo: ranks sharing a GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import paper_2605_25282_b200 as v

    M = args.samples
    g = v.Grid(NX, NY)
    lat, gas, pp = v.LatticeParams(), v.GasParams(), v.PerturbationParams()

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def _reduce(x, op):  # device tensors on NCCL, host tensors on gloo
        dv = "cpu" if torch.distributed.get_backend() == "gloo" else "cuda"
        t = torch.tensor([float(x)], device=dv, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=op)
        return float(t.item())

    def reduce_max(x):
        return _reduce(x, torch.distributed.ReduceOp.MAX)

    def reduce_sum(x):
        return _reduce(x, torch.distributed.ReduceOp.SUM)

    # ---- device-resident march ----
    sim = v.BatchSimulation.jet(g, lat, gas, pp, base_seed=42, m0=rank * M, n_samples=M,
                                device=local)
    stream = torch.cuda.ExternalStream(sim.stream(), device=torch.device("cuda", local))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:  # started under the untimed load, see begin()
        if args.t_start > 0:
            sim.run_to(args.t_start)
        sim.step(args.warmup)
        sim.set_timing(True)
        st0 = sim.stats()
        barrier()
        torch.cuda.synchronize()
        clk.begin()
        ev0.record(stream)
        torch.cuda.nvtx.range_push("timed")  # ncu --nvtx-include timed/ (tools/kprof.sh)
        sim.step(args.steps)
        torch.cuda.nvtx.range_pop()
        ev1.record(stream)
        torch.cuda.synchronize()
        clk.end()
    barrier()
    ms = ev0.elapsed_time(ev1)
    st1 = sim.stats()
    updates = st1["cell_updates"] - st0["cell_updates"]
    launches = st1["launches"] - st0["launches"]
    # per-kernel device times of the timed region: CUDA events around each
    # launch on the library stream (one sample group: kernels never overlap)
    kern = {k: (st1[k] - st0[k]) / args.steps for k in
            ("ms_theta_tiles", "ms_theta_hard", "ms_advance", "ms_sched")}
    t_max = ms
    upd_total = updates
    if ws > 1:
        t_max = reduce_max(ms)
        upd_total = reduce_sum(updates)
    value = upd_total / (t_max * 1e-3)
    sim.close()

    # ---- e2e through the public API from host buffers ----
    e2e = None
    if not args.no_e2e:
        # The user's call sequence, all inside the timed region: build the
        # batch from the seeds (host inlet rows through the reference's libm,
        # H2D of the rows, initial field laid out on the device), run_sample's
        # loop to t_start, the warm-up and timed steps, then every sample's
        # final field read back into pinned host memory.  Every cell update of
        # the call counts (the early steps included).
        out = torch.empty((M, 4, NY, NX), dtype=torch.float64).pin_memory().numpy()
        barrier()
        t0 = time.perf_counter()
        e = v.BatchSimulation.jet(g, lat, gas, pp, base_seed=42, m0=rank * M, n_samples=M,
                                  device=local)
        if args.t_start > 0:
            e.run_to(args.t_start)
        e.step(args.warmup + args.steps)
        v.vlbm._check(v.lib().vlbm_batch_get_fields(e._h, v.vlbm._dp(out)))
        t1 = time.perf_counter()
        barrier()
        st = e.stats()
        e.close()
        et = t1 - t0
        upd_e = st["cell_updates"]
        if ws > 1:
            et, upd_e = reduce_max(et), reduce_sum(upd_e)
        steps_e = st["cell_updates"] / (M * NX * NY)  # per-sample steps (mean) of the call
        h2d = M * (4 * NY * 8 + 10 * 2 * 8) + 4 * NY  # inlet rows + mode coefficients, counts
        e2e = {"value": upd_e / et, "unit": "sample-cell-updates/s",
               "h2d_bytes_per_step": int(h2d / steps_e),
               "d2h_bytes_per_step": int(out.nbytes / steps_e),
               "seconds": et, "steps_per_sample": steps_e,
               "note": "BatchSimulation.jet (IC) + run_to(t_start) + warmup + K steps + D2H of "
                       "every final field, wall clock; all cell updates of the call"}

    # ---- late-time window: the same march timed from t = 0.002, where the
    # jet is developed and ~28 % of the cells are limiter hard cells (the
    # regime of most of configs[2]'s run to t = 0.003) ----
    late = None
    if not args.no_late and args.t_start < 0.002:
        lt = v.BatchSimulation.jet(g, lat, gas, pp, base_seed=42, m0=rank * M, n_samples=M,
                                   device=local)
        lt.run_to(0.002)
        lt.step(args.warmup)
        lt.set_timing(True)
        l0 = lt.stats()
        barrier()
        lstream = torch.cuda.ExternalStream(lt.stream(), device=torch.device("cuda", local))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(lstream)
        lt.step(args.late_steps)
        e1.record(lstream)
        torch.cuda.synchronize()
        barrier()
        l1 = lt.stats()
        lms = e0.elapsed_time(e1)
        lupd = l1["cell_updates"] - l0["cell_updates"]
        if ws > 1:
            lms, lupd = reduce_max(lms), reduce_sum(lupd)
        t_end = float(lt.scalars()[0].min())
        lt.close()
        late = {"value": lupd / (lms * 1e-3), "unit": "sample-cell-updates/s",
                "steps": args.late_steps, "t_start": 0.002, "t_end_min": t_end,
                "ms_per_step": lms / args.late_steps,
                "kernel_ms_per_step": {k: (l1[k] - l0[k]) / args.late_steps for k in
                                       ("ms_theta_tiles", "ms_theta_hard", "ms_advance",
                                        "ms_sched")}}

    # ---- theta = 0 (Limiter::FirstOrder, lattice.hpp:10, solver.hpp:492-495):
    # the same march without the limiter -- the collide+stream kernel alone,
    # the HBM-roofline demonstration of BASELINE.md §3 ----
    fo_line = None
    if not args.no_first_order:
        lat0 = v.LatticeParams(limiter=v.Limiter.FirstOrder)
        f0 = v.BatchSimulation.jet(g, lat0, gas, pp, base_seed=42, m0=rank * M, n_samples=M,
                                   device=local)
        if args.t_start > 0:
            f0.run_to(args.t_start)
        f0.step(args.warmup)
        f0.set_timing(True)
        a0 = f0.stats()
        barrier()
        fstream = torch.cuda.ExternalStream(f0.stream(), device=torch.device("cuda", local))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(fstream)
        f0.step(args.steps)
        e1.record(fstream)
        torch.cuda.synchronize()
        barrier()
        a1 = f0.stats()
        f0.close()
        fms = e0.elapsed_time(e1)
        fupd = a1["cell_updates"] - a0["cell_updates"]
        adv_ms = (a1["ms_advance"] - a0["ms_advance"]) / args.steps
        if ws > 1:
            fms, fupd = reduce_max(fms), reduce_sum(fupd)
        hbm0, src0 = peaks()
        adv_gbs = BYTES_PER_UPDATE * M * NX * NY / (adv_ms * 1e-3) / 1e9
        fo_line = {"value": fupd / (fms * 1e-3), "unit": "sample-cell-updates/s",
                   "limiter": "FirstOrder (theta = 0)", "steps": args.steps,
                   "ms_per_step": fms / args.steps, "advance_ms": adv_ms,
                   "roofline": {"bound": "hbm", "kernel": "k_advance_tiled<1> (collide+stream)",
                                "achieved": adv_gbs, "peak": hbm0, "unit": "GB/s",
                                "frac": adv_gbs / hbm0, "peak_source": src0,
                                "bytes_per_cell": BYTES_PER_UPDATE},
                   "step_frac": BYTES_PER_UPDATE * fupd / (fms * 1e-3) / 1e9 / hbm0}

    # ---- post-processing (BASELINE configs[3]) ----
    post = None
    if not args.no_postproc and ws == 1:
        post = postproc_bench(torch, local)
    elif not args.no_postproc:
        try:
            post = postproc_bench_dist(torch, torch.distributed, local, ws, rank)
        except Exception as exc:  # the march line still stands
            post = {"error": f"{type(exc).__name__}: {exc}"}

    if rank == 0:
        hbm, src = peaks()
        cells_per_launch = M * NX * NY
        step_gbs = BYTES_PER_UPDATE * (updates / (ms * 1e-3)) / 1e9
        roof, fp64 = None, None
        if not args.no_roofline:
            # the committed ncu figures were captured on the default workload only
            prof = (fp64_profile() or {}) if (NX, NY, M) == (1000, 200, M_PER_GPU) else {}
            # The collide+stream kernel (BASELINE north_star: "roofline = bytes
            # moved per cell update / HBM BW"): 320 B algorithmic per cell.
            t_adv = kern["ms_advance"] * 1e-3
            adv_gbs = BYTES_PER_UPDATE * cells_per_launch / t_adv / 1e9
            roof = {"bound": "hbm", "kernel": "k_advance_tiled (collide+stream)",
                    "achieved": adv_gbs, "peak": hbm, "unit": "GB/s", "frac": adv_gbs / hbm,
                    "traffic": prof.get("k_advance_tiled_dram_bytes_per_launch"),
                    "peak_source": src, "bytes_per_cell": BYTES_PER_UPDATE,
                    "cells_per_launch": cells_per_launch, "launch_ms": kern["ms_advance"],
                    "note": "per-launch times: CUDA events around each launch in the timed "
                            f"region; traffic from {prof.get('source', 'profiles/')} (ncu --set full)"}
            # The limiter's tile pass, the longest kernel of the step: FP64-bound.
            t_tiles = kern["ms_theta_tiles"] * 1e-3
            lim_gbs = THETA_BYTES_PER_CELL * cells_per_launch / t_tiles / 1e9
            ops = prof.get("k_theta_tiled_fp64_inst_per_cell")
            fp64 = {"kernel": "k_theta_tiled (RLMP limiter tile pass)",
                    "launch_ms": kern["ms_theta_tiles"],
                    "hbm": {"achieved": lim_gbs, "peak": hbm, "unit": "GB/s",
                            "frac": lim_gbs / hbm, "bytes_per_cell": THETA_BYTES_PER_CELL,
                            "traffic": prof.get("k_theta_tiled_dram_bytes_per_launch")},
                    "source": prof.get("source")}
            if ops:
                rate = ops * cells_per_launch / t_tiles / 1e12
                fpk, fsrc = fp64_peak()
                fp64.update({"achieved": rate, "peak": fpk, "unit": "Tinst/s",
                             "frac": rate / fpk, "peak_source": fsrc,
                             "fp64_inst_per_cell": ops})
        line = {
            "metric": METRIC,
            "value": value, "unit": "sample-cell-updates/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (jet IC from splitmix64 seeds, base_seed 42)",
            "config": workload_config(args, M, ws),
            "glups": value / 1e9,
            "gpu_launches": launches,
            "roofline": roof,
            "limiter_roofline": fp64,
            "step_roofline": {"achieved": step_gbs, "peak": hbm, "unit": "GB/s",
                              "frac": step_gbs / hbm, "bytes_per_update": BYTES_PER_UPDATE},
            "kernel_ms_per_step": dict(kern, note="timed region; ms_theta_hard = k_theta_hard + "
                                                  "k_bisect_cert + k_bisect_unc + k_bisect_tail"),
            "clocks": clk.summary(),
        }
        if e2e:
            line["e2e"] = e2e
        if late:
            line["late_window"] = late
        if fo_line:
            line["first_order"] = fo_line
        if post:
            if ws == 1 and not args.no_cpu_baseline:
                try:
                    post["cpu_baseline"] = postproc_cpu_baseline()
                except Exception as exc:
                    post["cpu_baseline"] = {"error": f"{type(exc).__name__}: {exc}"}
            line["postproc"] = post
        if not args.no_cpu_baseline and ws == 1:  # the reference CPU path: N = 1 only
            line["cpu_baseline"] = cpu_reference(args, ws)
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
