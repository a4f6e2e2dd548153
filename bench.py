#!/usr/bin/env python
"""Benchmark of the MTI-pruned Lloyd's k-means hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--prune mti|none]
    python bench.py --impl reference ...     # the fp64 CPU oracle as the reference arm

A "step" is one full Lloyd iteration (S1 geometry/drift, S2 MTI assignment, S3 reduction +
allreduce, S4 update, plus any re-bucketing the runtime decides) over the whole data set of
the named config.  The first W iterations (iteration 1 is the dense no-bounds pass) are
warm-up; the next K are timed.  Default workload: C3 (n = 65,608,366, d = 8, k = 100,
spectral-embedding-shaped), the n = 66M configuration the metric is quoted on.

Multi-GPU (torchrun): rows are sharded contiguously over ranks (strong scaling: the global
data set is fixed); the library's NCCL communicator does one allreduce per iteration.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "k-means iters/s and effective point·centroid dists/s at n=66M; HBM GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=27)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--prune", default="mti", choices=["mti", "none", "ti"],
                    help="mti: the paper's method; none: knori- (all k distances); ti: Elkan's TI baseline")
    ap.add_argument("--algo", default="kmeans", choices=["kmeans", "skmeans"],
                    help="skmeans: spherical k-means (PAPER.md §4.2) on the same engine")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--stats-out", default=None)
    ap.add_argument("--engine", default="auto", choices=["auto", "cuda", "tensor", "screen", "tensor_screen", "tensor_chunked"],
                    help="MTI pass engine (auto = the CUDA-core walk k_walk)")
    ap.add_argument("--resort-fraction", type=float, default=0.0)
    ap.add_argument("--no-graph", action="store_true", help="launch each iteration eagerly (no CUDA graph)")
    ap.add_argument("--force-comm", action="store_true",
                    help="run the NCCL allreduce even at N = 1 (1-rank communicator)")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML polled every ~2 ms from
    a thread (the timed region of C3 is only ~70 ms), nvidia-smi as the fallback."""
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mx, self.reasons = [], [], set()
        self.stop = threading.Event()
        self.t = None
        self.src = "nvml"

    def _poll(self):
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        masks = [(nm, getattr(pynvml, attr, 0)) for nm, attr in self.REASONS]
        self.ready.set()
        while not self.stop.is_set():
            self.sm.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.mx.append(mx)
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            for nm, m in masks:
                if m and (r & m):
                    self.reasons.add(nm)
            time.sleep(0.002)
        pynvml.nvmlShutdown()

    def __enter__(self):
        self.ready = threading.Event()
        try:
            import pynvml  # noqa: F401
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            self.ready.wait(5.0)
        except Exception:
            self.t = None
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.t:
            self.t.join(timeout=5)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx),
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": self.src}


def traffic_from_profile(cfg: str, prune: str, kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of ``kernel`` from the committed
    ncu capture summary (profiles/traffic_<cfg>_<prune>.json), or None if it is for another kernel."""
    p = os.path.join(ROOT, "profiles", f"traffic_{cfg}_{prune}.json")
    if os.path.exists(p):
        try:
            j = json.load(open(p))
            return j.get("dram_bytes_per_launch") if j.get("kernel_name", "") == kernel else None
        except Exception:
            return None
    return None


# ------------------------------------------------------------------------------------------
def oracle_full_run(X, C0, k: int, warm: int, timed: int, spherical: bool = False):
    """The fp64 oracle (oracle/, as it stands, all host cores) on the FULL data set: iteration 1
    (brute force, no bounds) and warm-1 further MTI iterations untimed, then ``timed`` MTI
    iterations timed one by one (oracle_mti_pass + block sums + update: the same S1-S4 as a GPU
    step).  Returns (iterations/s over the timed window, seconds per timed iteration, threads)."""
    import numpy as np
    import oracle
    Xs = X
    if spherical:   # sk-means: the oracle's projection and re-normalised update
        Xs, C0 = oracle.normalize_rows(Xs), oracle.normalize_centroids(C0)
    renorm = (lambda Cm, cnt, Cold: oracle.renormalize(Cm, cnt, Cold)) if spherical else (lambda Cm, cnt, Cold: Cm)
    a, d1, _ = oracle.assign_brute(Xs, C0)
    u = np.sqrt(d1)
    del d1
    sums, counts = oracle.cluster_sums(Xs, a, k)
    C, _ = oracle.update(sums, counts, C0)
    C = renorm(C, counts, C0)
    Cprev = C0
    per = []
    for i in range(max(0, warm - 1) + timed):
        t0 = time.perf_counter()
        a, u, _, _, _ = oracle.mti_pass(Xs, C, Cprev, a, u)
        sums, counts = oracle.cluster_sums(Xs, a, k)
        Cprev, (C, _) = C, oracle.update(sums, counts, C)
        C = renorm(C, counts, Cprev)
        if i >= max(0, warm - 1):
            per.append(time.perf_counter() - t0)
    return len(per) / sum(per), per, oracle.num_threads()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, rank, world):
    """Reference arm: the oracle (fp64, OpenMP on all host cores) runs the SAME workload as our
    arm — the full data set of the config, iteration 1 + W-1 warm-up iterations untimed, then K
    timed iterations (the same window as the GPU arm's timed iterations W+1..W+K)."""
    import numpy as np
    from synth import CONFIGS, make_config
    if rank != 0:
        return 0
    spec = CONFIGS[args.config]
    X, idx, _ = make_config(args.config)
    C0 = X[idx].astype(np.float64)
    sph = args.algo == "skmeans"
    rate, per, cores = oracle_full_run(X, C0, spec.k, max(1, args.warmup), args.steps, sph)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "iters/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / rate, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY §8(d) recipe, seed 0)",
        "config": {"workload": f"{args.config}: n={spec.n}, d={spec.d}, k={spec.k}, Forgy init, iterations "
                               f"{max(1, args.warmup) + 1}..{max(1, args.warmup) + args.steps}",
                   "algo": args.algo, "prune": "mti", "parallelism": "host cores (OpenMP)"},
        "effective_dists_per_s": rate * spec.n * spec.k,
        "timed_s": sum(per),
        "cpu_baseline": {"value": rate, "unit": "iters/s", "cores": cores, "kind": "oracle",
                         "cpu": cpu_model(),
                         "sample": f"full {args.config} (n={spec.n}), {args.steps} timed MTI iterations after "
                                   f"iteration 1 (brute force) + {max(0, args.warmup - 1)} warm-up; no extrapolation"},
        "e2e": {"value": rate, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, rank, world, local_rank):
    import numpy as np
    from synth import CONFIGS, make_points, forgy_indices
    from paper_1902_09527_b200.dist import shard_bounds
    spec = CONFIGS[args.config]
    n, d, k = spec.n, spec.d, spec.k
    lo, hi = shard_bounds(n, rank, world)
    # generate before touching CUDA (fork pool)
    t_gen = time.perf_counter()
    X = make_points(args.config, rows=(lo, hi))
    idx = forgy_indices(n, k)
    if world == 1:
        C0 = X[idx].astype(np.float64)
    else:
        C0 = None
    t_gen = time.perf_counter() - t_gen

    import torch
    import torch.distributed as dist
    from paper_1902_09527_b200 import KMeans, nccl_unique_id
    from paper_1902_09527_b200.dist import broadcast_bytes, max_over_ranks

    torch.cuda.set_device(local_rank)
    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl")
        # Forgy rows live on different shards: gather them through the process group
        rows = torch.zeros((k, d), dtype=torch.float64, device="cuda")
        own = (idx >= lo) & (idx < hi)
        if own.any():
            rows[torch.from_numpy(np.nonzero(own)[0]).cuda()] = torch.from_numpy(
                X[idx[own] - lo].astype(np.float64)).cuda()
        dist.all_reduce(rows)
        C0 = rows.cpu().numpy()

    def fresh_nccl_id():
        """A new ncclUniqueId for every communicator (an id serves one ncclCommInitRank)."""
        if world == 1:
            return nccl_unique_id() if args.force_comm else None
        return broadcast_bytes(nccl_unique_id() if rank == 0 else b"\0" * 128)
    nccl_id = fresh_nccl_id()

    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    stream = torch.cuda.current_stream()
    km = KMeans(Xd, C0, prune=args.prune, stream=stream.cuda_stream, rank=rank, world=world,
                spherical=args.algo == "skmeans", graph=not args.no_graph, force_comm=args.force_comm,
                engine=args.engine, resort_fraction=args.resort_fraction, nccl_id=nccl_id, n_global=n)
    for _ in range(args.warmup):
        km.iterate()
    launches0 = km.launch_count
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            km.iterate()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    ms_max = max_over_ranks(ms)
    launches = km.launch_count - launches0
    engine = km.engine
    stats = km.stats()
    timed = stats[args.warmup:args.warmup + args.steps]
    assign_ms = [s["ms_assign"] for s in timed]
    avg_assign = sum(assign_ms) / len(assign_ms)
    # algorithmic bytes per row: MTI x + u r/w + a r/w; knori- x + a r/w;
    # TI additionally reads and writes its k fp32 lower bounds
    bytes_per_row = {"mti": 4 * d + 16, "none": 4 * d + 8, "ti": 4 * d + 16 + 8 * k}[args.prune]
    algo_bytes = (hi - lo) * bytes_per_row
    peak, peak_src = load_peaks()
    achieved = algo_bytes / (avg_assign * 1e-3) / 1e9
    sse = km.sse()
    dev_bytes = km.device_bytes
    km.close()
    del Xd
    torch.cuda.empty_cache()

    iters_per_s = args.steps / (ms_max * 1e-3)
    dists_computed = sum(s["dists"] for s in timed)
    iter_bytes = n * bytes_per_row
    line = {
        "metric": METRIC, "value": iters_per_s, "unit": "iters/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 distances / f64 sums+centroids (exact mode)",
        "data": "synthetic (SURVEY §8(d) recipe, seed 0; stands in for Friendster-8)",
        "config": {"workload": f"{args.config}: n={n}, d={d}, k={k}, Forgy init, iterations "
                               f"{args.warmup + 1}..{args.warmup + args.steps}",
                   "algo": args.algo, "prune": args.prune, "parallelism": f"rows sharded over {world} GPU(s)",
                   "launch": "eager" if args.no_graph else "CUDA graph per iteration (t >= 2)",
                   "collective": "NCCL allreduce" if (world > 1 or args.force_comm) else "none (1 GPU)",
                   "l2": f"inputs {n * 4 * d / 1e9:.2f} GB > 126 MB L2 (no flush needed)"},
        "effective_dists_per_s": iters_per_s * n * k,
        "dists_computed_per_s": dists_computed / (ms_max * 1e-3),
        "hbm_gbs_step": iter_bytes * iters_per_s / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic_from_profile(args.config, args.prune, engine) if args.algo == "kmeans" else None,
                     "kernel": engine,
                     "algorithmic_bytes_per_launch": algo_bytes, "avg_launch_ms": avg_assign,
                     "peak_source": peak_src},
        # FP32 pipe: the centred expansion form spends ~d+2 FP32 lane-operations per
        # computed distance; peak = 148 SMs x 128 lanes x sm clock (1.965 GHz max)
        "fp32_pipe": {"model": "(d+2) FP32 lane-ops per computed distance (expansion form)",
                      "achieved_ops_per_s": (d + 2) * (dists_computed / len(timed)) / (avg_assign * 1e-3),
                      "peak_ops_per_s": 148 * 128 * 1.965e9,
                      "frac": (d + 2) * (dists_computed / len(timed)) / (avg_assign * 1e-3) / (148 * 128 * 1.965e9)},
        "hbm_frac_nominal_8tbs": achieved / 8000.0,
        "device_bytes": dev_bytes,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "final_sse": sse,
        "gen_s": t_gen,
    }
    if args.stats_out and rank == 0:
        json.dump(stats, open(args.stats_out, "w"), indent=1)

    # ---- e2e: the public API end to end from pinned host memory -----------------------------
    if not args.no_e2e:
        Xh = torch.empty((hi - lo, d), dtype=torch.float32, pin_memory=True)
        Xh.numpy()[:] = X
        total_iters = args.warmup + args.steps
        a_out = torch.empty(hi - lo, dtype=torch.int32, pin_memory=True)   # caller-owned, pinned
        # two passes of the whole end-to-end run; the first (untimed) is the e2e warm-up — the first
        # DMA from a freshly pinned buffer pays a one-time mapping cost (measured: create 140 ms
        # instead of 45 ms for C3's 2.1 GB)
        for rep in range(2):
            nid = fresh_nccl_id()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            km2 = KMeans(Xh, C0, prune=args.prune, rank=rank, world=world, nccl_id=nid, n_global=n,
                         spherical=args.algo == "skmeans", graph=not args.no_graph, force_comm=args.force_comm,
                         engine=args.engine, resort_fraction=args.resort_fraction,
                         device=local_rank)
            t1 = time.perf_counter()
            for _ in range(total_iters):
                km2.iterate()
            t2 = time.perf_counter()
            km2.assignments(out=a_out)
            C_out = km2.centroids()
            t_e2e = time.perf_counter() - t0
            phases = {"create_ms": 1e3 * (t1 - t0), "iterate_ms": 1e3 * (t2 - t1),
                      "d2h_ms": 1e3 * (t0 + t_e2e - t2)}
            km2.close()
            if rep == 0:
                phases_warm = phases
        phases["warmup_pass"] = phases_warm
        t_e2e = max_over_ranks(t_e2e)
        line["e2e"] = {"value": total_iters / t_e2e, "unit": "iters/s",
                       "h2d_bytes_per_step": (hi - lo) * d * 4 / total_iters,
                       "d2h_bytes_per_step": ((hi - lo) * 4 + C_out.nbytes) / total_iters,
                       "iterations": total_iters, "includes": "create(H2D) + all iterations + D2H a, C (second of two passes)",
                       "phases": phases}
        del Xh
    # ---- CPU baseline: the oracle on the host cores (rank 0, N=1 only) ------------------------
    if world == 1 and not args.no_cpu_baseline:
        if n * k * d <= 65_608_366 * 100 * 8:
            # the full data set (C3: iteration 1 brute force ~5 s + 2 MTI iterations on 16 cores)
            rate, per, cores = oracle_full_run(X, C0, k, 1, 2, args.algo == "skmeans")
            smp = (f"full {args.config} (n={n}), MTI iterations 2-3 timed after iteration 1 (brute force); "
                   f"{sum(per):.1f} s timed; no extrapolation")
        else:
            # d = 32 / k = 1000: a prefix of the rows (a full brute-force iteration 1 of C5 takes minutes)
            m = 2_000_000 if k <= 100 else 400_000
            rate, per, cores = oracle_full_run(np.ascontiguousarray(X[:m]), C0, k, 1, 2, args.algo == "skmeans")
            rate *= m / n
            smp = (f"first {m} rows of {args.config}, MTI iterations 2-3 after iteration 1 ({sum(per):.1f} s), "
                   f"scaled x{n / m:.1f} by rows (extrapolated: not the same workload)")
        line["cpu_baseline"] = {"value": rate, "unit": "iters/s", "cores": cores, "kind": "oracle",
                                "cpu": cpu_model(), "sample": smp}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def relaunch(args) -> int:
    """--gpus N > 1 without a torchrun environment: start the N ranks ourselves (one process per
    GPU, torch.distributed.run on 127.0.0.1) and return its exit code."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
