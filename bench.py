"""HAPOD hot-path benchmark (BASELINE.json metric: snapshot cols/sec fp64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config 1] [--d D]

Workload (N=1 default): BASELINE config 1 -- two-level distributed HAPOD,
S = Q1 diag(sigma) Q2^T, 200,000 x 8,192 fp64, sigma_i = 10^(-10 (i-1)/8191),
16 leaves x 512 columns + one root, eps* = 1e-6 ||S||_F, omega = 0.75,
target = eps* / sqrt(8192).  One step = one full HAPOD of that
snapshot set (16 leaf PODs + the root POD, every kernel of the hot path).

value  : whole-job snapshot columns per second with S resident in HBM.
e2e    : the same through the public API from pinned HOST memory: each step
         SnapshotBlock(space, host S, defer_upload=True) (per-leaf H2D copies on a
         shared copy stream + device finiteness checks, overlapping the leaf PODs),
         distribute_columns, assign_tolerances, run_parallel, sigmas read back.
roofline: the dominant kernel family by device time inside the timed region
         (CUDA events on the launching stream), its algorithmic FP64 flops
          / its time, against the measured FP64 DMMA peak.
cpu_baseline / --impl reference: the reference algorithm (the oracle port of
         hapod, NumPy + OpenBLAS with all host threads) on a bounded sample of
         the same workload: the first leaves of config 1 at full d.

For N > 1 the script is launched with torch.distributed.run (one process per
GPU, NCCL); leaves are placed on ranks in contiguous chunks, child -> parent
edges move sigma-scaled mode blocks with NCCL send/recv, the root runs on
rank 0; timing is the max over ranks of CUDA-event durations.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.1  # measured on this pool's B200: tools/microbench/fp64_peak.cu (DMMA m8n8k4)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--d", type=int, default=None, help="override the row count (smoke runs only)")
    ap.add_argument("--workers", type=int, default=None, help="stream workers for the leaf wave (N=1)")
    ap.add_argument("--cpu-leaves", type=int, default=2, help="leaves in the CPU baseline sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg (profiling runs only)")
    ap.add_argument("--root", default="rows", choices=["rows", "gather"],
                    help="N > 1: evaluate the root on row blocks on every GPU (rows) or gather the "
                         "children's modes on rank 0 (gather)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() in ("active", "1", "yes"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU baseline
def cpu_sample(host_cols: np.ndarray, eps_leaf: float, steps: int, warmup: int):
    """The reference hot path (oracle port of hapod.pod, NumPy/SciPy + OpenBLAS, all host
    threads) on c1 leaf blocks at full d.  Returns seconds per sample."""
    from oracle import hapod_oracle as O

    def one():
        for j in range(host_cols.shape[1] // 512):
            O.pod(host_cols[:, 512 * j: 512 * (j + 1)], eps_leaf)

    for _ in range(warmup):
        one()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        one()
        times.append(time.perf_counter() - t0)
    return times


def cpu_info():
    cores = os.cpu_count() or 1
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        blas = [f"{i.get('internal_api')} {i.get('version')} threads={i.get('num_threads')}" for i in info]
        threads = max([i.get("num_threads", 1) for i in info] or [cores])
    except Exception:  # pragma: no cover
        blas, threads = [], cores
    return cores, threads, blas


# ----------------------------------------------------------------------------- main
def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    import torch.distributed as dist

    if a.impl == "reference":
        return run_reference(a, world, rank, local)

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1607_05210_b200 as H
    from paper_1607_05210_b200 import _device as D
    from paper_1607_05210_b200 import _native as N
    from paper_1607_05210_b200 import distributed as DI
    from paper_1607_05210_b200 import workloads as W

    lib = N.load()
    cfg = W.CONFIGS[a.config]
    wl = W.make(a.config, d=a.d)
    d, m = wl.d, wl.m
    nleaves = max(1, m // wl.block)
    tree = H.build_star(nleaves) if nleaves > 1 else H.RootedTree(((),), 0)
    maps = H.derive_maps(tree)
    place = DI.plan_placement(tree, world, maps)
    my_leaves = [leaf for leaf in maps.leaf_order if place[leaf] == rank]
    col0 = {leaf: i * wl.block for i, leaf in enumerate(maps.leaf_order)}
    sp = H.InnerProductSpace(d)
    # device-resident snapshot views of this rank's leaves
    full = H.SnapshotBlock(sp, wl.values)
    leaf_blocks = {leaf: full.column_block(col0[leaf], col0[leaf] + wl.block) for leaf in my_leaves}
    counts = {leaf: wl.block for leaf in maps.leaf_order}
    target = H.eps_star_to_target(wl.eps_star, m)
    tol = H.assign_tolerances(tree, counts, target, omega=wl.omega)
    workers = a.workers or (min(16, len(my_leaves)) if world == 1 else 1)

    def step_device():
        if world == 1:
            la = H.LeafAssignment(leaf_blocks)
            if workers > 1:
                res, _ = H.run_parallel(tree, la, tol, worker_count=workers)
            else:
                res = H.run_hapod(tree, la, tol)
            return res.modes
        ev = DI.DeviceEvaluator(sp, leaf_blocks, tol)
        root, _, _ = DI.run_distributed(tree, ev, rank, world, place, root_rows=(a.root == "rows"))
        return root

    # host copy (pinned, column-major) for the end-to-end leg
    lo = min(col0[leaf] for leaf in my_leaves) if my_leaves else 0
    hi = max(col0[leaf] for leaf in my_leaves) + wl.block if my_leaves else 0
    host = torch.empty((hi - lo, d), dtype=torch.float64, pin_memory=True)
    host.copy_(wl.values[:, lo:hi].t())
    host_view = host.t()  # (d, cols) column-major view of pinned host memory

    def step_e2e():
        # deferred upload: each leaf's columns go host -> device through one shared copy stream
        # when its POD starts, so the 13 GB transfer overlaps the other leaves' PODs
        blk = H.SnapshotBlock(sp, host_view, defer_upload=True)
        blocks = {leaf: blk.column_block(col0[leaf] - lo, col0[leaf] - lo + wl.block) for leaf in my_leaves}
        if world == 1:
            la = H.LeafAssignment(blocks)
            tol_e = H.assign_tolerances(tree, la, target, omega=wl.omega)
            res = (H.run_parallel(tree, la, tol_e, worker_count=workers)[0] if workers > 1
                   else H.run_hapod(tree, la, tol_e))
            out = res.modes
        else:
            ev = DI.DeviceEvaluator(sp, blocks, tol)
            out, _, _ = DI.run_distributed(tree, ev, rank, world, place, root_rows=(a.root == "rows"))
        if out is not None:
            np.asarray(out.sigmas).sum()  # sigmas already read back to the host
        return out

    summ_root = {}

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    prof_range = os.environ.get("HP_PROFILE_RANGE") == "1"  # ncu --profile-from-start off

    def timed(fn, steps, profile=False):
        barrier()
        if profile:
            D.Profiler.reset(True)
            if prof_range:
                torch.cuda.cudart().cudaProfilerStart()
        launches0 = lib.hp_launch_count()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        out = None
        for _ in range(steps):
            out = fn()
        e1.record()
        torch.cuda.synchronize()
        if profile and prof_range:
            torch.cuda.cudart().cudaProfilerStop()
        barrier()
        ms = e0.elapsed_time(e1)
        launches = lib.hp_launch_count() - launches0
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            c = torch.tensor([launches], dtype=torch.int64, device="cuda")
            dist.all_reduce(c, op=dist.ReduceOp.SUM)
            launches = int(c.item())
        summary = D.Profiler.summary() if profile else None
        if profile:
            nonlocal summ_root
            summ_root = D.Profiler.summary(tag=tree.root)
        D.Profiler.reset(False)
        return ms, out, launches, summary

    for _ in range(a.warmup):
        step_device()
    clocks = ClockSampler(local)
    clocks.start()
    ms, out, launches, summ = timed(step_device, a.steps, profile=True)
    clk = clocks.stop()
    if a.no_e2e:
        ms_e2e = float("nan")
    else:
        for _ in range(max(1, a.warmup // 3)):
            step_e2e()
        ms_e2e, out_e2e, _, _ = timed(step_e2e, a.steps)

    cols_per_s = m * a.steps / (ms * 1e-3)
    e2e_cols = m * a.steps / (ms_e2e * 1e-3)
    h2d = (hi - lo) * d * 8
    if world > 1:
        t = torch.tensor([h2d], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        h2d = int(t.item())

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # --------------------------------------------------------------- roofline (rank 0)
    # The root node runs alone on the GPU (the leaf wave overlaps 16 nodes on 16 streams,
    # which inflates per-phase event times), so the per-kernel rates are taken on the root
    # node's launches inside the timed region; whole-step phase totals are reported beside.
    phases = {k: {"launches": n // a.steps, "ms_per_step": ms_ / a.steps, "flop_per_step": fl / a.steps}
              for k, (n, ms_, fl) in summ.items()}
    root_s = summ_root
    step_ms = ms / a.steps
    gemm_phases = [k for k in ("gram", "assemble", "drift", "reortho", "eigvec", "polish_q0", "polish_x",
                               "polish_rr") if k in root_s]
    g_fl = sum(root_s[k][2] for k in gemm_phases) / a.steps
    g_ms = sum(root_s[k][1] for k in gemm_phases) / a.steps
    e_fl = sum(root_s[k][2] for k in ("eigensolve", "eigensolve_polish") if k in root_s) / a.steps
    e_ms = sum(root_s[k][1] for k in ("eigensolve", "eigensolve_polish") if k in root_s) / a.steps
    root_ms = sum(v[1] for v in root_s.values()) / a.steps
    g_tf = g_fl / (g_ms * 1e-3) / 1e12 if g_ms else 0.0
    e_tf = e_fl / (e_ms * 1e-3) / 1e12 if e_ms else 0.0
    roofline = {
        "bound": "tensor",
        "kernel": "gemm_kernel (FP64 DMMA GEMM engine: Gram SYRK, reconstruction, drift SYRK, CholQR TRMM, "
                  "Ritz products) on the root node",
        "achieved": round(g_tf, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
        "frac": round(g_tf / FP64_PEAK_TFLOPS, 4),
        # DRAM bytes of the family's largest launch (root Gram SYRK, gemm_tma_kernel<1,1>, m=8192,
        # d=200,000) from one ncu --set full capture (profiles/r1g_gemm_gram8192_metrics.txt):
        # 104.4 GB read + 0.56 GB written against 13.65 GB algorithmic (S once + G).  The 2080
        # output tiles run in 14 waves; with the grouped tile raster (8 column panels per group,
        # hp_gemm.cu tile_coords) a wave shares ~26 panels (L2 hit rate 82 %; the column-major order
        # read 269 GB at 64 %).  At 0.26 TB/s (3 % of HBM) the launch is tensor-bound (98.8 %
        # tensor-pipe active), so the remaining re-reads cost no time
        "traffic": 105.0e9, "traffic_algorithmic": 13.65e9,
        "peak_source": "measured FP64 DMMA peak on this pool's B200 (tools/microbench/fp64_peak.cu, "
                       "profiles/r1_fp64_peak.txt); MEASURED_PEAKS.json carries no FP64 figure",
        "share_of_step": round(g_ms / step_ms, 4),
        "root_share_of_step": round(root_ms / step_ms, 4),
        "eigensolver": {"kernel": "jac_local + jac_apply (block Jacobi; DMMA rotation products counted)",
                        "achieved": round(e_tf, 3), "frac": round(e_tf / FP64_PEAK_TFLOPS, 4),
                        "share_of_step": round(e_ms / step_ms, 4)},
        "root_phases_ms_per_step": {k: round(v[1] / a.steps, 3) for k, v in sorted(root_s.items())},
        "all_phases_ms_per_step (leaf wave overlapped)": {k: round(v["ms_per_step"], 3)
                                                           for k, v in phases.items()},
    }

    # --------------------------------------------------------------- CPU baseline (rank 0, N=1)
    cpu = None
    if world == 1 and not a.no_cpu:
        nl = max(1, min(a.cpu_leaves, nleaves))
        cols = np.asfortranarray(wl.values[:, : nl * wl.block].cpu().numpy())
        eps_leaf = tol.epsilons[maps.leaf_order[0]]
        cores, threads, blas = cpu_info()
        t = cpu_sample(cols, eps_leaf, 1, 0)
        cpu = {"value": round(nl * wl.block / t[0], 3), "unit": "cols/s", "cores": threads, "kind": "port",
               "sample": f"{nl} leaf POD(s) of config {a.config} at full d={d} ({nl * wl.block} columns, "
                         f"oracle port of hapod.pod, NumPy/OpenBLAS); root excluded, so this over-states "
                         f"CPU throughput", "blas": blas}

    res_modes = out.count if out is not None else None
    line = {
        "metric": "HAPOD snapshot cols/sec fp64",
        "value": round(cols_per_s, 3),
        "unit": "cols/s",
        "n_gpus": world,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": round(step_ms, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded on device, BASELINE config generator; no dataset involved)",
        "config": {"workload": f"config {a.config}: {cfg['name']}", "rows": d, "cols": m,
                   "leaves": nleaves, "leaf_cols": wl.block, "eps_star_rel": cfg["rel"], "omega": wl.omega,
                   "eps_star": wl.eps_star, "target": target, "modes": res_modes,
                   "l2_flush": f"inputs {d * m * 8 / 1e9:.1f} GB >> 126 MB L2 (no explicit flush)",
                   "parallelism": f"tree over {world} GPU(s); leaf wave on {workers} stream worker(s)"
                                  + (f"; root on {world} row blocks" if world > 1 and a.root == "rows" else "")},
        "e2e": {"value": round(e2e_cols, 3), "unit": "cols/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": 8 * (res_modes or 0)},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference(a, world, rank, local):
    """--impl reference: the reference hot path on the host cores (the oracle port; the
    reference package itself cannot travel to the GPU box).  Rank 0 only."""
    import torch
    if rank != 0:
        return
    cfg_rows = a.d
    from oracle import hapod_oracle as O  # noqa: F401
    cores, threads, blas = cpu_info()
    # the same seeded snapshot columns as the b200 arm (generated on the GPU when present)
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
        from paper_1607_05210_b200 import workloads as W
        wl = W.make(a.config, d=cfg_rows)
        nl = a.cpu_leaves
        cols = np.asfortranarray(wl.values[:, : nl * wl.block].cpu().numpy())
        d, m, eps_star, block, omega = wl.d, wl.m, wl.eps_star, wl.block, wl.omega
        del wl
        torch.cuda.empty_cache()
    else:
        print(json.dumps({"impl": "reference", "unavailable": "needs the seeded config generator (CUDA)"}))
        return
    nleaves = m // block
    target = eps_star / math.sqrt(m)
    depth_spread = math.sqrt(1.0 - omega * omega) / math.sqrt(1)  # star: depth 2
    eps_leaf = math.sqrt(block) * depth_spread * target
    times = cpu_sample(cols, eps_leaf, a.steps, a.warmup)
    v = cols.shape[1] / (sum(times) / len(times))
    line = {"impl": "reference", "metric": "HAPOD snapshot cols/sec fp64", "value": round(v, 3), "unit": "cols/s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": round(1e3 * sum(times) / len(times), 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config {a.config}", "rows": d, "cols": m, "sample_cols": cols.shape[1]},
            "cpu_baseline": {"value": round(v, 3), "unit": "cols/s", "cores": threads, "kind": "port",
                             "sample": f"{cols.shape[1] // block} leaf POD(s) of config {a.config} at full "
                                       f"d={d} per step (oracle port of hapod.pod; root excluded)",
                             "blas": blas},
            "e2e": {"value": round(v, 3), "unit": "cols/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
