"""HAPOD hot-path benchmark (BASELINE.json metric: snapshot cols/sec fp64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config 0..4]

Default workload (N=1): BASELINE config 1 -- two-level distributed HAPOD,
S = Q1 diag(sigma) Q2^T, 200,000 x 8,192 fp64, sigma_i = 10^(-10 (i-1)/8191),
16 leaves x 512 columns + one root, eps* = 1e-6 ||S||_F, omega = 0.75,
target = eps* / sqrt(8192).  One step = one full HAPOD of that
snapshot set (16 leaf PODs + the root POD, every kernel of the hot path).

value  : whole-job snapshot columns per second with S resident in HBM.
e2e    : the same through the public API from pinned HOST memory: each step
         SnapshotBlock(space, host S, defer_upload=True) (per-leaf H2D copies on a
         shared copy stream + device finiteness checks, overlapping the leaf PODs),
         distribute_columns, assign_tolerances, run_parallel, sigmas read back.  The
         final ModeSet stays device-resident: a caller that touches
         ``.modes`` on the host pays another d x N x 8 bytes of D2H (7.3 GB at config 1),
         reported as ``e2e.modes_d2h_bytes_if_requested`` and NOT inside the timed region.
roofline: the dominant kernel family by device time inside the timed region
         (CUDA events on the launching stream), its algorithmic FP64 flops
          / its time, against the measured FP64 DMMA peak.
         ``roofline.eigensolver``: the HBM-bound side of the step -- the tridiagonalisation
         kernel (sytrd_panel) of the root's eigensolve, its algorithmic matrix reads
         (8 r^3 / 3 bytes, reported by hp_syev_tri with its own CUDA-event time) against
         MEASURED_PEAKS.json's copy bandwidth -- and the polish Jacobi's DMMA rate.
cpu_baseline / --impl reference: the reference algorithm (the oracle port of hapod,
         NumPy + SciPy + OpenBLAS with all host threads; data from oracle/hostgen.py -- no
         product code, no CUDA) over the WHOLE tree of the config (all leaves + the root,
         including the root's Python MGS sweep pod.py:227-237) on a bounded instance:
         reduced rows d' and reduced columns per leaf, because the full-size reference takes
         ~12 h.  ``cpu_baseline.sample`` states the instance exactly; the b200
         arm runs the SAME instance on the GPU and reports it as ``like_for_like``.

--gpus N (N > 1) without a torchrun environment starts N ranks of this script itself (one process
per GPU with RANK / LOCAL_RANK / WORLD_SIZE / MASTER_ADDR=127.0.0.1 set as torchrun would, NCCL,
``NCCL_DEBUG=INFO`` so the init lines show the rank count); under torchrun it uses the given ranks.
Leaves are placed on ranks in contiguous chunks, child -> parent edges move sigma-scaled mode
blocks with grouped NCCL send/recv, a star's root is evaluated on row blocks by all ranks
(rowroot.py); timing is the max over ranks of CUDA-event durations.  Config 2 (one chain)
does not shard: ``--gpus N`` runs N independent replicas ("replicas only").
``--protocol-check`` rehearses the same launch + placement + edge path on CPU (gloo, the
oracle as the node arithmetic) -- used by tests/test_bench_launch.py; it is not a measurement.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.1  # measured on this pool's B200: tools/microbench/fp64_peak.cu (DMMA m8n8k4)
METRIC = "HAPOD snapshot cols/sec fp64"

# BASELINE.json configs (static description shared by both arms; no package import)
CFG = {
    0: dict(name="c0-single-pod", tree="one node", rows=20_000, cols=1_000, leaves=1, leaf_cols=1_000, rel=1e-4,
            omega=1.0),
    1: dict(name="c1-star16", tree="star(16) + root", rows=200_000, cols=8_192, leaves=16, leaf_cols=512, rel=1e-6,
            omega=0.75),
    2: dict(name="c2-chain64", tree="incremental chain of 64 slices", rows=500_000, cols=32_768, leaves=64,
            leaf_cols=512, rel=1e-3, omega=0.9),
    3: dict(name="c3-star64", tree="star(64) + root", rows=2_000_000, cols=32_768, leaves=64, leaf_cols=512,
            rel=1e-5, omega=0.75),
    4: dict(name="c4-8chains16", tree="8 chains of 16 slices under a root", rows=1_000_000, cols=65_536, leaves=128,
            leaf_cols=512, rel=1e-4, omega=0.8),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=1, choices=sorted(CFG))
    ap.add_argument("--d", type=int, default=None, help="override the row count (smoke runs only)")
    ap.add_argument("--workers", type=int, default=None, help="stream workers for the leaf wave (N=1)")
    ap.add_argument("--ref-d", type=int, default=None, help="rows of the reference arm's bounded instance")
    ap.add_argument("--ref-leaf-cols", type=int, default=None,
                    help="columns per leaf of the reference arm's bounded instance")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg (profiling runs only)")
    ap.add_argument("--root", default="rows", choices=["rows", "gather"],
                    help="N > 1: evaluate a star's root on row blocks on every GPU (rows) or gather the "
                         "children's modes on rank 0 (gather)")
    ap.add_argument("--protocol-check", action="store_true",
                    help="CPU rehearsal of the multi-rank launch/edge path (gloo + oracle arithmetic)")
    ap.add_argument("--shared-gpu-check", action="store_true",
                    help="rehearsal of the N > 1 DEVICE path with all ranks on cuda:0 over gloo (host-staged "
                         "tensors, tests/_gloo_cuda_shim.py); a correctness check of the bench path, not a measurement")
    return ap.parse_args()


def static_config(a) -> dict:
    """The workload description both arms print (identical dicts => same config)."""
    c = CFG[a.config]
    d = a.d or c["rows"]
    return {"workload": f"config {a.config}: {c['name']} ({c['tree']})", "rows": d, "cols": c["cols"],
            "leaves": c["leaves"], "leaf_cols": c["leaf_cols"], "eps_star_rel": c["rel"], "omega": c["omega"],
            "l2_flush": f"inputs {d * c['cols'] * 8 / 1e9:.1f} GB >> 126 MB L2 (no explicit flush)"}


# ----------------------------------------------------------------------------- launch
def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def visible_gpus() -> int:
    try:
        out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=30).stdout
        n = sum(1 for ln in out.splitlines() if ln.startswith("GPU "))
    except (OSError, subprocess.SubprocessError):
        return 0
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis is not None and vis.strip() != "":
        n = min(n, len([v for v in vis.split(",") if v.strip() != ""]))
    return n


def self_launch(a) -> int:
    """--gpus N outside torchrun: start N ranks of this script (one per GPU) and pass the
    exit code through.  Rank 0 prints the JSON line."""
    if not a.protocol_check and not a.shared_gpu_check and a.impl == "b200":
        have = visible_gpus()
        if have < a.gpus:
            print(json.dumps({"metric": METRIC, "n_gpus": a.gpus, "error": f"--gpus {a.gpus} needs {a.gpus} visible "
                              f"GPUs, this box shows {have}"}), flush=True)
            return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", str(max(1, (os.cpu_count() or 1) // a.gpus)))
    # one process per GPU with the torchrun environment (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_*), started
    # directly: torch.distributed.run's own option parser takes abbreviated script flags (e.g. --d) for its own
    env.update(WORLD_SIZE=str(a.gpus), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()),
               LOCAL_WORLD_SIZE=str(a.gpus))
    procs = []
    for r in range(a.gpus):
        e = dict(env, RANK=str(r), LOCAL_RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=e))
    rc = 0
    try:
        pending = list(procs)
        while pending:
            for p in list(pending):
                code = p.poll()
                if code is None:
                    continue
                pending.remove(p)
                if code != 0 and rc == 0:      # one rank failed: stop the others instead of hanging in a collective
                    rc = code
                    for q in pending:
                        q.terminate()
            time.sleep(0.2)
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    return rc


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


# ----------------------------------------------------------------------------- reference sample (CPU, oracle only)
def cpu_info():
    cores = os.cpu_count() or 1
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        blas = [f"{i.get('internal_api')} {i.get('version')} threads={i.get('num_threads')}" for i in info]
        threads = max([i.get("num_threads", 1) for i in info] or [cores])
    except Exception:  # pragma: no cover
        blas, threads = [], cores
    try:
        model = open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": \t")
    except Exception:  # pragma: no cover
        model = "unknown"
    return cores, threads, blas, model


class RefSample:
    """The reference arm's bounded instance of a config: the WHOLE tree of the config (every
    leaf and the root / every merge) with the config's generator, spectrum, eps* rule and omega,
    at reduced rows d' and reduced columns per leaf.  Built with oracle/hostgen.py and run with
    oracle/hapod_oracle.py only -- nothing of the product is imported."""

    def __init__(self, a):
        from oracle import hapod_oracle as O
        from oracle import hostgen
        self.O = O
        c = CFG[a.config]
        self.index = a.config
        idx = a.config
        if idx == 0:      # the config itself: it is the reference's own CPU-runnable case
            d, lc, nl = a.ref_d or c["rows"], a.ref_leaf_cols or c["cols"], 1
        elif idx == 1:    # star(16) + root at d' = 10,000 (BASELINE.md 2.1's d'), 64 columns per leaf
            d, lc, nl = a.ref_d or 10_000, a.ref_leaf_cols or 64, 16
        elif idx == 2:    # chain of 8 slices of 512 at d' = 20,000
            d, lc, nl = a.ref_d or 20_000, a.ref_leaf_cols or 512, 8
        elif idx == 3:    # star(8) + root, 128-column leaves at d' = 8,000
            d, lc, nl = a.ref_d or 8_000, a.ref_leaf_cols or 128, 8
        else:             # 2 chains of 4 slices of 256 under a root at d' = 10,000
            d, lc, nl = a.ref_d or 10_000, a.ref_leaf_cols or 256, 8
        self.d, self.leaf_cols, self.nleaves = d, lc, nl
        m = lc * nl
        self.m = m
        seed = idx
        if idx in (0, 1):
            dec = 8.0 if idx == 0 else 10.0
            s, _ = hostgen.decay(d, m, dec, seed)
        elif idx == 2:
            s = hostgen.pulse(d, np.arange(m), seed)
        elif idx == 3:
            s = np.asfortranarray(np.hstack([hostgen.sine(d, np.arange(b * lc, (b + 1) * lc), seed, b)
                                             for b in range(nl)]))
        else:
            s = np.asfortranarray(np.hstack([hostgen.mixed(d, np.arange(b * lc, (b + 1) * lc), m, seed, b)
                                             for b in range(nl)]))
        self.values = s
        self.fro = float(np.linalg.norm(s))
        self.eps_star = c["rel"] * self.fro
        self.target = self.eps_star / math.sqrt(m)
        self.omega = c["omega"]
        # tree (children lists, root 0) and leaf order
        if idx == 0:
            self.children, self.leaf_ids = [[]], [0]
        elif idx in (1, 3):
            self.children, self.leaf_ids = [list(range(1, nl + 1))] + [[] for _ in range(nl)], list(range(1, nl + 1))
        elif idx == 2:
            self.children, self.leaf_ids = None, None   # incremental session (hierarchy.py:370-509)
        else:
            chains, per = 2, nl // 2
            ch = [[]]
            for _ in range(chains):
                sub_children, sub_root = O.chain(per)
                off = len(ch)
                ch[0].append(off + sub_root)
                ch.extend([[off + k for k in kids] for kids in sub_children])
            self.children = ch
            self.leaf_ids = O.leaf_order(ch, 0)
        if self.children is not None:
            counts = {leaf: lc for leaf in self.leaf_ids}
            self.eps = O.assign_tolerances(self.children, 0, counts, self.target, self.omega,
                                           zero_leaf_tolerance=(idx == 4))
        self.blocks = ({leaf: s[:, lc * i: lc * (i + 1)] for i, leaf in enumerate(self.leaf_ids)}
                       if self.leaf_ids is not None else None)

    def describe(self) -> str:
        c = CFG[self.index]
        shape = {0: "pod(S, eps*)", 1: "run_hapod(build_star(16))", 2: f"IncrementalSession over {self.nleaves} slices",
                 3: f"run_hapod(build_star({self.nleaves}))",
                 4: f"run_hapod on 2 chains of {self.nleaves // 2} slices under a root, zero leaf tolerance"}[self.index]
        full = (self.d == c["rows"] and self.m == c["cols"])
        return (f"config {self.index} generator, eps* = {c['rel']:g}*||S||_F, omega = {c['omega']}: {shape} -- "
                f"the whole tree incl. the root and its MGS sweep -- on {self.d} rows x {self.m} columns "
                f"({self.nleaves} leaves x {self.leaf_cols})"
                + ("; the full-size config" if full else
                   f"; REDUCED from {c['rows']} x {c['cols']}: the full-size reference run takes hours "
                   "(root MGS is O(N^2 d) in a Python loop, BASELINE.md 2), so this instance over-states the "
                   "reference's full-size throughput") + "; oracle port of hapod (NumPy/SciPy/OpenBLAS)")

    def step(self):
        O = self.O
        if self.index == 0:
            return O.pod(self.values, self.eps_star).count
        if self.index == 2:
            lc = self.leaf_cols
            cur, _, _ = O.incremental([self.values[:, lc * j: lc * (j + 1)] for j in range(self.nleaves)],
                                      self.target, self.omega)
            return cur.count
        return O.run_hapod(self.children, 0, self.blocks, self.eps).modes.count

    def time_steps(self, steps: int, warmup: int):
        for _ in range(warmup):
            self.step()
        times, modes = [], None
        for _ in range(steps):
            t0 = time.perf_counter()
            modes = self.step()
            times.append(time.perf_counter() - t0)
        return times, modes


def committed_full_tree():
    """The committed full-tree reference run of config 1 (all 8,192 columns, d' = 10,000;
    tests/golden/c1_d10000.json, written by tests/golden/make_c1_fixture.py --variant ref)."""
    p = os.path.join(ROOT, "tests", "golden", "c1_d10000.json")
    try:
        with open(p) as f:
            ref = json.load(f)["reference"]
        return {"cols_per_s": round(ref["m"] / ref["run_s"], 3), "run_s": round(ref["run_s"], 1), "rows": ref["d"],
                "cols": ref["m"], "modes": ref["N"], "cpu": ref.get("cpu"), "nproc": ref.get("nproc"),
                "note": "unmodified reference hapod.run_hapod(build_star(16)) incl. the root's MGS, measured in the "
                        "build container at d' (node GEMM time grows ~ d, eigh time does not; not extrapolated)",
                "source": "tests/golden/c1_d10000.json"}
    except (OSError, KeyError, ValueError):
        return None


def run_reference(a, world, rank):
    """--impl reference: the reference hot path on the host cores.  Rank 0 only; no CUDA, no
    product code (data from oracle/hostgen.py, arithmetic from oracle/hapod_oracle.py)."""
    if rank != 0:
        return 0
    cores, threads, blas, model = cpu_info()
    smp = RefSample(a)
    times, modes = smp.time_steps(a.steps, a.warmup)
    mean = sum(times) / len(times)
    v = smp.m / mean
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "cols/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(1e3 * mean, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded on the host, oracle/hostgen.py; no dataset involved)",
            "config": static_config(a),
            "cpu_baseline": {"value": round(v, 3), "unit": "cols/s", "cores": threads, "kind": "port",
                             "sample": smp.describe(), "sample_rows": smp.d, "sample_cols": smp.m, "modes": modes,
                             "cpu": model, "host_cores": cores, "blas": blas,
                             "full_tree_at_reduced_rows": committed_full_tree() if a.config == 1 else None},
            "e2e": {"value": round(v, 3), "unit": "cols/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- CPU protocol rehearsal
def run_protocol_check(a, world, rank):
    """gloo + oracle arithmetic: the --gpus N launch, placement, post-order and edge path of
    the b200 arm on CPU (tests/test_bench_launch.py).  Prints a JSON line that is NOT a
    measurement (metric 'protocol-check')."""
    import torch.distributed as dist

    from oracle import hapod_oracle as O
    from oracle.dist_evaluator import OracleEvaluator
    from paper_1607_05210_b200 import distributed as DI
    from paper_1607_05210_b200.tree import RootedTree

    if world > 1:
        dist.init_process_group("gloo")
    try:
        nl, lc, d = 8, 12, 60
        data = O.synthetic_decay(d, nl * lc, 0.08, seed=5)
        children = [list(range(1, nl + 1))] + [[] for _ in range(nl)]
        tree = RootedTree(tuple(tuple(c) for c in children), 0)
        blocks = {leaf: data[:, lc * (leaf - 1): lc * leaf] for leaf in range(1, nl + 1)}
        eps = O.assign_tolerances(children, 0, {leaf: lc for leaf in blocks}, 1e-3, 0.75)
        place = DI.plan_placement(tree, world)
        mine = {leaf: blk for leaf, blk in blocks.items() if place[leaf] == rank}
        ev = OracleEvaluator(children, mine if world > 1 else blocks, eps)
        t0 = time.perf_counter()
        root, _, stats = DI.run_distributed(tree, ev, rank, world, place)
        dt = time.perf_counter() - t0
        if world > 1:
            import torch
            t = torch.tensor([dt], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        if rank == 0:
            ref = O.run_hapod(children, 0, blocks, eps)
            same = bool(np.array_equal(root.sigmas, ref.modes.sigmas) and np.array_equal(root.modes, ref.modes.modes))
            print(json.dumps({"metric": "protocol-check", "n_gpus": 0, "ranks": world, "backend": "gloo",
                              "edges_received_on_rank0": stats.recvs, "modes": int(root.count),
                              "bitwise_equal_to_single_process": same, "seconds": round(dt, 4)}), flush=True)
    finally:
        if world > 1:
            dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- b200 arm helpers
class EventClock:
    """Sum of CUDA-event intervals on the current stream (device synchronize on both sides)."""

    def __init__(self, torch):
        self.torch = torch
        self.ms = 0.0

    def __enter__(self):
        self.torch.cuda.synchronize()
        self.e0 = self.torch.cuda.Event(enable_timing=True)
        self.e0.record()
        return self

    def __exit__(self, *exc):
        e1 = self.torch.cuda.Event(enable_timing=True)
        e1.record()
        self.torch.cuda.synchronize()
        self.ms += self.e0.elapsed_time(e1)
        return False


def chains_under_root(H, chains, per):
    children = [[]]
    for _ in range(chains):
        sub = H.build_chain(per)
        off = len(children)
        children[0].append(off + sub.root)
        children.extend([[off + k for k in kids] for kids in sub.children])
    return H.RootedTree(tuple(tuple(k) for k in children), 0)


def hbm_peak_gbs():
    """Measured copy bandwidth of this pool's B200 (MEASURED_PEAKS.json, driver-written); the
    profiling recipe's fallback otherwise."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, ValueError, KeyError):
        return 6500.0, "B200_PROFILING.md fallback"


def gemm_roofline(summ, steps, step_ms, label, extra=None):
    """Roofline of the contraction family (Gram / block Gram / reconstruction / drift / CholQR /
    Ritz products) from the Profiler's CUDA-event records."""
    names = ("gram", "assemble", "drift", "reortho", "eigvec", "polish_q0", "polish_x", "polish_rr")
    fl = sum(summ[k][2] for k in names if k in summ) / steps
    ms = sum(summ[k][1] for k in names if k in summ) / steps
    tf = fl / (ms * 1e-3) / 1e12 if ms else 0.0
    e_names = ("eigensolve", "eigensolve_polish")
    e_fl = sum(summ[k][2] for k in e_names if k in summ) / steps
    e_ms = sum(summ[k][1] for k in e_names if k in summ) / steps
    e_tf = e_fl / (e_ms * 1e-3) / 1e12 if e_ms else 0.0
    eig = {"kernel": "pstrf + jac_round/jac_apply (block Jacobi; DMMA rotation products counted)",
           "achieved": round(e_tf, 3), "frac": round(e_tf / FP64_PEAK_TFLOPS, 4),
           "share_of_step": round(e_ms / step_ms, 4) if step_ms else None}
    tri = (extra or {}).get("sytrd_panel")
    if tri and tri[1] > 0.0:
        # the large preconditioned eigenproblems go through hp_syev_tri: its dominant kernel is the
        # HBM/L2-bound tridiagonalisation (one matrix-vector product per column)
        peak, src = hbm_peak_gbs()
        gbs = tri[2] / (tri[1] * 1e-3) / 1e9
        t_ms = summ.get("eigensolve_tri", (0, 0.0, 0.0))[1] / steps
        eig = {"kernel": "sytrd_panel (Householder tridiagonalisation of H = L^T L: one symmetric matrix-vector "
                         "product per column, column dots over the trailing matrix; + syr2k GEMM per 64 columns)",
               "bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s", "frac": round(gbs / peak, 4),
               "peak_source": src, "algorithmic_bytes_per_solve": tri[2] / max(tri[0], 1),
               "ms_per_solve": round(tri[1] / max(tri[0], 1), 3),
               "note": "8 r^3 / 3 bytes of matrix reads per solve (full symmetric storage); the last ~40 % of the "
                       "columns are L2-resident and latency-bound (two grid barriers per column)",
               "eigensolve_tri_ms_per_step": round(t_ms, 3),
               "share_of_step": round(t_ms / step_ms, 4) if step_ms else None,
               "polish_jacobi": {"achieved_tflops": round(e_tf, 3), "frac": round(e_tf / FP64_PEAK_TFLOPS, 4),
                                 "share_of_step": round(e_ms / step_ms, 4) if step_ms else None}}
    return {"bound": "tensor", "kernel": label, "achieved": round(tf, 3), "peak": FP64_PEAK_TFLOPS,
            "unit": "TFLOP/s", "frac": round(tf / FP64_PEAK_TFLOPS, 4), "traffic": None,
            "peak_source": "measured FP64 DMMA peak on this pool's B200 (tools/microbench/fp64_peak.cu, "
                           "profiles/r1_fp64_peak.txt); MEASURED_PEAKS.json carries no FP64 figure",
            "share_of_step": round(ms / step_ms, 4) if step_ms else None,
            "eigensolver": eig,
            "phases_ms_per_step": {k: round(v[1] / steps, 3) for k, v in sorted(summ.items())}}


def measured_traffic(kernel_key: str):
    """DRAM bytes per launch of the family's largest kernel from the committed ncu --set full
    capture (profiles/traffic.json, written by tools/ncu_summary.py from the .ncu-rep); None
    when no capture of this workload's shape is committed."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(kernel_key)
    except (OSError, ValueError):
        return None


def like_for_like(a, H, torch, workers):
    """The reference arm's bounded instance (RefSample) on the GPU: same host-generated bytes,
    same tree and tolerances, through the public API with the input resident in HBM."""
    if a.config not in (0, 1, 3):
        return None, None
    smp = RefSample(a)
    sp = H.InnerProductSpace(smp.d)
    blk = H.SnapshotBlock(sp, smp.values)
    if a.config == 0:
        def step():
            return H.pod(blk, smp.eps_star)
    else:
        tree = H.build_star(smp.nleaves)
        leaves = H.distribute_columns(tree, blk, block_size=smp.leaf_cols)
        tol = H.assign_tolerances(tree, leaves, smp.target, omega=smp.omega)

        def step():
            return H.run_parallel(tree, leaves, tol, worker_count=min(workers, smp.nleaves))[0].modes
    for _ in range(2):
        out = step()
    clk = EventClock(torch)
    reps = 3
    with clk:
        for _ in range(reps):
            out = step()
    return smp, {"rows": smp.d, "cols": smp.m, "leaves": smp.nleaves, "b200_cols_per_s": round(smp.m * reps / (clk.ms * 1e-3), 1),
                 "b200_ms": round(clk.ms / reps, 3), "b200_modes": int(out.count)}


# ----------------------------------------------------------------------------- b200 arm
def run_b200(a, world, rank, local):
    import torch
    import torch.distributed as dist

    if a.shared_gpu_check:
        local = 0
    torch.cuda.set_device(local)
    if world > 1 and a.shared_gpu_check:
        import datetime
        dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=300))
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import _gloo_cuda_shim
        _gloo_cuda_shim.install()
    elif world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        print(f"[bench] rank {rank}/{world} on cuda:{local} ({torch.cuda.get_device_name(local)})", file=sys.stderr,
              flush=True)
    import paper_1607_05210_b200 as H
    from paper_1607_05210_b200 import _device as D
    from paper_1607_05210_b200 import _native as N
    from paper_1607_05210_b200 import distributed as DI
    from paper_1607_05210_b200 import workloads as W

    lib = N.load()
    env = dict(a=a, world=world, rank=rank, local=local, torch=torch, dist=dist, H=H, D=D, DI=DI, W=W, lib=lib)
    try:
        if a.config in (0, 1):
            line = bench_resident(**env)
        elif a.config == 2:
            line = bench_chain(**env)
        else:
            line = bench_streamed_tree(**env)
    finally:
        if world > 1:
            dist.barrier()
    if rank == 0 and line is not None:
        if world > 1 and a.shared_gpu_check:
            line["metric"] = "shared-gpu-check (NOT a measurement: all ranks time-slice one GPU over gloo)"
            line["comm"] = {"backend": "gloo", "nranks": dist.get_world_size()}
        elif world > 1:
            line["comm"] = {"backend": "nccl", "nranks": dist.get_world_size(),
                            "nccl_version": ".".join(str(x) for x in torch.cuda.nccl.version())}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def allmax_ms(ms, world, torch, dist):
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def allsum_int(v, world, torch, dist):
    if world > 1:
        t = torch.tensor([v], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        v = int(t.item())
    return v


def base_line(a, world, cols_per_s, step_ms, scaling, data, parallelism, e2e, launches, roofline, cpu, clk, extra=None):
    line = {"metric": METRIC, "value": round(cols_per_s, 3), "unit": "cols/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(step_ms, 3), "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": data, "config": static_config(a),
            "parallelism": parallelism, "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline,
            "cpu_baseline": cpu, "clocks": clk}
    if extra:
        line.update(extra)
    return line


def cpu_baseline_sample(a):
    """cpu_baseline of the b200 line: the reference arm's bounded instance, run once (N=1)."""
    cores, threads, blas, model = cpu_info()
    smp = RefSample(a)
    times, modes = smp.time_steps(1, 0)
    return smp, {"value": round(smp.m / times[0], 3), "unit": "cols/s", "cores": threads, "kind": "port",
                 "sample": smp.describe(), "sample_rows": smp.d, "sample_cols": smp.m, "modes": modes,
                 "seconds": round(times[0], 2), "cpu": model, "host_cores": cores, "blas": blas,
                 "full_tree_at_reduced_rows": committed_full_tree() if a.config == 1 else None}


def bench_resident(a, world, rank, local, torch, dist, H, D, DI, W, lib):
    """Configs 0 and 1: the whole snapshot matrix resident in HBM, star (or single node) tree."""
    wl = W.make(a.config, d=a.d)
    d, m = wl.d, wl.m
    nleaves = max(1, m // wl.block)
    tree = H.build_star(nleaves) if nleaves > 1 else H.RootedTree(((),), 0)
    maps = H.derive_maps(tree)
    place = DI.plan_placement(tree, world, maps)
    my_leaves = [leaf for leaf in maps.leaf_order if place[leaf] == rank]
    col0 = {leaf: i * wl.block for i, leaf in enumerate(maps.leaf_order)}
    sp = H.InnerProductSpace(d)
    full = H.SnapshotBlock(sp, wl.values)
    leaf_blocks = {leaf: full.column_block(col0[leaf], col0[leaf] + wl.block) for leaf in my_leaves}
    counts = {leaf: wl.block for leaf in maps.leaf_order}
    target = H.eps_star_to_target(wl.eps_star, m)
    tol = H.assign_tolerances(tree, counts, target, omega=wl.omega)
    workers = a.workers or (min(16, len(my_leaves)) if world == 1 else 1)
    root_rows = (a.root == "rows") and nleaves > 1

    def step_device():
        if world == 1:
            la = H.LeafAssignment(leaf_blocks)
            if workers > 1:
                res, _ = H.run_parallel(tree, la, tol, worker_count=workers)
            else:
                res = H.run_hapod(tree, la, tol)
            return res.modes
        ev = DI.DeviceEvaluator(sp, leaf_blocks, tol)
        root, _, _ = DI.run_distributed(tree, ev, rank, world, place, root_rows=root_rows)
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
            out, _, _ = DI.run_distributed(tree, ev, rank, world, place, root_rows=root_rows)
        if out is not None:
            np.asarray(out.sigmas).sum()  # sigmas already read back to the host
        return out

    summ_root = {}
    tri_extra = {}

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    prof_range = os.environ.get("HP_PROFILE_RANGE") == "1"  # ncu --profile-from-start off
    if prof_range:
        # per-kernel profiling of the timed step: launch the Jacobi sweeps directly (ncu cannot attribute
        # the kernels of a replayed CUDA graph one by one); never set for a measurement
        from paper_1607_05210_b200 import _native as _N
        _N.load().hp_set_debug(16)

    def timed(fn, steps, profile=False):
        nonlocal summ_root
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
        ms = allmax_ms(e0.elapsed_time(e1), world, torch, dist)
        launches = allsum_int(lib.hp_launch_count() - launches0, world, torch, dist)
        summary = D.Profiler.summary() if profile else None
        if profile:
            summ_root = D.Profiler.summary(tag=tree.root)
        if profile:
            tri_extra.update(D.Profiler.extra)
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
        ms_e2e, _, _, _ = timed(step_e2e, a.steps)

    cols_per_s = m * a.steps / (ms * 1e-3)
    e2e_cols = m * a.steps / (ms_e2e * 1e-3)
    h2d = allsum_int((hi - lo) * d * 8, world, torch, dist)
    if rank != 0:
        return None

    # ---- roofline (rank 0).  The root node runs alone on the GPU (the leaf wave overlaps 16
    # nodes on 16 streams, which inflates per-phase event times), so the per-kernel rates are
    # taken on the root node's launches inside the timed region.
    step_ms = ms / a.steps
    root_s = summ_root if summ_root else summ
    roofline = gemm_roofline(root_s, a.steps, step_ms,
                             "gemm_tma_kernel (FP64 DMMA GEMM engine: Gram SYRK, reconstruction, drift SYRK, CholQR "
                             "TRMM, Ritz products) on the root node", tri_extra)
    root_ms = sum(v[1] for v in root_s.values()) / a.steps
    roofline["root_share_of_step"] = round(root_ms / step_ms, 4)
    roofline["all_phases_ms_per_step (leaf wave overlapped)"] = {k: round(v[1] / a.steps, 3) for k, v in summ.items()}
    if a.config == 1 and a.d is None:
        tr = measured_traffic("gram_syrk_m8192_d200000")
        if tr:
            roofline["traffic"] = tr["dram_bytes"]
            roofline["traffic_algorithmic"] = tr["algorithmic_bytes"]
            roofline["traffic_source"] = tr["source"]

    cpu, lfl = None, None
    if world == 1 and not a.no_cpu:
        smp, cpu = cpu_baseline_sample(a)
        _, lfl = like_for_like(a, H, torch, workers)
        if lfl is not None:
            lfl["cpu_cols_per_s"] = cpu["value"]
            lfl["note"] = "both arms on the reference arm's bounded instance (host-generated bytes, input resident)"

    res_modes = int(out.count) if out is not None else None
    par = (f"tree over {world} GPU(s); leaf wave on {workers} stream worker(s) per GPU"
           + (f"; root on {world} row blocks (8 fixed row shards, fixed-tree sum)" if world > 1 and root_rows else ""))
    e2e = {"value": round(e2e_cols, 3), "unit": "cols/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": 8 * (res_modes or 0),
           "modes_d2h_bytes_if_requested": 8 * d * (res_modes or 0),
           "note": "sigmas read back; the final ModeSet stays device-resident (SURVEY.md 8d); under the upload-bound leaf wave run_parallel accumulates the root Gramian child pair by child pair (bit-identical to the monolithic launch)"}
    return base_line(a, world, cols_per_s, step_ms, "strong",
                     "synthetic (seeded on device, BASELINE config generator; no dataset involved)", par, e2e,
                     launches, roofline, cpu, clk,
                     {"result": {"modes": res_modes, "eps_star": wl.eps_star, "target": target},
                      "like_for_like": lfl})


def bench_chain(a, world, rank, local, torch, dist, H, D, DI, W, lib):
    """Config 2: incremental HAPOD over 64 streamed slices (one resident at a time).  The chain is
    sequential -- 'replicas only': with --gpus N every rank runs its own replica and the value is
    N x cols / max-over-ranks time (weak scaling)."""
    cfg = W.CONFIGS[2]
    d = a.d or cfg["d"]
    m, blk = cfg["m"], cfg["block"]
    nsl = m // blk
    fro = W.frobenius_norm(2, d=d)
    eps_star = cfg["rel"] * fro
    target = H.eps_star_to_target(eps_star, m)
    sp = H.InnerProductSpace(d)
    pinned = torch.empty((blk, d), dtype=torch.float64, pin_memory=True)

    def one_pass(e2e: bool, clock: EventClock):
        sess = H.incremental_open(target, cfg["omega"], nsl)
        for b in range(nsl):
            vals = W.slice_values(2, b, d=d)          # generated untimed
            if e2e:
                pinned.copy_(vals.t())
                del vals
                torch.cuda.synchronize()
                with clock:                            # H2D from pinned memory + finiteness check + merge
                    sess.push(H.SnapshotBlock(sp, pinned.t()))
            else:
                block = H.SnapshotBlock(sp, vals)      # resident slice (checked), untimed
                with clock:
                    sess.push(block)
                del block, vals
        with clock:
            res = sess.finalize()
            if e2e:
                np.asarray(res.modes.sigmas).sum()
        return res

    for _ in range(min(a.warmup, 1)):
        one_pass(False, EventClock(torch))
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    D.Profiler.reset(True)
    launches0 = lib.hp_launch_count()
    clock = EventClock(torch)
    for _ in range(a.steps):
        res = one_pass(False, clock)
    launches = allsum_int(lib.hp_launch_count() - launches0, world, torch, dist)
    summ = D.Profiler.summary()
    D.Profiler.reset(False)
    clk = clocks.stop()
    ms = allmax_ms(clock.ms, world, torch, dist)
    ms_e2e = float("nan")
    if not a.no_e2e:
        ce = EventClock(torch)
        for _ in range(a.steps):
            one_pass(True, ce)
        ms_e2e = allmax_ms(ce.ms, world, torch, dist)
    if rank != 0:
        return None
    step_ms = ms / a.steps
    roofline = gemm_roofline(summ, a.steps, step_ms, "gemm_tma_kernel (block Gram + merge reconstruction + drift)")
    cpu = None
    if world == 1 and not a.no_cpu:
        _, cpu = cpu_baseline_sample(a)
    e2e = {"value": round(world * m * a.steps / (ms_e2e * 1e-3), 3), "unit": "cols/s",
           "h2d_bytes_per_step": world * m * d * 8, "d2h_bytes_per_step": 8 * int(res.mode_count),
           "note": "every slice uploaded from pinned host memory inside the timed region"}
    return base_line(a, world, world * m * a.steps / (ms * 1e-3), step_ms, "weak",
                     "synthetic (seeded on device per slice; generation outside the timed intervals)",
                     f"{world} independent chain replica(s) (a chain does not shard: replicas only)", e2e, launches,
                     roofline, cpu, clk, {"result": {"modes": int(res.mode_count), "eps_star": eps_star,
                                                     "target": target}})


def bench_streamed_tree(a, world, rank, local, torch, dist, H, D, DI, W, lib):
    """Configs 3 and 4: snapshot sets larger than HBM, leaves generated on the device one at a time
    (generation time measured with CUDA events and subtracted).  Config 4: 8 chains of 16 slices
    under a root, chains placed on ranks; config 3: star(64), its 306 GB root input needs the
    row-distributed root on >= 4 GPUs (on fewer GPUs only the 64 leaf PODs are timed and the
    line says so)."""
    idx = a.config
    cfg = W.CONFIGS[idx]
    d = a.d or cfg["d"]
    m, blk = cfg["m"], cfg["block"]
    tree = chains_under_root(H, 8, 16) if idx == 4 else H.build_star(m // blk)
    maps = H.derive_maps(tree)
    order = maps.leaf_order
    slice_of = {leaf: i for i, leaf in enumerate(order)}
    counts = {leaf: blk for leaf in order}
    eps_star = cfg["rel"] * W.frobenius_norm(idx, d=d)
    target = H.eps_star_to_target(eps_star, m)
    tol = H.assign_tolerances(tree, counts, target, omega=cfg["omega"], zero_leaf_tolerance=(idx == 4))
    sp = H.InnerProductSpace(d)
    place = DI.plan_placement(tree, world, maps)
    leaves_only = (idx == 3 and world < 4 and d * 19_200 * 8 > 100e9)
    gen = EventClock(torch)

    def source(v):
        with gen:
            return H.SnapshotBlock(sp, W.slice_values(idx, slice_of[v], d=d))

    class StreamEvaluator(DI.DeviceEvaluator):
        def evaluate_leaf(self, node):
            from paper_1607_05210_b200.pod import pod
            return pod(source(node), self.tol.epsilons[node], self.backend)

    def step():
        if leaves_only:
            n = 0
            for leaf in order:
                if place[leaf] == rank:
                    n = H.pod(source(leaf), tol.epsilons[leaf]).count
            return n
        if world == 1:
            return H.run_hapod_streaming(tree, source, counts, tol).mode_count
        ev = StreamEvaluator(sp, {}, tol)
        root, _, _ = DI.run_distributed(tree, ev, rank, world, place, root_rows=(idx == 3))
        return root.count if root is not None else 0

    for _ in range(min(a.warmup, 1)):
        step()
    gen.ms = 0.0
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    D.Profiler.reset(True)
    launches0 = lib.hp_launch_count()
    total = EventClock(torch)
    with total:
        for _ in range(a.steps):
            modes = step()
    launches = allsum_int(lib.hp_launch_count() - launches0, world, torch, dist)
    summ = D.Profiler.summary()
    D.Profiler.reset(False)
    clk = clocks.stop()
    ms = allmax_ms(total.ms - gen.ms, world, torch, dist)
    if rank != 0:
        return None
    step_ms = ms / a.steps
    roofline = gemm_roofline(summ, a.steps, step_ms, "gemm_tma_kernel (Gram / reconstruction / drift / CholQR)")
    cpu = None
    if world == 1 and not a.no_cpu:
        _, cpu = cpu_baseline_sample(a)
    note = ("64 leaf PODs only: the 306 GB root input needs the row-distributed root on >= 4 GPUs" if leaves_only
            else "whole tree")
    return base_line(a, world, m * a.steps / (ms * 1e-3), step_ms, "strong",
                     "synthetic (seeded on device per leaf; generation time measured with CUDA events and subtracted)",
                     f"tree over {world} GPU(s), leaves streamed ({note})", None, launches, roofline, cpu, clk,
                     {"result": {"modes": int(modes), "eps_star": eps_star, "target": target, "timed": note}})


# ----------------------------------------------------------------------------- main
def main() -> int:
    a = parse()
    in_torchrun = "WORLD_SIZE" in os.environ and "RANK" in os.environ
    if a.gpus > 1 and not in_torchrun:
        if a.impl == "reference":
            return run_reference(a, a.gpus, 0)   # rank 0 alone runs the CPU arm
        return self_launch(a)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        return run_reference(a, world, rank)
    if a.protocol_check:
        return run_protocol_check(a, world, rank)
    return run_b200(a, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
