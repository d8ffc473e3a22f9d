"""Summarise the ncu outputs of tools/ncu_round.sh into small text files for profiles/.

    python tools/ncu_summary.py <round tag>      e.g. r1b

  <tag>_launches.csv      -> profiles/<tag>_launch_summary.txt   (per-kernel launches / time / share)
  <tag>_*.ncu-rep          -> profiles/<tag>_<name>_metrics.txt  (key metrics of the --set full capture)
"""
import collections
import csv
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles")

KEYS = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_active.avg", "sm__cycles_elapsed.avg"]


def launches():
    path = os.path.join(src, f"{tag}_launches.csv")
    if not os.path.exists(path):
        return
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "nsecond": 1e-6}
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values())
    n = sum(a[0] for a in agg.values())
    out = [f"# ncu launch list of the bench timed step ({tag}): {n} launches, {tot:.2f} ms summed "
           f"(serialised, cold-cache, per-launch gpu__time_duration.sum)",
           f"{'kernel':60s} {'launches':>9s} {'ms':>10s} {'share':>7s}"]
    for k, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:60s} {c:9d} {ms:10.3f} {100 * ms / tot:6.2f}%")
    open(os.path.join(dst, f"{tag}_launch_summary.txt"), "w").write("\n".join(out) + "\n")
    print("\n".join(out[:25]))


def traffic(h, u, v, source):
    """profiles/traffic.json (read by bench.py's roofline.traffic): DRAM bytes of the config-1 root
    Gram SYRK launch from its ncu --set full capture."""
    import json
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

    def val(k):
        i = h.index(k)
        return float(v[i].replace(",", "")) * scale.get(u[i], 1.0)

    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    i = h.index("gpu__time_duration.sum")
    ms = float(v[i].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(u[i].replace("econd", ""), 1.0)
    entry = {"kernel": "gemm_tma_kernel<1, 1, 4> (root Gram SYRK, m = 8192, d = 200000)",
             "dram_bytes": int(rd + wr), "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
             "algorithmic_bytes": 13650000000, "duration_ms": ms,
             "source": f"{source} (ncu --set full --clock-control none: dram__bytes_read.sum + "
                       f"dram__bytes_write.sum of one launch)"}
    path = os.path.join(dst, "traffic.json")
    try:
        data = json.load(open(path))
    except (OSError, ValueError):
        data = {}
    data["gram_syrk_m8192_d200000"] = entry
    json.dump(data, open(path, "w"), indent=1)
    print("traffic.json:", entry)


def reports():
    for rep in sorted(glob.glob(os.path.join(src, f"{tag}_*.ncu-rep"))):
        name = os.path.basename(rep)[len(tag) + 1: -len(".ncu-rep")]
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(txt.splitlines()))
        if len(rows) < 3:
            continue
        h, u = rows[0], rows[1]
        out = [f"# ncu --set full --clock-control none: {name} ({tag})"]
        for v in rows[2:]:
            for k in KEYS:
                if k in h:
                    i = h.index(k)
                    out.append(f"{k:70s} {v[i]} {u[i]}")
            st = []
            for i, k in enumerate(h):
                if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                    try:
                        st.append((float(v[i]), k))
                    except ValueError:
                        pass
            for x, k in sorted(st, reverse=True)[:6]:
                out.append(f"{k:70s} {x:.3f}")
            out.append("")
        open(os.path.join(dst, f"{tag}_{name}_metrics.txt"), "w").write("\n".join(out) + "\n")
        print("\n".join(out))
        if name == "gemm_gram8192":
            traffic(h, u, rows[2], f"profiles/{tag}_{name}_metrics.txt")


launches()
reports()
