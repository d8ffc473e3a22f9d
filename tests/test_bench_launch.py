"""bench.py's launch paths on CPU: `--gpus 2` outside torchrun must start two ranks itself
(torch.distributed.run on 127.0.0.1) and rank 0 must print ONE JSON line; the reference arm must
run without importing the product package (so the driver sees no repo .so mapped); the static
config printed by both arms must be identical."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_gpus2_self_launch_protocol_on_gloo():
    line = _run(["--gpus", "2", "--protocol-check"])
    assert line["ranks"] == 2 and line["backend"] == "gloo"
    assert line["edges_received_on_rank0"] == 4          # star(8): leaves 5..8 live on rank 1
    assert line["bitwise_equal_to_single_process"] is True


def test_reference_arm_is_host_only_and_labels_its_sample():
    code = (
        "import sys, json, runpy\n"
        f"sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0', "
        "'--ref-d', '600', '--ref-leaf-cols', '8']\n"
        f"sys.path.insert(0, {ROOT!r})\n"
        "try:\n"
        f"    runpy.run_path({os.path.join(ROOT, 'bench.py')!r}, run_name='__main__')\n"
        "except SystemExit as e:\n"
        "    assert not e.code\n"
        "assert not any(m.startswith('paper_1607_05210_b200') for m in sys.modules), 'product imported'\n"
        "assert 'torch' not in sys.modules, 'torch imported by the reference arm'\n"
        "maps = open('/proc/self/maps').read()\n"
        "assert 'libhapod_b200' not in maps\n"
    )
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][0])
    assert line["impl"] == "reference" and line["unit"] == "cols/s" and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["sample_rows"] == 600 and cb["sample_cols"] == 128 and "root" in cb["sample"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    # the same static config as the b200 arm prints
    sys.path.insert(0, ROOT)
    import bench
    a = type("A", (), {"config": 1, "d": None})()
    assert line["config"] == bench.static_config(a)


def test_reference_arm_under_torchrun_runs_on_rank0_only():
    """N > 1: rank 0 alone runs and prints the reference line; the other ranks exit 0 without work."""
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1", MASTER_ADDR="127.0.0.1", MASTER_PORT="29999")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert p.returncode == 0 and p.stdout.strip() == ""
    env["RANK"] = env["LOCAL_RANK"] = "0"
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
                        "--warmup", "0", "--ref-d", "500", "--ref-leaf-cols", "6"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-1500:]
    line = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2


def test_gpus_more_than_visible_is_refused_loudly():
    """--gpus N on a box with fewer GPUs must not silently run on one: an error line and a non-zero exit."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "64"], capture_output=True, text=True,
                       timeout=120, env=env, cwd=ROOT)
    assert p.returncode == 2
    line = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][0])
    assert "error" in line and line["n_gpus"] == 64
