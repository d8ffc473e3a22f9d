"""bench.py's N > 1 code path (launch, placement, DeviceEvaluator edges, row-distributed root,
max-over-ranks timing, summed launch counts and H2D bytes, the e2e leg) rehearsed with 2 ranks that
share this box's one GPU (``--shared-gpu-check``: gloo + host-staged tensors instead of NCCL).
Not a measurement -- the line says so -- but the same Python that a multi-GPU node runs."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=900, env=env, cwd=ROOT)
    assert p.returncode == 0, (p.stdout[-1500:], p.stderr[-3000:])
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("root", ["rows", "gather"])
def test_bench_two_ranks_on_one_gpu(root):
    common = ["--d", "6000", "--steps", "1", "--warmup", "1", "--no-cpu"]
    one = _bench(common)
    two = _bench(common + ["--gpus", "2", "--shared-gpu-check", "--root", root])
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["comm"] == {"backend": "gloo", "nranks": 2}
    assert "NOT a measurement" in two["metric"]
    assert two["config"] == one["config"]
    assert two["result"]["modes"] == one["result"]["modes"] > 0
    assert two["gpu_launches"] > 0 and two["e2e"]["h2d_bytes_per_step"] == one["e2e"]["h2d_bytes_per_step"]
    assert two["value"] > 0 and two["e2e"]["value"] > 0


@pytest.mark.parametrize("config,d", [(4, 1500), (3, 1500), (2, 3000)])
def test_bench_streamed_configs_two_ranks_on_one_gpu(config, d):
    """The streamed legs at N = 2: config 4 (chains placed on ranks + gathered root), config 3 (streamed
    leaves + row-distributed root), config 2 (independent replicas) -- same mode counts as N = 1."""
    common = ["--config", str(config), "--d", str(d), "--steps", "1", "--warmup", "0", "--no-cpu", "--no-e2e"]
    one = _bench(common)
    two = _bench(common + ["--gpus", "2", "--shared-gpu-check"])
    assert two["n_gpus"] == 2 and two["config"] == one["config"]
    assert two["result"]["modes"] == one["result"]["modes"] > 0
    assert two["scaling"] == ("weak" if config == 2 else "strong")
