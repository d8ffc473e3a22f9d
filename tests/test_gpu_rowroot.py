"""The row-distributed root (rowroot.py) with the device arithmetic (DeviceRowArith: the
libhapod_b200.so kernels) over NCCL, at world size 1 -- the only multi-process configuration a
single B200 admits.  The protocol itself (row all-to-all, reductions, broadcast, sign
resolution across ranks) is covered at world sizes 2 and 3 on CPU by
test_distributed_gloo.py::test_row_distributed_root_matches_oracle."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

import paper_1607_05210_b200 as H  # noqa: E402
from paper_1607_05210_b200 import distributed as DI  # noqa: E402
from paper_1607_05210_b200 import workloads as W  # noqa: E402
from oracle import hapod_oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def nccl_group():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


# The row root sums its Gram over 8 fixed row shards (bitwise independent of the rank count), the
# gathered root over all rows at once: the two differ by the Gram's summation order, i.e. by the
# CPU-vs-CPU "row-permuted" floor of the same workload.  Floors (max rel dsigma, max angle sine)
# are the ones test_gpu_configs.py measures with the oracle on these exact shapes
# (c1-mini: 1.2e-6 / 2.3e-4; c3-mini: 4.9e-8 / 2.5e-8); gate = max(BASELINE gate, 4 x floor).
@pytest.mark.parametrize("config,d,nleaves,frel,fang", [(1, 6000, 4, 1.2e-6, 2.3e-4), (3, 8000, 8, 4.9e-8, 2.5e-8)])
def test_row_root_device_matches_gathered_root(nccl_group, config, d, nleaves, frel, fang):
    m = 512 * nleaves
    wl = W.make(config, d=d, m=m)
    sp = H.InnerProductSpace(d)
    tree = H.build_star(nleaves)
    blk = H.SnapshotBlock(sp, wl.values)
    leaves = H.distribute_columns(tree, blk, block_size=512)
    tol = H.assign_tolerances(tree, leaves, H.eps_star_to_target(wl.eps_star, m), omega=wl.omega)
    ref = H.run_hapod(tree, leaves, tol)
    ev = DI.DeviceEvaluator(sp, dict(leaves.blocks), tol)
    root, _, _ = DI.run_distributed(tree, ev, 0, 1, root_rows=True)
    n = min(root.count, ref.mode_count)
    rel = np.abs(root.sigmas[:n] - ref.modes.sigmas[:n]) / ref.modes.sigmas[:n]
    ang = O.principal_angle_sines(root.modes, ref.modes.modes)
    g = root.modes.T @ root.modes
    print(f"\n[row root c{config} d={d} m={m}] counts rows={root.count} gathered={ref.mode_count} "
          f"max rel dsigma={rel.max():.2e} max angle sine={ang.max():.2e} "
          f"orthonormality={np.abs(g - np.eye(g.shape[0])).max():.1e}")
    assert root.count == ref.mode_count
    assert rel.max() <= max(1e-10, 4.0 * frel)
    assert np.median(rel) <= 1e-10          # the well-conditioned bulk agrees to the BASELINE gate
    assert ang.max() <= max(1e-8, 4.0 * fang)
    assert np.abs(g - np.eye(g.shape[0])).max() < 1e-8  # reference: re-orthonormalise above 1e-8 drift
    # same sign convention: the largest-|.| entry of every mode is positive
    idx = np.argmax(np.abs(root.modes), axis=0)
    assert np.all(root.modes[idx, np.arange(root.count)] > 0)
