"""The multi-rank DEVICE path -- DeviceEvaluator edges, the row-distributed root with its row
all-to-all, fixed-tree Gram sum, REPLICATED eigensolve (hp_syev_rows shares + all-gather), global
drift / CholQR / sign resolution -- executed by 2 and 3 processes that share this box's one GPU,
over gloo with host-staged tensors (tests/_gloo_cuda_shim.py; production uses NCCL, which refuses
two ranks on one device).  The distributed result must equal the single-process device run:
identical counts, sigma and modes to rounding.  Replaces nothing in the NCCL path; it checks the
rank logic that otherwise first runs on a multi-GPU node."""

import datetime
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402


def _problem():
    import paper_1607_05210_b200 as H
    from oracle import hapod_oracle as O
    d, nl, lc = 2600, 6, 96
    vals = O.synthetic_decay(d, nl * lc, 0.03, seed=11)
    tree = H.build_star(nl)
    target = 1e-5 * float(np.linalg.norm(vals)) / np.sqrt(nl * lc)
    return H, vals, tree, nl, lc, d, target


def _worker(rank, world, port, root_rows, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=120))
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        import _gloo_cuda_shim
        _gloo_cuda_shim.install()
        from paper_1607_05210_b200 import distributed as DI
        H, vals, tree, nl, lc, d, target = _problem()
        maps = H.derive_maps(tree)
        place = DI.plan_placement(tree, world, maps)
        sp = H.InnerProductSpace(d)
        counts = {leaf: lc for leaf in maps.leaf_order}
        tol = H.assign_tolerances(tree, counts, target, omega=0.75)
        blocks = {leaf: H.SnapshotBlock(sp, vals[:, lc * i: lc * (i + 1)])
                  for i, leaf in enumerate(maps.leaf_order) if place[leaf] == rank}
        ev = DI.DeviceEvaluator(sp, blocks, tol)
        root, _, stats = DI.run_distributed(tree, ev, rank, world, place, root_rows=root_rows)
        if rank == 0:
            out_q.put(("ok", np.asarray(root.sigmas), np.asarray(root.modes), root.diagnostics.get("nkeep")))
        else:
            out_q.put(("ok", None, None, stats.sends))
    except Exception as exc:  # surface the failure instead of hanging the peer
        import traceback
        out_q.put(("fail", f"rank {rank}: {exc}\n{traceback.format_exc()}", None, None))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_ranks(world, root_rows):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, root_rows, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        msgs = [q.get(timeout=300) for _ in range(world)]
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    fails = [m[1] for m in msgs if m[0] == "fail"]
    assert not fails, fails[0]
    return next((m[1], m[2], m[3]) for m in msgs if m[1] is not None)


def test_row_distributed_root_is_bitwise_independent_of_the_rank_count():
    """SURVEY.md H5 / reference tests/test_parallel.py:50-58 (bit-identical across worker counts): the
    8 fixed row shards and the fixed-tree Gram sum make the root's bits the same for 2 and 3 ranks."""
    s2, m2, _ = _run_ranks(2, True)
    s3, m3, _ = _run_ranks(3, True)
    assert np.array_equal(s2, s3) and np.array_equal(m2, m3)


@pytest.mark.parametrize("world,root_rows", [(2, True), (3, True), (2, False)])
def test_device_ranks_sharing_one_gpu_match_single_process(world, root_rows):
    sig, modes, nkeep = _run_ranks(world, root_rows)

    H, vals, tree, nl, lc, d, target = _problem()
    sp = H.InnerProductSpace(d)
    leaves = H.distribute_columns(tree, H.SnapshotBlock(sp, vals), block_size=lc)
    tol = H.assign_tolerances(tree, leaves, target, omega=0.75)
    ref = H.run_hapod(tree, leaves, tol)
    rs, rm = np.asarray(ref.modes.sigmas), np.asarray(ref.modes.modes)
    print(f"\n[{world} ranks on one GPU, root_rows={root_rows}] modes {len(sig)} vs {len(rs)}; max rel dsigma "
          f"{np.max(np.abs(sig - rs) / rs):.2e}; max |dU| {np.max(np.abs(modes - rm)):.2e}")
    assert len(sig) == len(rs)
    if not root_rows:
        # gathered root: the very kernels of the single-process run on the very same bytes
        assert np.array_equal(sig, rs) and np.array_equal(modes, rm)
    else:
        # row-distributed root: Gram summed over 8 fixed row shards (a different, fixed, summation order)
        # method-of-snapshots floor: a Gram rounding of u * sigma_1^2 moves sigma_i by u * sigma_1^2 / (2 sigma_i)
        assert np.all(np.abs(sig - rs) <= 64.0 * 2.0 ** -53 * rs[0] ** 2 / rs)
        from oracle import hapod_oracle as O
        # subspaces: the leading half to 1e-8; the full span, whose last modes sit at the method-of-snapshots
        # floor u sigma_1^2 / (gap sigma_N^2), through the projection error it leaves
        k = len(sig) // 2
        assert O.principal_angle_sines(modes[:, :k], rm[:, :k]).max() < 1e-8
        e_d = np.linalg.norm(vals - modes @ (modes.T @ vals))
        e_r = np.linalg.norm(vals - rm @ (rm.T @ vals))
        assert abs(e_d - e_r) <= 1e-8 * e_r
        assert np.max(np.abs(modes.T @ modes - np.eye(len(sig)))) < 1e-8
